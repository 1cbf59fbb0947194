/* oracle/mlip_oracle.c — TEST INFRASTRUCTURE: fp64 CPU restatement of the
 * four-phase training step (see mlip_oracle.h for scope and pinning).
 *
 * Deliberately written as the plain DEFINITIONS, not the GPU's algorithm:
 *  - transposed aggregations are scatters over sender j (CSC meaning), not
 *    the GPU's symmetric-CSR gathers;
 *  - forces use both endpoints explicitly: F_i += q u, F_j -= q u;
 *  - every per-edge quantity is recomputed from positions in fp64.
 * Phase semantics: PAPER.md:171-178; gradient routing Eq. (2) PAPER.md:323-332;
 * dependency/flow directions graph.hpp:133-153 (FE up, FF down, BF up, BE down).
 */
#include "mlip_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define ALLOC(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

/* ------------------------------------------------------------------ model */
int mo_num_units(const mo_model* m) { return 2 * m->L + 2; }

int64_t mo_unit_param_count(const mo_model* m, int unit) {
  const int64_t H = m->H, R = m->R, S = m->n_species;
  if (unit == 0) return S * H;
  if (unit == 2 * m->L + 1) return H * H + 2 * H + S;
  if (unit % 2 == 1) return R * H + H + H * H + H + H * H; /* msg */
  return H * H + H + H * H;                                /* upd */
}

int64_t mo_unit_param_offset(const mo_model* m, int unit) {
  int64_t off = 0;
  for (int u = 0; u < unit; ++u) off += mo_unit_param_count(m, u);
  return off;
}

int64_t mo_param_count(const mo_model* m) { return mo_unit_param_offset(m, mo_num_units(m)); }

/* --------------------------------------------------------------- SiLU etc */
static double sig(double x) { return 1.0 / (1.0 + exp(-x)); }
static double silu(double x) { return x * sig(x); }
static double dsilu(double x) {
  const double s = sig(x);
  return s * (1.0 + x * (1.0 - s));
}
static double d2silu(double x) {
  const double s = sig(x);
  return s * (1.0 - s) * (2.0 + x * (1.0 - 2.0 * s));
}

/* -------------------------------------------------------- neighbour list */
static int struct_range(const mo_batch* b, int s, int* begin) {
  int n = 0, first = -1;
  for (int i = 0; i < b->n_atoms; ++i) {
    if (b->struct_id[i] == s) {
      if (first < 0) first = i;
      ++n;
    }
  }
  *begin = first;
  return n;
}

int64_t mo_build_nbrlist(const mo_model* m, const mo_batch* b, int64_t max_edges, int* row_ptr,
                         int* col, int* shift, int* rev) {
  const double rc2 = m->r_c * m->r_c;
  int64_t E = 0;
  row_ptr[0] = 0;
  for (int i = 0; i < b->n_atoms; ++i) {
    const int s = b->struct_id[i];
    const double Lb = b->cell[s];
    int first;
    const int n_in = struct_range(b, s, &first);
    const int nimg = (int)ceil(m->r_c / Lb);
    for (int j = first; j < first + n_in; ++j) {
      for (int sx = -nimg; sx <= nimg; ++sx)
        for (int sy = -nimg; sy <= nimg; ++sy)
          for (int sz = -nimg; sz <= nimg; ++sz) {
            if (i == j && sx == 0 && sy == 0 && sz == 0) continue;
            const double* xi = b->pos + 3 * i;
            const double* xj = b->pos + 3 * j;
            volatile double rx = (xj[0] + sx * Lb) - xi[0];
            volatile double ry = (xj[1] + sy * Lb) - xi[1];
            volatile double rz = (xj[2] + sz * Lb) - xi[2];
            volatile double ax = rx * rx, ay = ry * ry, az = rz * rz;
            volatile double d2 = (ax + ay) + az;
            if (!(d2 < rc2)) continue;
            if (E >= max_edges) return -1;
            col[E] = j;
            shift[3 * E + 0] = sx;
            shift[3 * E + 1] = sy;
            shift[3 * E + 2] = sz;
            ++E;
          }
    }
    row_ptr[i + 1] = (int)E;
  }
  for (int64_t e = 0; e < E; ++e) rev[e] = -1;
  for (int i = 0; i < b->n_atoms; ++i) {
    for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const int j = col[e];
      for (int f = row_ptr[j]; f < row_ptr[j + 1]; ++f) {
        if (col[f] == i && shift[3 * f] == -shift[3 * e] && shift[3 * f + 1] == -shift[3 * e + 1] &&
            shift[3 * f + 2] == -shift[3 * e + 2]) {
          rev[e] = f;
          break;
        }
      }
    }
  }
  return E;
}

/* ----------------------------------------------------------- edge geometry */
typedef struct {
  int N, E, H, R;
  const int *row_ptr, *col, *rev;
  int* src; /* receiver i of edge e */
  double *d, *u, *c, *dc;
  double *phi, *dphi; /* [E][R] */
} Geo;

static void geo_build(Geo* g, const mo_model* m, const mo_batch* b, int64_t E, const int* row_ptr,
                      const int* col, const int* shift, const int* rev) {
  g->N = b->n_atoms;
  g->E = (int)E;
  g->H = m->H;
  g->R = m->R;
  g->row_ptr = row_ptr;
  g->col = col;
  g->rev = rev;
  g->src = ALLOC(int, E);
  g->d = ALLOC(double, E);
  g->u = ALLOC(double, 3 * E);
  g->c = ALLOC(double, E);
  g->dc = ALLOC(double, E);
  g->phi = ALLOC(double, E * m->R);
  g->dphi = ALLOC(double, E * m->R);
  const double rc = m->r_c;
  const double delta = rc / (m->R - 1);
  const double gamma = 1.0 / (2.0 * delta * delta);
  for (int i = 0; i < b->n_atoms; ++i) {
    const double Lb = b->cell[b->struct_id[i]];
    for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const int j = col[e];
      double r[3];
      for (int k = 0; k < 3; ++k) r[k] = (b->pos[3 * j + k] + shift[3 * e + k] * Lb) - b->pos[3 * i + k];
      const double d = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
      g->src[e] = i;
      g->d[e] = d;
      for (int k = 0; k < 3; ++k) g->u[3 * e + k] = r[k] / d;
      const double arg = M_PI * d / rc;
      g->c[e] = d < rc ? 0.5 * (cos(arg) + 1.0) : 0.0;
      g->dc[e] = d < rc ? -0.5 * (M_PI / rc) * sin(arg) : 0.0;
      for (int k = 0; k < m->R; ++k) {
        const double mu = k * delta;
        const double x = d - mu;
        const double p = exp(-gamma * x * x);
        g->phi[(int64_t)e * m->R + k] = p;
        g->dphi[(int64_t)e * m->R + k] = -2.0 * gamma * x * p;
      }
    }
  }
}

static void geo_free(Geo* g) {
  free(g->src);
  free(g->d);
  free(g->u);
  free(g->c);
  free(g->dc);
  free(g->phi);
  free(g->dphi);
}

/* ----------------------------------------------------------- small linalg */
/* out[M][N] (+)= in[M][K] W[K][N] */
static void mm(int M, int K, int N, const double* in, const double* W, double* out, int acc) {
  for (int i = 0; i < M; ++i) {
    double* o = out + (int64_t)i * N;
    if (!acc) memset(o, 0, sizeof(double) * (size_t)N);
    for (int k = 0; k < K; ++k) {
      const double a = in[(int64_t)i * K + k];
      const double* w = W + (int64_t)k * N;
      for (int n = 0; n < N; ++n) o[n] += a * w[n];
    }
  }
}
/* out[M][K] (+)= in[M][N] W^T, W[K][N] */
static void mmT(int M, int N, int K, const double* in, const double* W, double* out, int acc) {
  for (int i = 0; i < M; ++i) {
    for (int k = 0; k < K; ++k) {
      double s = 0;
      for (int n = 0; n < N; ++n) s += in[(int64_t)i * N + n] * W[(int64_t)k * N + n];
      out[(int64_t)i * K + k] = (acc ? out[(int64_t)i * K + k] : 0.0) + s;
    }
  }
}
/* G[K][N] += a[M][K]^T b[M][N] */
static void wgrad(int M, int K, int N, const double* a, const double* b, double* G) {
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) {
      const double x = a[(int64_t)i * K + k];
      for (int n = 0; n < N; ++n) G[(int64_t)k * N + n] += x * b[(int64_t)i * N + n];
    }
}
/* vec[K] (+)= v[K] M[K][N]... per-edge row ops */
static void vecmat(int K, int N, const double* v, const double* W, double* out) {
  for (int n = 0; n < N; ++n) out[n] = 0.0;
  for (int k = 0; k < K; ++k) {
    const double a = v[k];
    for (int n = 0; n < N; ++n) out[n] += a * W[(int64_t)k * N + n];
  }
}
static void vecmatT(int N, int K, const double* v, const double* W, double* out) {
  /* out[k] = sum_n v[n] W[k][n] */
  for (int k = 0; k < K; ++k) {
    double s = 0;
    for (int n = 0; n < N; ++n) s += v[n] * W[(int64_t)k * N + n];
    out[k] = s;
  }
}

/* ------------------------------------------------------------ per-edge MLP */
typedef struct {
  double *z, *s, *g, *w, *zp, *sp, *gp, *wp; /* [H] each; zp = dz/dd etc. */
} EdgeVec;

static void edge_alloc(EdgeVec* v, int H) {
  double* buf = ALLOC(double, 8 * H);
  v->z = buf;
  v->s = buf + H;
  v->g = buf + 2 * H;
  v->w = buf + 3 * H;
  v->zp = buf + 4 * H;
  v->sp = buf + 5 * H;
  v->gp = buf + 6 * H;
  v->wp = buf + 7 * H;
}

/* z = phi A + alpha, s = SiLU z, g = s B + beta, w = c g;  and d/dd of each. */
static void edge_eval(const Geo* G, int e, const double* A, const double* alpha, const double* Bm,
                      const double* beta, EdgeVec* v) {
  const int H = G->H, R = G->R;
  vecmat(R, H, G->phi + (int64_t)e * R, A, v->z);
  vecmat(R, H, G->dphi + (int64_t)e * R, A, v->zp);
  for (int h = 0; h < H; ++h) {
    v->z[h] += alpha[h];
    v->s[h] = silu(v->z[h]);
    v->sp[h] = dsilu(v->z[h]) * v->zp[h];
  }
  vecmat(H, H, v->s, Bm, v->g);
  vecmat(H, H, v->sp, Bm, v->gp);
  for (int h = 0; h < H; ++h) {
    v->g[h] += beta[h];
    v->w[h] = G->c[e] * v->g[h];
    v->wp[h] = G->dc[e] * v->g[h] + G->c[e] * v->gp[h];
  }
}

/* -------------------------------------------------------------- the step */
typedef struct {
  double *h_in, *v;      /* msg: saved input h, v = hW */
  double *m_in, *p;      /* upd: saved input m, p = mU + upsilon */
  double *t;             /* readout: t = hO + o (h_in reused) */
  double *ff_am, *ff_Y;  /* msg FF intermediates */
  double* ff_a;          /* upd FF intermediate a' */
  double *inj_h, *inj_m; /* BF -> BE injections at the unit input */
} UnitSave;

static void put_trace(double* trace, int unit, int slot, const double* x, int64_t NH) {
  if (!trace || !x) return;
  memcpy(trace + ((int64_t)unit * 8 + slot) * NH, x, sizeof(double) * (size_t)NH);
}

static int run_step(const mo_model* m, const mo_batch* b, int64_t n_edges, const int* row_ptr,
                    const int* col, const int* shift, const int* rev, const double* params, double* E_out,
                    double* F_out, double* loss_out, double* grad, double* grad1, double* grad2,
                    double* trace, int energy_only) {
  const int N = b->n_atoms, H = m->H, R = m->R, L = m->L, S = m->n_species, U = mo_num_units(m);
  const int64_t NH = (int64_t)N * H;
  const int64_t NP = mo_param_count(m);
  Geo G;
  geo_build(&G, m, b, n_edges, row_ptr, col, shift, rev);
  const int Ecount = (int)n_edges;

  double* g1 = ALLOC(double, NP);
  double* g2 = ALLOC(double, NP);
  UnitSave* sv = ALLOC(UnitSave, U);
  double* Es = ALLOC(double, b->n_struct);
  double* F = ALLOC(double, 3 * N);
  EdgeVec ev;
  edge_alloc(&ev, H);
  double* tmpH = ALLOC(double, H);
  double* tmpH2 = ALLOC(double, H);
  double* tmpR = ALLOC(double, R);
  if (trace) memset(trace, 0, sizeof(double) * (size_t)(U * 8 * NH));

  /* ================================ FE ================================ */
  double* h = ALLOC(double, NH);
  double* mcar = NULL; /* m carrier (present after a msg unit) */
  for (int u = 0; u < U; ++u) {
    const double* th = params + mo_unit_param_offset(m, u);
    if (u == 0) { /* embed: h = Emb[Z] */
      for (int i = 0; i < N; ++i) memcpy(h + (int64_t)i * H, th + (int64_t)b->species[i] * H, sizeof(double) * (size_t)H);
    } else if (u == U - 1) { /* readout */
      const double *O = th, *o = th + H * H, *om = th + H * H + H, *bias = th + H * H + 2 * H;
      sv[u].h_in = ALLOC(double, NH);
      memcpy(sv[u].h_in, h, sizeof(double) * (size_t)NH);
      sv[u].t = ALLOC(double, NH);
      mm(N, H, H, h, O, sv[u].t, 0);
      for (int i = 0; i < N; ++i) {
        double e = bias[b->species[i]];
        for (int k = 0; k < H; ++k) {
          sv[u].t[(int64_t)i * H + k] += o[k];
          e += silu(sv[u].t[(int64_t)i * H + k]) * om[k];
        }
        Es[b->struct_id[i]] += e;
      }
    } else if (u % 2 == 1) { /* msg */
      const double *A = th, *alpha = A + R * H, *Bm = alpha + H, *beta = Bm + H * H, *W = beta + H;
      sv[u].h_in = ALLOC(double, NH);
      memcpy(sv[u].h_in, h, sizeof(double) * (size_t)NH);
      sv[u].v = ALLOC(double, NH);
      mm(N, H, H, h, W, sv[u].v, 0);
      free(mcar);
      mcar = ALLOC(double, NH);
      for (int e = 0; e < Ecount; ++e) {
        edge_eval(&G, e, A, alpha, Bm, beta, &ev);
        const int i = G.src[e], j = G.col[e];
        for (int k = 0; k < H; ++k) mcar[(int64_t)i * H + k] += ev.w[k] * sv[u].v[(int64_t)j * H + k];
      }
    } else { /* upd */
      const double *Um = th, *ups = Um + H * H, *V = ups + H;
      sv[u].m_in = mcar;
      mcar = NULL;
      sv[u].p = ALLOC(double, NH);
      mm(N, H, H, sv[u].m_in, Um, sv[u].p, 0);
      for (int i = 0; i < N; ++i)
        for (int k = 0; k < H; ++k) {
          sv[u].p[(int64_t)i * H + k] += ups[k];
          tmpH[k] = silu(sv[u].p[(int64_t)i * H + k]);
        }
      /* h += SiLU(p) V, row by row */
      for (int i = 0; i < N; ++i) {
        for (int k = 0; k < H; ++k) tmpH[k] = silu(sv[u].p[(int64_t)i * H + k]);
        vecmat(H, H, tmpH, V, tmpH2);
        for (int k = 0; k < H; ++k) h[(int64_t)i * H + k] += tmpH2[k];
      }
    }
    if (u < U - 1) {
      put_trace(trace, u, 0, h, NH);
      put_trace(trace, u, 1, mcar, NH);
    }
  }
  free(h);
  free(mcar);
  if (E_out) memcpy(E_out, Es, sizeof(double) * (size_t)b->n_struct);
  if (energy_only) goto cleanup;

  {
    /* ================================ FF ================================ */
    double* ah = ALLOC(double, NH); /* adjoint on h carrier at the current boundary */
    double* am = NULL;              /* adjoint on m carrier */
    for (int u = U - 1; u >= 1; --u) {
      const double* th = params + mo_unit_param_offset(m, u);
      if (u == U - 1) { /* readout seed: a = (SiLU'(t) * omega) O^T */
        const double *O = th, *om = th + H * H + H;
        for (int i = 0; i < N; ++i) {
          for (int k = 0; k < H; ++k) tmpH[k] = dsilu(sv[u].t[(int64_t)i * H + k]) * om[k];
          vecmatT(H, H, tmpH, O, ah + (int64_t)i * H);
        }
      } else if (u % 2 == 1) { /* msg */
        const double *A = th, *alpha = A + R * H, *Bm = alpha + H, *beta = Bm + H * H, *W = beta + H;
        sv[u].ff_am = am;
        am = NULL;
        sv[u].ff_Y = ALLOC(double, NH);
        for (int e = 0; e < Ecount; ++e) {
          edge_eval(&G, e, A, alpha, Bm, beta, &ev);
          const int i = G.src[e], j = G.col[e];
          double q = 0;
          for (int k = 0; k < H; ++k) {
            const double wbar = sv[u].ff_am[(int64_t)i * H + k] * sv[u].v[(int64_t)j * H + k];
            q += wbar * ev.wp[k];
            sv[u].ff_Y[(int64_t)j * H + k] += ev.w[k] * sv[u].ff_am[(int64_t)i * H + k];
          }
          for (int k = 0; k < 3; ++k) {
            F[3 * i + k] += q * G.u[3 * e + k];
            F[3 * j + k] -= q * G.u[3 * e + k];
          }
        }
        mmT(N, H, H, sv[u].ff_Y, W, ah, 1); /* a_h = a_h' + Y W^T */
      } else { /* upd: a_h = a', a_m = ((a' V^T) * SiLU'(p)) U^T */
        const double *Um = th, *V = Um + H * H + H;
        sv[u].ff_a = ALLOC(double, NH);
        memcpy(sv[u].ff_a, ah, sizeof(double) * (size_t)NH);
        am = ALLOC(double, NH);
        for (int i = 0; i < N; ++i) {
          vecmatT(H, H, ah + (int64_t)i * H, V, tmpH);
          for (int k = 0; k < H; ++k) tmpH[k] *= dsilu(sv[u].p[(int64_t)i * H + k]);
          vecmatT(H, H, tmpH, Um, am + (int64_t)i * H);
        }
      }
      put_trace(trace, u, 2, ah, NH);
      put_trace(trace, u, 3, am, NH);
    }
    free(ah);
    free(am);
    if (F_out) memcpy(F_out, F, sizeof(double) * (size_t)(3 * N));

    /* ================================ loss ============================== */
    double loss = 0;
    double* eps = ALLOC(double, b->n_struct);
    double* Fbar = ALLOC(double, 3 * N);
    for (int s = 0; s < b->n_struct; ++s) {
      const double de = Es[s] - b->E_target[s];
      loss += m->w_E * de * de;
      eps[s] = 2.0 * m->w_E * de;
    }
    for (int i = 0; i < 3 * N; ++i) {
      const double df = F[i] - b->F_target[i];
      loss += m->w_F * df * df;
      Fbar[i] = 2.0 * m->w_F * df;
    }
    if (loss_out) *loss_out = loss;
    double* qbar = ALLOC(double, Ecount);
    for (int e = 0; e < Ecount; ++e) {
      const int i = G.src[e], j = G.col[e];
      double s = 0;
      for (int k = 0; k < 3; ++k) s += (Fbar[3 * i + k] - Fbar[3 * j + k]) * G.u[3 * e + k];
      qbar[e] = s;
    }

    /* ================================ BF ================================ */
    double* abh = ALLOC(double, NH); /* tangent on the FF adjoint, unit input side */
    double* abm = NULL;
    for (int u = 1; u < U; ++u) {
      const double* th = params + mo_unit_param_offset(m, u);
      double* t2 = g2 + mo_unit_param_offset(m, u);
      if (u == U - 1) { /* readout */
        const double *O = th, *om = th + H * H + H;
        double *dO = t2, *dob = t2 + H * H, *dom = t2 + H * H + H;
        sv[u].inj_h = ALLOC(double, NH);
        for (int i = 0; i < N; ++i) {
          const double* t = sv[u].t + (int64_t)i * H;
          vecmat(H, H, abh + (int64_t)i * H, O, tmpH); /* tdot */
          for (int k = 0; k < H; ++k) {
            dom[k] += tmpH[k] * dsilu(t[k]);
            tmpH2[k] = tmpH[k] * om[k] * d2silu(t[k]); /* tau */
            dob[k] += tmpH2[k];
          }
          vecmatT(H, H, tmpH2, O, sv[u].inj_h + (int64_t)i * H);
          for (int a = 0; a < H; ++a) {
            const double x1 = abh[(int64_t)i * H + a], x2 = sv[u].h_in[(int64_t)i * H + a];
            for (int k = 0; k < H; ++k) dO[(int64_t)a * H + k] += x1 * dsilu(t[k]) * om[k] + x2 * tmpH2[k];
          }
        }
      } else if (u % 2 == 1) { /* msg */
        const double *A = th, *alpha = A + R * H, *Bm = alpha + H, *beta = Bm + H * H, *W = beta + H;
        double *dA = t2, *dalpha = dA + R * H, *dB = dalpha + H, *dbeta = dB + H * H, *dW = dbeta + H;
        double* vdot = ALLOC(double, NH);
        mm(N, H, H, abh, W, vdot, 0);
        double* mdot = ALLOC(double, NH);
        double* X = ALLOC(double, NH);
        double* mu = ALLOC(double, H);
        double* nu = ALLOC(double, H);
        double* zb = ALLOC(double, H);
        double* zpb = ALLOC(double, H);
        for (int e = 0; e < Ecount; ++e) {
          edge_eval(&G, e, A, alpha, Bm, beta, &ev);
          const int i = G.src[e], j = G.col[e];
          const double qb = qbar[e], c = G.c[e], dc = G.dc[e];
          for (int k = 0; k < H; ++k) {
            const double ami = sv[u].ff_am[(int64_t)i * H + k];
            const double vj = sv[u].v[(int64_t)j * H + k], vdj = vdot[(int64_t)j * H + k];
            mdot[(int64_t)i * H + k] += qb * ev.wp[k] * vj + ev.w[k] * vdj;
            X[(int64_t)j * H + k] += qb * ev.wp[k] * ami;
            const double rho = ami * vj, kap = ami * vdj;
            mu[k] = qb * dc * rho + c * kap;
            nu[k] = qb * c * rho;
            dbeta[k] += mu[k];
          }
          /* B grads: s^T mu + sdot^T nu */
          for (int a = 0; a < H; ++a)
            for (int k = 0; k < H; ++k) dB[(int64_t)a * H + k] += ev.s[a] * mu[k] + ev.sp[a] * nu[k];
          vecmatT(H, H, mu, Bm, tmpH);  /* sbar */
          vecmatT(H, H, nu, Bm, tmpH2); /* sdotbar */
          for (int k = 0; k < H; ++k) {
            const double z = ev.z[k];
            zb[k] = tmpH[k] * dsilu(z) + tmpH2[k] * d2silu(z) * ev.zp[k];
            zpb[k] = tmpH2[k] * dsilu(z);
            dalpha[k] += zb[k];
          }
          for (int r = 0; r < R; ++r) {
            const double p = G.phi[(int64_t)e * R + r], dp = G.dphi[(int64_t)e * R + r];
            for (int k = 0; k < H; ++k) dA[(int64_t)r * H + k] += p * zb[k] + dp * zpb[k];
          }
        }
        /* W: h^T X + abar_h^T Y */
        wgrad(N, H, H, sv[u].h_in, X, dW);
        wgrad(N, H, H, abh, sv[u].ff_Y, dW);
        sv[u].inj_h = ALLOC(double, NH);
        mmT(N, H, H, X, W, sv[u].inj_h, 0);
        /* outputs: abar_h passes through, abar_m = mdot */
        free(abm);
        abm = mdot;
        free(vdot);
        free(X);
        free(mu);
        free(nu);
        free(zb);
        free(zpb);
      } else { /* upd */
        const double *Um = th, *V = Um + H * H + H;
        double *dU = t2, *dups = dU + H * H, *dV = dups + H;
        double* pdot = ALLOC(double, NH);
        mm(N, H, H, abm, Um, pdot, 0);
        sv[u].inj_m = ALLOC(double, NH);
        double* pb = ALLOC(double, NH);
        double* pdb = ALLOC(double, NH);
        double* sp_pdot = ALLOC(double, NH);
        for (int i = 0; i < N; ++i) {
          vecmatT(H, H, sv[u].ff_a + (int64_t)i * H, V, tmpH); /* r = a' V^T */
          for (int k = 0; k < H; ++k) {
            const double p = sv[u].p[(int64_t)i * H + k], pd = pdot[(int64_t)i * H + k];
            pb[(int64_t)i * H + k] = tmpH[k] * pd * d2silu(p);
            pdb[(int64_t)i * H + k] = tmpH[k] * dsilu(p);
            sp_pdot[(int64_t)i * H + k] = dsilu(p) * pd;
            dups[k] += pb[(int64_t)i * H + k];
          }
        }
        mmT(N, H, H, pb, Um, sv[u].inj_m, 0);
        wgrad(N, H, H, sp_pdot, sv[u].ff_a, dV);
        wgrad(N, H, H, sv[u].m_in, pb, dU);
        wgrad(N, H, H, abm, pdb, dU);
        /* abar' = abar_h + (SiLU'(p) pdot) V */
        mm(N, H, H, sp_pdot, V, abh, 1);
        free(abm);
        abm = NULL;
        free(pdot);
        free(pb);
        free(pdb);
        free(sp_pdot);
      }
      if (u < U - 1) {
        put_trace(trace, u, 4, abh, NH);
        put_trace(trace, u, 5, abm, NH);
      }
    }
    free(abh);
    free(abm);

    /* ================================ BE ================================ */
    double* bh = ALLOC(double, NH);
    double* bm = NULL;
    for (int u = U - 1; u >= 0; --u) {
      const double* th = params + mo_unit_param_offset(m, u);
      double* t1 = g1 + mo_unit_param_offset(m, u);
      if (u == U - 1) { /* readout: seed eps */
        const double *O = th, *om = th + H * H + H;
        double *dO = t1, *dob = t1 + H * H, *dom = t1 + H * H + H, *dbias = t1 + H * H + 2 * H;
        double* tb = ALLOC(double, NH);
        for (int i = 0; i < N; ++i) {
          const double ep = eps[b->struct_id[i]];
          dbias[b->species[i]] += ep;
          for (int k = 0; k < H; ++k) {
            const double t = sv[u].t[(int64_t)i * H + k];
            tb[(int64_t)i * H + k] = ep * dsilu(t) * om[k];
            dob[k] += tb[(int64_t)i * H + k];
            dom[k] += ep * silu(t);
          }
        }
        wgrad(N, H, H, sv[u].h_in, tb, dO);
        mmT(N, H, H, tb, O, bh, 0);
        for (int64_t x = 0; x < NH; ++x) bh[x] += sv[u].inj_h[x];
        free(tb);
      } else if (u == 0) { /* embed */
        for (int i = 0; i < N; ++i)
          for (int k = 0; k < H; ++k) t1[(int64_t)b->species[i] * H + k] += bh[(int64_t)i * H + k];
      } else if (u % 2 == 1) { /* msg */
        const double *A = th, *alpha = A + R * H, *Bm = alpha + H, *beta = Bm + H * H, *W = beta + H;
        double *dA = t1, *dalpha = dA + R * H, *dB = dalpha + H, *dbeta = dB + H * H, *dW = dbeta + H;
        double* Yb = ALLOC(double, NH);
        for (int e = 0; e < Ecount; ++e) {
          edge_eval(&G, e, A, alpha, Bm, beta, &ev);
          const int i = G.src[e], j = G.col[e];
          const double c = G.c[e];
          for (int k = 0; k < H; ++k) {
            const double bmi = bm[(int64_t)i * H + k];
            Yb[(int64_t)j * H + k] += ev.w[k] * bmi;
            tmpH[k] = c * bmi * sv[u].v[(int64_t)j * H + k]; /* gbar */
            dbeta[k] += tmpH[k];
          }
          for (int a = 0; a < H; ++a)
            for (int k = 0; k < H; ++k) dB[(int64_t)a * H + k] += ev.s[a] * tmpH[k];
          vecmatT(H, H, tmpH, Bm, tmpH2); /* sbar */
          for (int k = 0; k < H; ++k) {
            tmpH2[k] *= dsilu(ev.z[k]); /* zbar */
            dalpha[k] += tmpH2[k];
          }
          for (int r = 0; r < R; ++r) {
            const double p = G.phi[(int64_t)e * R + r];
            for (int k = 0; k < H; ++k) dA[(int64_t)r * H + k] += p * tmpH2[k];
          }
        }
        wgrad(N, H, H, sv[u].h_in, Yb, dW);
        mmT(N, H, H, Yb, W, bh, 1);
        for (int64_t x = 0; x < NH; ++x) bh[x] += sv[u].inj_h[x];
        free(Yb);
        free(bm);
        bm = NULL;
      } else { /* upd */
        const double *Um = th, *V = Um + H * H + H;
        double *dU = t1, *dups = dU + H * H, *dV = dups + H;
        double* pb = ALLOC(double, NH);
        double* sp = ALLOC(double, NH);
        for (int i = 0; i < N; ++i) {
          vecmatT(H, H, bh + (int64_t)i * H, V, tmpH);
          for (int k = 0; k < H; ++k) {
            const double p = sv[u].p[(int64_t)i * H + k];
            pb[(int64_t)i * H + k] = tmpH[k] * dsilu(p);
            sp[(int64_t)i * H + k] = silu(p);
            dups[k] += pb[(int64_t)i * H + k];
          }
        }
        wgrad(N, H, H, sp, bh, dV);
        wgrad(N, H, H, sv[u].m_in, pb, dU);
        bm = ALLOC(double, NH);
        mmT(N, H, H, pb, Um, bm, 0);
        for (int64_t x = 0; x < NH; ++x) bm[x] += sv[u].inj_m[x];
        free(pb);
        free(sp);
      }
      if (u > 0) {
        put_trace(trace, u, 6, bh, NH);
        put_trace(trace, u, 7, bm, NH);
      }
    }
    free(bh);
    free(bm);
    free(eps);
    free(Fbar);
    free(qbar);
  }

  if (grad1) memcpy(grad1, g1, sizeof(double) * (size_t)NP);
  if (grad2) memcpy(grad2, g2, sizeof(double) * (size_t)NP);
  if (grad)
    for (int64_t x = 0; x < NP; ++x) grad[x] = g1[x] + g2[x];

cleanup:
  for (int u = 0; u < U; ++u) {
    free(sv[u].h_in);
    free(sv[u].v);
    free(sv[u].m_in);
    free(sv[u].p);
    free(sv[u].t);
    free(sv[u].ff_am);
    free(sv[u].ff_Y);
    free(sv[u].ff_a);
    free(sv[u].inj_h);
    free(sv[u].inj_m);
  }
  free(sv);
  free(g1);
  free(g2);
  free(Es);
  free(F);
  free(ev.z);
  free(tmpH);
  free(tmpH2);
  free(tmpR);
  geo_free(&G);
  (void)S;
  (void)L;
  return 0;
}

int mo_step(const mo_model* m, const mo_batch* b, int64_t n_edges, const int* row_ptr, const int* col,
            const int* shift, const int* rev, const double* params, double* E, double* F, double* loss,
            double* grad, double* grad1, double* grad2, double* trace) {
  return run_step(m, b, n_edges, row_ptr, col, shift, rev, params, E, F, loss, grad, grad1, grad2, trace, 0);
}

int mo_energy(const mo_model* m, const mo_batch* b, int64_t n_edges, const int* row_ptr, const int* col,
              const int* shift, const double* params, double* E) {
  return run_step(m, b, n_edges, row_ptr, col, shift, NULL, params, E, NULL, NULL, NULL, NULL, NULL, NULL, 1);
}

void mo_adam(int64_t n, double* p, double* m1, double* m2, const double* g, double lr, double beta1,
             double beta2, double eps, int step) {
  const double c1 = 1.0 - pow(beta1, step), c2 = 1.0 - pow(beta2, step);
  for (int64_t i = 0; i < n; ++i) {
    m1[i] = beta1 * m1[i] + (1.0 - beta1) * g[i];
    m2[i] = beta2 * m2[i] + (1.0 - beta2) * g[i] * g[i];
    p[i] -= lr * (m1[i] / c1) / (sqrt(m2[i] / c2) + eps);
  }
}

/* ------------------------------------------------------- synthetic inputs
 * Restatement of the seeded synthetic data: SplitMix64 as
 * reference rng.hpp:11-38 (next(), next() % n, 53-bit doubles), Box-Muller
 * cosine branch on (1 - u1, u2), per-tensor streams seed ^ (tag * gamma).
 * Lets the CPU reference arm build its inputs without the product library;
 * tests/test_oracle.py pins it bit-for-bit to janus_synth_params / _cell. */
typedef struct { uint64_t s; } mo_rng;
static uint64_t rng_next(mo_rng* g) {
  g->s += 0x9e3779b97f4a7c15ULL;
  uint64_t x = g->s;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static double rng_double(mo_rng* g) { return (double)(rng_next(g) >> 11) * 0x1.0p-53; }
static double rng_normal(mo_rng* g) {
  const double u1 = 1.0 - rng_double(g);
  const double u2 = rng_double(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

void mo_synth_params(const mo_model* m, uint64_t seed, float* out) {
  const int H = m->H, R = m->R, S = m->n_species, U = 2 * m->L + 2;
  int64_t off = 0;
  const double sH = 1.0 / sqrt((double)H), sR = 1.0 / sqrt((double)R);
#define FILL(unit, tensor, n, sd)                                                              \
  do {                                                                                         \
    mo_rng g = {seed ^ (((uint64_t)(unit) * 16u + (uint64_t)(tensor) + 1u) * 0x9e3779b97f4a7c15ULL)}; \
    for (int64_t x = 0; x < (int64_t)(n); ++x) out[off + x] = (float)((sd) * rng_normal(&g));  \
    off += (int64_t)(n);                                                                       \
  } while (0)
  for (int u = 0; u < U; ++u) {
    if (u == 0) {
      FILL(u, 0, (int64_t)S * H, 1.0);
    } else if (u == U - 1) {
      FILL(u, 0, (int64_t)H * H, sH);
      FILL(u, 1, H, 0.1);
      FILL(u, 2, H, sH);
      FILL(u, 3, S, 1.0);
    } else if (u % 2 == 1) {
      FILL(u, 0, (int64_t)R * H, sR);
      FILL(u, 1, H, 0.1);
      FILL(u, 2, (int64_t)H * H, sH);
      FILL(u, 3, H, 0.1);
      FILL(u, 4, (int64_t)H * H, sH);
    } else {
      FILL(u, 0, (int64_t)H * H, sH);
      FILL(u, 1, H, 0.1);
      FILL(u, 2, (int64_t)H * H, sH);
    }
  }
#undef FILL
}

double mo_synth_cell(int n, double rho, int n_species, uint64_t seed, double* pos, int* species, float* E_target,
                     float* F_target) {
  if (n < 1 || !(rho > 0) || n_species < 1) return -1.0;
  const double L = cbrt((double)n / rho);
  double* sites = ALLOC(double, 3 * (int64_t)n);
  int ns = 0;
  int k = (int)lround(cbrt(n / 4.0));
  if (k >= 1 && 4 * k * k * k == n) {
    const double a = L / k;
    const double basis[4][3] = {{0, 0, 0}, {0.5, 0.5, 0}, {0.5, 0, 0.5}, {0, 0.5, 0.5}};
    for (int x = 0; x < k; ++x)
      for (int y = 0; y < k; ++y)
        for (int z = 0; z < k; ++z)
          for (int q = 0; q < 4; ++q, ++ns) {
            sites[3 * ns] = (x + basis[q][0]) * a;
            sites[3 * ns + 1] = (y + basis[q][1]) * a;
            sites[3 * ns + 2] = (z + basis[q][2]) * a;
          }
  } else {
    k = (int)ceil(cbrt((double)n) - 1e-9);
    const double a = L / k;
    for (int x = 0; x < k && ns < n; ++x)
      for (int y = 0; y < k && ns < n; ++y)
        for (int z = 0; z < k && ns < n; ++z, ++ns) {
          sites[3 * ns] = x * a;
          sites[3 * ns + 1] = y * a;
          sites[3 * ns + 2] = z * a;
        }
  }
  mo_rng g = {seed};
  const double sigma = 0.1 * L / cbrt((double)n);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      double x = sites[3 * i + c] + sigma * rng_normal(&g);
      x = fmod(x, L);
      if (x < 0) x += L;
      if (x >= L) x -= L;
      pos[3 * i + c] = x;
    }
  for (int i = 0; i < n; ++i) species[i] = n_species <= 1 ? 0 : (int)(rng_next(&g) % (uint64_t)n_species);
  *E_target = (float)(sqrt((double)n) * rng_normal(&g));
  for (int x = 0; x < 3 * n; ++x) F_target[x] = (float)(0.1 * rng_normal(&g));
  free(sites);
  return L;
}
