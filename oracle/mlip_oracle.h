/* oracle/mlip_oracle.h — TEST INFRASTRUCTURE: fp64 CPU oracle of the
 * four-phase (FE/FF/BF/BE) training step of the canonical conservative MLIP.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library (as the checker); the product path never does.
 *
 * Parity status: the reference (/root/reference) contains NO numeric
 * implementation of this path (SPEC.md:15 rules out real double-backward
 * compute).  The math follows PAPER.md:171-178 (four phases), 313-332
 * (Eq. 1-2 merged/second-order split) and the builder-pinned model of
 * SURVEY.md Appendix A.  It is pinned instead by (i) golden vectors produced
 * by PyTorch fp64 autograd double-backward (the arithmetic engine the paper
 * used) — tests/golden/make_mlip_golden.py — and (ii) central
 * finite differences, (iii) staged == unstaged, (iv) the Eq. (2) ledger
 * identity grad = grad_BE(merged first order) + grad_BF(second order).
 *
 * Units (the pipeline partition granule, SURVEY.md §7 hard part 5):
 *   0 = embed, 1+2l = msg_l (edge filter + aggregation), 2+2l = upd_l
 *   (node update MLP), 2L+1 = readout.
 * Parameter layout (flat, in unit order):
 *   embed   : Emb[S][H]
 *   msg_l   : A[R][H] alpha[H] B[H][H] beta[H] W[H][H]
 *   upd_l   : U[H][H] upsilon[H] V[H][H]
 *   readout : O[H][H] o[H] omega[H] bias[S]
 */
#ifndef JANUS_MLIP_ORACLE_H
#define JANUS_MLIP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int L, H, R, n_species;
  double r_c, w_E, w_F;
} mo_model;

/* Structures are concatenated: atoms of structure s are contiguous. */
typedef struct {
  int n_atoms, n_struct;
  const double* pos;       /* [N*3] */
  const int* species;      /* [N]   */
  const int* struct_id;    /* [N]   */
  const double* cell;      /* [n_struct] cubic box length */
  const double* E_target;  /* [n_struct] */
  const double* F_target;  /* [N*3] */
} mo_batch;

int mo_num_units(const mo_model* m);
int64_t mo_unit_param_offset(const mo_model* m, int unit);
int64_t mo_unit_param_count(const mo_model* m, int unit);
int64_t mo_param_count(const mo_model* m);

/* Periodic neighbour list, CSR by receiver i, edges sorted by (i, j, sx, sy,
 * sz); d^2 < r_c^2 tested in fp64 as dx*dx+dy*dy+dz*dz (no FMA contraction).
 * rev[e] = index of the reverse edge (j, i, -s).  Returns the edge count or
 * -1 if more than max_edges. */
int64_t mo_build_nbrlist(const mo_model* m, const mo_batch* b, int64_t max_edges, int* row_ptr,
                         int* col, int* shift, int* rev);

/* Full four-phase step.  Outputs (any may be NULL):
 *   E[n_struct], F[N*3], loss[1],
 *   grad[n_params] = grad1 + grad2 (total dL/dtheta),
 *   grad1 = BE merged first-order term, grad2 = BF second-order term.
 * trace (may be NULL): [n_units][8][N*H] doubles —
 *   slot 0/1: FE output carrier (h, m) of the unit,
 *   slot 2/3: FF adjoint at the unit INPUT (a_h, a_m),
 *   slot 4/5: BF tangent at the unit OUTPUT (abar_h, abar_m),
 *   slot 6/7: BE adjoint at the unit INPUT (b_h, b_m).
 * Slots that do not apply are zero.  Returns 0 on success. */
int mo_step(const mo_model* m, const mo_batch* b, int64_t n_edges, const int* row_ptr, const int* col,
            const int* shift, const int* rev, const double* params, double* E, double* F, double* loss,
            double* grad, double* grad1, double* grad2, double* trace);

/* Energies only (for finite differences of forces). */
int mo_energy(const mo_model* m, const mo_batch* b, int64_t n_edges, const int* row_ptr, const int* col,
              const int* shift, const double* params, double* E);

/* Adam update (bias-corrected), in place; step is 1-based. */
void mo_adam(int64_t n, double* p, double* m1, double* m2, const double* g, double lr, double beta1,
             double beta2, double eps, int step);

/* Seeded synthetic inputs, bit-identical to the product's janus_synth_params /
 * janus_synth_cell (SplitMix64 of reference rng.hpp:11-38).  mo_synth_cell
 * returns the box length (-1 on bad arguments). */
void mo_synth_params(const mo_model* m, uint64_t seed, float* out);
double mo_synth_cell(int n, double rho, int n_species, uint64_t seed, double* pos, int* species, float* E_target,
                     float* F_target);

#ifdef __cplusplus
}
#endif
#endif
