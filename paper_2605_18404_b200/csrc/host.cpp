// host.cpp — host-side data for the LM instruction: synthetic cells and
// parameters (seeded by the pinned SplitMix64, reference rng.hpp:11-38) and
// the periodic neighbour list.  Compiled with -ffp-contract=off: the d^2 test
// must round exactly like the oracle (oracle/mlip_oracle.c mo_build_nbrlist)
// so the CSR is bit-identical (integer work is bit-exact, BASELINE north star).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/janus/errors.hpp"
#include "../../include/janus/rng.hpp"
#include "../../include/janus_cuda.h"
#include "host.hpp"

namespace janus {

int64_t host_unit_param_count(const janus_model_desc& m, int u) {
  const int64_t H = m.H, R = m.R, S = m.n_species;
  if (u == 0) return S * H;
  if (u == 2 * m.L + 1) return H * H + 2 * H + S;
  if (u % 2 == 1) return R * H + H + H * H + H + H * H;
  return H * H + H + H * H;
}

int64_t host_unit_param_offset(const janus_model_desc& m, int u) {
  int64_t o = 0;
  for (int x = 0; x < u; ++x) o += host_unit_param_count(m, x);
  return o;
}

void synth_params(const janus_model_desc& m, uint64_t seed, float* out) {
  const int H = m.H, R = m.R, S = m.n_species, U = 2 * m.L + 2;
  int64_t off = 0;
  auto fill = [&](int unit, int tensor, int64_t n, double stddev) {
    SplitMix64 g = SplitMix64::derive(seed, static_cast<uint64_t>(unit) * 16u + static_cast<uint64_t>(tensor) + 1u);
    for (int64_t x = 0; x < n; ++x) out[off + x] = static_cast<float>(stddev * g.normal());
    off += n;
  };
  const double sH = 1.0 / std::sqrt(static_cast<double>(H)), sR = 1.0 / std::sqrt(static_cast<double>(R));
  for (int u = 0; u < U; ++u) {
    if (u == 0) {
      fill(u, 0, static_cast<int64_t>(S) * H, 1.0);
    } else if (u == U - 1) {
      fill(u, 0, static_cast<int64_t>(H) * H, sH);  // O
      fill(u, 1, H, 0.1);                           // o
      fill(u, 2, H, sH);                            // omega
      fill(u, 3, S, 1.0);                           // bias
    } else if (u % 2 == 1) {
      fill(u, 0, static_cast<int64_t>(R) * H, sR);  // A
      fill(u, 1, H, 0.1);                           // alpha
      fill(u, 2, static_cast<int64_t>(H) * H, sH);  // B
      fill(u, 3, H, 0.1);                           // beta
      fill(u, 4, static_cast<int64_t>(H) * H, sH);  // W
    } else {
      fill(u, 0, static_cast<int64_t>(H) * H, sH);  // U
      fill(u, 1, H, 0.1);                           // upsilon
      fill(u, 2, static_cast<int64_t>(H) * H, sH);  // V
    }
  }
}

double synth_cell(int n, double rho, int n_species, uint64_t seed, double* pos, int32_t* species, float* E_target,
                  float* F_target) {
  if (n < 1 || !(rho > 0) || n_species < 1) throw domain_error("synth_cell: bad arguments");
  const double L = std::cbrt(static_cast<double>(n) / rho);
  // lattice: fcc when n = 4 k^3, else simple cubic on ceil(cbrt n)^3 sites
  std::vector<std::array<double, 3>> sites;
  int k = static_cast<int>(std::lround(std::cbrt(n / 4.0)));
  if (k >= 1 && 4 * k * k * k == n) {
    const double a = L / k;
    const double basis[4][3] = {{0, 0, 0}, {0.5, 0.5, 0}, {0.5, 0, 0.5}, {0, 0.5, 0.5}};
    for (int x = 0; x < k; ++x)
      for (int y = 0; y < k; ++y)
        for (int z = 0; z < k; ++z)
          for (const auto& b : basis) sites.push_back({(x + b[0]) * a, (y + b[1]) * a, (z + b[2]) * a});
  } else {
    k = static_cast<int>(std::ceil(std::cbrt(static_cast<double>(n)) - 1e-9));
    const double a = L / k;
    for (int x = 0; x < k && static_cast<int>(sites.size()) < n; ++x)
      for (int y = 0; y < k && static_cast<int>(sites.size()) < n; ++y)
        for (int z = 0; z < k && static_cast<int>(sites.size()) < n; ++z) sites.push_back({x * a, y * a, z * a});
  }
  SplitMix64 g(seed);
  const double sigma = 0.1 * L / std::cbrt(static_cast<double>(n));
  for (int i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) {
      double x = sites[static_cast<size_t>(i)][static_cast<size_t>(c)] + sigma * g.normal();
      x = std::fmod(x, L);
      if (x < 0) x += L;
      if (x >= L) x -= L;
      pos[3 * i + c] = x;
    }
  }
  for (int i = 0; i < n; ++i) species[i] = static_cast<int32_t>(g.next_below(static_cast<uint64_t>(n_species)));
  *E_target = static_cast<float>(std::sqrt(static_cast<double>(n)) * g.normal());
  for (int x = 0; x < 3 * n; ++x) F_target[x] = static_cast<float>(0.1 * g.normal());
  return L;
}

int nbrlist_build(int n, const double* pos, const int32_t* struct_id, const double* cell, double rc, int max_edges,
                  int32_t* row_ptr, int32_t* col, int32_t* shift, int32_t* rev) {
  const double rc2 = rc * rc;
  // structure ranges (atoms of a structure are contiguous)
  std::vector<int> first(static_cast<size_t>(n)), count(static_cast<size_t>(n));
  for (int i = 0; i < n;) {
    int j = i;
    while (j < n && struct_id[j] == struct_id[i]) ++j;
    for (int x = i; x < j; ++x) {
      first[static_cast<size_t>(x)] = i;
      count[static_cast<size_t>(x)] = j - i;
    }
    i = j;
  }
  int E = 0;
  row_ptr[0] = 0;
  for (int i = 0; i < n; ++i) {
    const double L = cell[struct_id[i]];
    const int nimg = static_cast<int>(std::ceil(rc / L));
    const double* xi = pos + 3 * i;
    for (int j = first[static_cast<size_t>(i)]; j < first[static_cast<size_t>(i)] + count[static_cast<size_t>(i)]; ++j) {
      const double* xj = pos + 3 * j;
      for (int sx = -nimg; sx <= nimg; ++sx)
        for (int sy = -nimg; sy <= nimg; ++sy)
          for (int sz = -nimg; sz <= nimg; ++sz) {
            if (i == j && sx == 0 && sy == 0 && sz == 0) continue;
            const double rx = (xj[0] + sx * L) - xi[0];
            const double ry = (xj[1] + sy * L) - xi[1];
            const double rz = (xj[2] + sz * L) - xi[2];
            const double d2 = (rx * rx + ry * ry) + rz * rz;
            if (!(d2 < rc2)) continue;
            if (E >= max_edges) throw domain_error("neighbour list exceeds max_edges");
            col[E] = j;
            shift[3 * E] = sx;
            shift[3 * E + 1] = sy;
            shift[3 * E + 2] = sz;
            ++E;
          }
    }
    row_ptr[i + 1] = E;
  }
  // reverse edge: (j, i, -s) is in row j, rows sorted by (j', s') => binary search
  for (int i = 0; i < n; ++i) {
    for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const int j = col[e];
      const std::array<int, 4> key{i, -shift[3 * e], -shift[3 * e + 1], -shift[3 * e + 2]};
      int lo = row_ptr[j], hi = row_ptr[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        const std::array<int, 4> k2{col[mid], shift[3 * mid], shift[3 * mid + 1], shift[3 * mid + 2]};
        if (k2 < key) lo = mid + 1; else hi = mid;
      }
      if (lo >= row_ptr[j + 1] || col[lo] != i || shift[3 * lo] != key[1] || shift[3 * lo + 1] != key[2] ||
          shift[3 * lo + 2] != key[3])
        throw state_error("neighbour list is not symmetric");
      rev[e] = lo;
    }
  }
  return E;
}

}  // namespace janus
