// level_sets.cuh -- best level set of a TV solution on the device.
//
// The reference evaluates discrete_gap at every level set {x > v}, v over
// the distinct values of x plus the all-ones labeling, and keeps the first
// one with the smallest gap (certify.py:50-65 with solvers.level_sets,
// solvers.py:86-97) -- O(K n) numpy work for K distinct values.  The dual
// term of the gap does not depend on the labeling, so the best level set is
// the one of least energy, and all K+1 energies come out of one sort:
//
//   rank(i)   = 1-based rank of x_i among the distinct values (sorted order)
//   E(k)      = cut(k) - sum_{rank(i) > k} w_i,   k = 0 (all ones) .. K (empty)
//   cut(k)    = sum over edges (i, j) of a_ij [min rank <= k < max rank]
//
// cut() is a difference array over ranks (+a at the lower rank, -a at the
// upper) followed by a prefix sum; the unary part is a prefix sum of w in
// sorted order read at each rank's last position.  The edge scatter uses
// fp64 atomics, so E(k) is exact for integer-valued weights (the
// certification case) and otherwise carries rounding in the last
// bits; the chosen labeling is then re-evaluated by the deterministic
// pcb_check reductions, which give the reported energy and gap.
#pragma once
#include <cub/cub.cuh>

namespace pcb {
namespace levels {

__global__ void k_iota(int* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

// new-value flags in sorted order (-0.0 == 0.0, like np.unique)
__global__ void k_flags(const double* xs, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || xs[i] != xs[i - 1]) ? 1 : 0;
}

// node rank, sorted unaries, and each rank's last sorted position
__global__ void k_scatter_ranks(const int* rs, const int* idx, const double* w, int64_t n,
                                int* rank_of, double* ws, int64_t* last_of) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int node = idx[i];
    rank_of[node] = rs[i];
    ws[i] = w[node];
    if (i == n - 1 || rs[i + 1] != rs[i]) last_of[rs[i]] = i;
  }
}

// difference array of the cut over ranks, one thread per node and direction
__global__ void k_cut_diff(Dims D, DirGeom DG, DirPtrs dw, const int* rank_of, double* diff) {
  int64_t n = 1;
  for (int a = 0; a < D.nd; ++a) n *= D.d[a];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t co[3];
    int64_t rem = i;
    for (int a = D.nd - 1; a >= 0; --a) {
      co[a] = rem % D.d[a];
      rem /= D.d[a];
    }
    const int ri = rank_of[i];
    for (int k = 0; k < DG.ndir; ++k) {
      bool ok = true;
      int64_t e = 0, j = 0;
      for (int a = 0; a < D.nd; ++a) {
        const int o = DG.off[k][a];
        const int64_t len = D.d[a] - (o < 0 ? -o : o);
        const int64_t lo = o >= 0 ? 0 : -o;
        const int64_t q = co[a] - lo;
        if (q < 0 || q >= len) ok = false;
        e = e * (len > 0 ? len : 1) + q;
        j = j * D.d[a] + (co[a] + o);
      }
      if (!ok) continue;
      const double av = dw.p[k][e];
      if (av == 0.0) continue;
      const int rj = rank_of[j];
      if (ri == rj) continue;
      atomicAdd(&diff[ri < rj ? ri : rj], av);
      atomicAdd(&diff[ri < rj ? rj : ri], -av);
    }
  }
}

// E(k) for k = 0..K from the cut prefix and the unary prefix; cutp[k] =
// sum_{t <= k} diff[t] (diff[0] = 0), wp = inclusive prefix of ws
__global__ void k_energies(const double* cutp, const double* wp, const int64_t* last_of, int K,
                           int64_t n, double* E) {
  const double wt = wp[n - 1];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= K;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double below = k == 0 ? 0.0 : wp[last_of[k]];  // sum of w over rank <= k
    E[k] = cutp[k] - (wt - below);
  }
}

// first index of the minimum (the reference keeps the first strictly better)
struct ArgMin {
  double v;
  int64_t k;
};

__device__ __forceinline__ ArgMin better(ArgMin a, ArgMin b) {
  return (b.v < a.v || (b.v == a.v && b.k < a.k)) ? b : a;
}

__global__ void k_argmin(const double* E, int64_t cnt, ArgMin* parts) {
  ArgMin best{INFINITY, INT64_MAX};
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x)
    best = better(best, ArgMin{E[k], k});
  __shared__ ArgMin sh[256];  // launched with 256 threads
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] = better(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) parts[blockIdx.x] = sh[0];
}

__global__ void k_argmin_final(const ArgMin* parts, int np, const double* xs,
                               const int64_t* last_of, double* out) {
  ArgMin best{INFINITY, INT64_MAX};
  for (int b = 0; b < np; ++b) best = better(best, parts[b]);
  out[0] = best.k == 0 ? -INFINITY : xs[last_of[best.k]];  // level set {x > u_k}
  out[1] = best.v;
  out[2] = (double)best.k;
}

}  // namespace levels
}  // namespace pcb
