// paracut_b200.cu -- sm_100a kernels and the C ABI (include/paracut_b200.h)
// for the AAR chain-prox hot path of arXiv 1503.01563 (reference: paracut).
//
// Layout in HBM:
//   node arrays      n entries, C order of dims (w, c, x, G, labels, z_j, y_j)
//   family weights   Wf_j[i * C_j + c]: edge i of chain c, chain-interleaved
//                    so that threads owning adjacent chains read adjacent words
//   direction weights natural graph.direction_shape arrays (certificates)
//
// Kernels:
//   k_family_exact   fp64 prox of one chain family, z_j -> y_j = z_j - prox
//                    (projections.py:89-104 / _kernels.py:145-180)
//   k_update_exact   z += Pi_L(2y - z) - y in the reference's operation order
//                    (solvers.py:295-298, projections.py:107-122)
//   fast::k_sweep    staged fp32-state sweep (fast_sweep.cuh): prox of
//                    z_j = p_j + c, p_j in place, accumulator G, the last
//                    family applies the drift/primal update
//   k_apply_fast     check-iteration update from an fp64 shadow
//   k_check_nodes / k_check_edges   threshold, unary, dual, cut partials
//   k_reduce_*       deterministic fixed-order final reductions
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cerrno>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/paracut_b200.h"
#include "taut_string.cuh"

#define PCB_VERSION 1

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (void)cudaGetLastError();                                                            \
      return fail(e_ == cudaErrorMemoryAllocation ? PCB_E_NOMEM : PCB_E_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                      \
    }                                                                                      \
  } while (0)

#define LAUNCH_CHECK(h)                                                                    \
  do {                                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return fail(PCB_E_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                               \
    if (h) (h)->launches++;                                                                \
  } while (0)

constexpr int HC = 8;          // hull entries kept in shared memory per thread
constexpr int FAM_BLOCK = 128;  // threads (chains) per block in family kernels
constexpr int RED_BLOCK = 256;
constexpr int MAXR = 4;
constexpr int MAXT = 8;         // thresholds per check

// ----------------------------------------------------------------- geometry

enum FamKind { K_ROW2 = 0, K_COL2, K_ZZ0, K_ZZ1, K_X3, K_Y3, K_Z3 };

// node(c, i) = (c / cdiv) * chi + (c % cdiv) * clo + i * ns + zz * ((i + phase) & 1)
struct Fam {
  int kind;
  int m;          // nodes per chain
  int64_t C;      // chains
  int64_t cdiv, chi, clo, ns, zz;
  int phase;
};

__device__ __forceinline__ int64_t fam_base(const Fam& F, int64_t c) {
  return (c / F.cdiv) * F.chi + (c % F.cdiv) * F.clo;
}
__device__ __forceinline__ int64_t fam_node(const Fam& F, int64_t b, int i) {
  return b + (int64_t)i * F.ns + F.zz * (int64_t)((i + F.phase) & 1);
}

struct Dims {
  int nd;
  int64_t d[3];
  int conn;
};

// Which direction array and element hold edge i of chain c (decompose.py:142-183).
__device__ __forceinline__ void fam_edge(const Fam& F, const Dims& D, int64_t c, int i, int* dir,
                                         int64_t* idx) {
  switch (F.kind) {
    case K_ROW2:  // dir 0, shape (H, W-1)
      *dir = 0;
      *idx = c * (D.d[1] - 1) + i;
      return;
    case K_COL2:  // dir 1, shape (H-1, W)
      *dir = 1;
      *idx = (int64_t)i * D.d[1] + c;
      return;
    case K_ZZ0:  // even edge: d1 (dir 2), odd: d2 (dir 3); shape (H-1, W-1)
      *dir = (i & 1) ? 3 : 2;
      *idx = c * (D.d[1] - 1) + i;
      return;
    case K_ZZ1:
      *dir = (i & 1) ? 2 : 3;
      *idx = c * (D.d[1] - 1) + i;
      return;
    case K_X3:  // dir 0, shape (D0, D1, D2-1), chain c = z*D1 + y
      *dir = 0;
      *idx = c * (D.d[2] - 1) + i;
      return;
    case K_Y3: {  // dir 1, shape (D0, D1-1, D2), chain c = z*D2 + x
      *dir = 1;
      int64_t z = c / D.d[2], x = c % D.d[2];
      *idx = z * (D.d[1] - 1) * D.d[2] + (int64_t)i * D.d[2] + x;
      return;
    }
    default:  // K_Z3: dir 2, shape (D0-1, D1, D2), chain c = y*D2 + x
      *dir = 2;
      *idx = (int64_t)i * D.d[1] * D.d[2] + c;
      return;
  }
}

// Inverse of fam_node: chain and position of grid node nd in family F
// (false for the border nodes a zig-zag family leaves as singletons).
__device__ __forceinline__ bool fam_index(const Fam& F, const Dims& D, int64_t nd, int64_t* c,
                                          int* i) {
  switch (F.kind) {
    case K_ROW2:
      *c = nd / D.d[1];
      *i = (int)(nd % D.d[1]);
      return true;
    case K_COL2:
      *c = nd % D.d[1];
      *i = (int)(nd / D.d[1]);
      return true;
    case K_ZZ0:
    case K_ZZ1: {
      const int64_t y = nd / D.d[1], x = nd % D.d[1];
      const int64_t r = y - ((x + F.phase) & 1);
      if (r < 0 || r >= F.C) return false;
      *c = r;
      *i = (int)x;
      return true;
    }
    case K_X3:
      *c = nd / D.d[2];
      *i = (int)(nd % D.d[2]);
      return true;
    case K_Y3: {
      const int64_t plane = D.d[1] * D.d[2];
      const int64_t z = nd / plane, rem = nd % plane;
      *c = z * D.d[2] + rem % D.d[2];
      *i = (int)(rem / D.d[2]);
      return true;
    }
    default: {
      const int64_t plane = D.d[1] * D.d[2];
      *c = nd % plane;
      *i = (int)(nd / plane);
      return true;
    }
  }
}

__host__ __device__ inline bool fam_rowlike(int kind) {
  return kind == K_ROW2 || kind == K_ZZ0 || kind == K_ZZ1 || kind == K_X3;
}

struct FamSet {
  Fam f[MAXR];
  int r;
};

struct DirPtrs {
  const double* p[4];
};

template <class T>
__global__ void k_build_family_weights(Fam F, Dims D, DirPtrs dw, T* out) {
  const int64_t total = F.C * (int64_t)(F.m - 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / F.C);
    const int64_t c = t % F.C;
    int dir;
    int64_t idx;
    fam_edge(F, D, c, i, &dir, &idx);
    // +0.0 canonicalises -0.0 so a split gate sees the reference's literal 0.0
    out[t] = (T)(dw.p[dir][idx] + 0.0);
  }
}

// ----------------------------------------------------------------- reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum in a fixed order (deterministic); result valid in thread 0.
__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int k = 0; k < nw; ++k) r += sh[k];
  }
  return r;
}

// out[slot] = sqrt?(sum of parts[0..count)) in index order; one block.
__global__ void k_reduce_norm(const double* parts, int64_t count, double* out, int do_sqrt) {
  double acc = 0.0;
  // each thread sums a contiguous slice; slices combined in thread order
  const int64_t per = (count + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(count, lo + per);
  for (int64_t k = lo; k < hi; ++k) acc += parts[k];
  // slices combined by a fixed shuffle tree (deterministic; a serial sum of
  // 1024 values by one thread cost ~4 us per iteration)
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) *out = do_sqrt ? sqrt(t) : t;
  }
}

// vals[j] = sum over blocks b of parts[b * nv + j]; one block, fixed order.
__global__ void k_reduce_cols(const double* parts, int nblocks, int nv, double* vals) {
  // one warp per column: lane l sums blocks l, l + 32, ... in order, then a
  // fixed shuffle tree (deterministic; a single thread per column was load
  // latency bound, ~55 us per call at 1184 blocks)
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= nv) return;
  double t = 0.0;
#pragma unroll 8
  for (int b = lane; b < nblocks; b += 32) t += parts[(int64_t)b * nv + j];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if (lane == 0) vals[j] = t;
}

// ----------------------------------------------------------------- accessors

struct AccExact {  // fp64 grid family: y = z - prox(z)
  const double* z;
  double* y;
  const double* wf;
  Fam F;
  int64_t c, b;
  __device__ __forceinline__ double s(int i) const { return z[fam_node(F, b, i)]; }
  __device__ __forceinline__ double a(int i) const { return wf[(int64_t)i * F.C + c]; }
  __device__ __forceinline__ void emit(int i, double fill) {
    const int64_t nd = fam_node(F, b, i);
    y[nd] = z[nd] - fill;
  }
};

struct AccCSR {  // _kernels.prox_chains gather/scatter
  const double* v;
  double* out;
  const int64_t* ids;
  const double* ew;
  int proj;
  __device__ __forceinline__ double s(int i) const { return v[ids[i]]; }
  __device__ __forceinline__ double a(int i) const { return ew[i]; }
  __device__ __forceinline__ void emit(int i, double fill) {
    const int64_t nd = ids[i];
    out[nd] = proj ? v[nd] - fill : fill;
  }
};

struct AccTv1d {  // tv1d_prox on contiguous signals
  const double* s_;
  const double* a_;
  double* x;
  __device__ __forceinline__ double s(int i) const { return s_[i]; }
  __device__ __forceinline__ double a(int i) const { return a_[i]; }
  __device__ __forceinline__ void emit(int i, double fill) { x[i] = fill; }
};

// ----------------------------------------------------------------- family kernels

struct Spill {
  int* cx;
  double* cy;
  int* fx;
  double* fy;
};

template <class Acc>
__device__ __forceinline__ void run_chain(Acc& A, int m, const Spill& sp, int64_t gtid,
                                          int64_t gstride) {
  __shared__ int s_cx[HC * FAM_BLOCK];
  __shared__ int s_fx[HC * FAM_BLOCK];
  __shared__ double s_cy[HC * FAM_BLOCK];
  __shared__ double s_fy[HC * FAM_BLOCK];
  pcb::Hull<HC> cH{s_cx + threadIdx.x, s_cy + threadIdx.x, (int)blockDim.x,
                   sp.cx + gtid, sp.cy + gtid, gstride};
  pcb::Hull<HC> fH{s_fx + threadIdx.x, s_fy + threadIdx.x, (int)blockDim.x,
                   sp.fx + gtid, sp.fy + gtid, gstride};
  pcb::taut_chain(A, cH, fH, m);
}

__global__ void __launch_bounds__(FAM_BLOCK) k_family_exact(Fam F, const double* z, double* y,
                                                            const double* wf, Spill sp) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  AccExact A{z, y, wf, F, c, fam_base(F, c)};
  run_chain(A, F.m, sp, c, (int64_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(FAM_BLOCK) k_prox_csr(const int64_t* node_idx,
                                                        const int64_t* chain_ptr,
                                                        const double* edge_w, int64_t c_lo,
                                                        int64_t c_hi, const double* v, double* out,
                                                        int proj, Spill sp, const int64_t* soff) {
  const int64_t c = c_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= c_hi) return;
  const int64_t b = chain_ptr[c];
  const int m = (int)(chain_ptr[c + 1] - b);
  if (m <= 0) return;
  AccCSR A{v, out, node_idx + b, edge_w + (b - c), proj};
  // per-chain contiguous spill region (stride 1)
  __shared__ int s_cx[HC * FAM_BLOCK];
  __shared__ int s_fx[HC * FAM_BLOCK];
  __shared__ double s_cy[HC * FAM_BLOCK];
  __shared__ double s_fy[HC * FAM_BLOCK];
  const int64_t o = soff[c - c_lo];
  pcb::Hull<HC> cH{s_cx + threadIdx.x, s_cy + threadIdx.x, (int)blockDim.x, sp.cx + o, sp.cy + o, 1};
  pcb::Hull<HC> fH{s_fx + threadIdx.x, s_fy + threadIdx.x, (int)blockDim.x, sp.fx + o, sp.fy + o, 1};
  pcb::taut_chain(A, cH, fH, m);
}

__global__ void __launch_bounds__(FAM_BLOCK) k_tv1d(const double* s, const double* a,
                                                    const int64_t* ptr, int64_t nch, double* x,
                                                    Spill sp, const int64_t* soff) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nch) return;
  const int64_t b = ptr[c];
  const int m = (int)(ptr[c + 1] - b);
  if (m <= 0) return;
  AccTv1d A{s + b, a + (b - c), x + b};
  __shared__ int s_cx[HC * FAM_BLOCK];
  __shared__ int s_fx[HC * FAM_BLOCK];
  __shared__ double s_cy[HC * FAM_BLOCK];
  __shared__ double s_fy[HC * FAM_BLOCK];
  const int64_t o = soff[c];
  pcb::Hull<HC> cH{s_cx + threadIdx.x, s_cy + threadIdx.x, (int)blockDim.x, sp.cx + o, sp.cy + o, 1};
  pcb::Hull<HC> fH{s_fx + threadIdx.x, s_fy + threadIdx.x, (int)blockDim.x, sp.fx + o, sp.fy + o, 1};
  pcb::taut_chain(A, cH, fH, m);
}

}  // namespace

#include "fast_sweep.cuh"
#include "lean_verify.cuh"
#include "generator.cuh"
#include "exact_sweep.cuh"

namespace {

// ----------------------------------------------------------------- node-wise kernels

// z <- z + ((2y - z) + corr) - y with corr = (w - sum_j (2y_j - z_j)) / r
// (projections.py:118-122 then solvers.py:295-297, same rounding order).
template <int R>
__global__ void k_update_exact(double* z, const double* y, const double* w, int64_t n,
                               double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[R];
    double total = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      v[j] = 2.0 * y[j * n + i] - z[j * n + i];
      total = (j == 0) ? v[0] : total + v[j];
    }
    const double corr = (w[i] - total) / (double)R;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double dz = (v[j] + corr) - y[j * n + i];
      z[j * n + i] = z[j * n + i] + dz;
      acc += dz * dz;
    }
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// z^0 = Pi_L(0): lam = (0 + (w - 0)/r) * 1 per class.
__global__ void k_init_exact(double* z, const double* w, int64_t n, int r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double corr = (w[i] - 0.0) / (double)r;
    for (int j = 0; j < r; ++j) z[j * n + i] = 0.0 + corr;
  }
}

// fp32 state from an fp64 z (natural [j][node]): c = mean_j z_j, p_j = z_j - c
// stored chain-interleaved, x = w - sum_j p_j.
template <class ST>
__global__ void k_set_fast(const double* z, ST* p, double* cdrift, ST* X, const double* w,
                           int64_t n, FamSet FS, Dims D) {
  const int r = FS.r;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // z_j = p_j + c.  A zig-zag border node keeps no state in that family
    // (p = 0), so there c = its z; elsewhere c = mean_j z_j.  (States the
    // solver produces have z equal across the border families of a node.)
    double m = 0.0;
    int border = -1;
    for (int j = 0; j < r; ++j) {
      int64_t c;
      int pos;
      m += z[j * n + i];
      if (border < 0 && !fam_index(FS.f[j], D, i, &c, &pos)) border = j;
    }
    m = border >= 0 ? z[border * n + i] : m / (double)r;
    double sp = 0.0;
    for (int j = 0; j < r; ++j) {
      int64_t c;
      int pos;
      if (!fam_index(FS.f[j], D, i, &c, &pos)) continue;  // zig-zag border: p = 0
      const ST pj = (ST)(z[j * n + i] - m);
      p[j * n + (int64_t)pos * FS.f[j].C + c] = pj;
      sp += (double)pj;
    }
    cdrift[i] = m;
    X[i] = (ST)(w[i] - sp);
  }
}

// Fused-form state of another handle of the same instance (pcb_copy_state):
// p_j converted to this handle's state type element by element (the family
// layouts are the same), the drift copied, x = w - sum_j p_j recomputed in
// fp64 (the invariant the update keeps; zig-zag border nodes hold p = 0).
template <class SS, class SD>
__global__ void k_copy_fast(const SS* __restrict__ ps, const double* __restrict__ cs,
                            SD* __restrict__ pd, double* __restrict__ cd, SD* __restrict__ X,
                            const double* __restrict__ w, int64_t n, FamSet FS, Dims D) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double sp = 0.0;
    for (int j = 0; j < FS.r; ++j) {
      int64_t c;
      int pos;
      if (!fam_index(FS.f[j], D, i, &c, &pos)) continue;
      const int64_t q = (int64_t)j * n + (int64_t)pos * FS.f[j].C + c;
      const SD v = (SD)ps[q];
      pd[q] = v;
      sp += (double)v;
    }
    cd[i] = cs[i];
    X[i] = (SD)(w[i] - sp);
  }
}

template <class ST>
__global__ void k_init_fast(ST* p, double* cdrift, ST* X, const double* w, int64_t n, int r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < r; ++j) p[j * n + i] = ST(0);
    cdrift[i] = w[i] / (double)r;
    X[i] = (ST)w[i];
  }
}

template <class ST>
__global__ void k_get_fast(const ST* p, const double* cdrift, double* z, int64_t n, FamSet FS,
                           Dims D) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < FS.r; ++j) {
      int64_t c;
      int pos;
      const ST pj = fam_index(FS.f[j], D, i, &c, &pos)
                           ? p[j * n + (int64_t)pos * FS.f[j].C + c] : ST(0);
      z[j * n + i] = (double)pj + cdrift[i];
    }
  }
}

// Check-iteration update from the fp64 shadow y (state p^{k-1}, c^{k-1} -> p^k, c^k).
// The fp32 state p_j sits in family layout [pos][chain]; for the row-like
// families (pos = last grid coordinate) that is the transpose of node order,
// so the grid is walked in 32 x 32 tiles (32 rows of the flattened leading
// coordinates x 32 last-axis positions) and those families' p go through a
// shared-memory tile: both the family-layout and the node-order accesses are
// coalesced.  Per-node arithmetic is the same as a plain node loop.
// Check-iteration update for grids with one row-like family (2D-4 rows, 3D x;
// family 0), in two coalesced passes instead of one tiled pass:
//   k_apply_rows   32 x 32 (chain, position) tiles of family 0: its old state
//                  goes to G in node order (fp32, exact), its new state
//                  (float)y_0 to the family layout, both through shared memory;
//   k_apply_nodes  node order: every other family's state is node-ordered up
//                  to the 3D y permutation, so each node's update reads and
//                  writes coalesced arrays only.
// Same per-node arithmetic and family order as k_apply_fast.
template <class ST>
__global__ void __launch_bounds__(256) k_apply_rows(const double* __restrict__ y0,
                                                    ST* __restrict__ p0, ST* __restrict__ G,
                                                    int C, int L) {
  __shared__ ST tp[32][33];   // [pos][chain]: old state
  __shared__ double ty[32][33];  // [chain][pos]: shadow
  const int tiles_c = (C + 31) / 32;
  const int tiles = tiles_c * ((L + 31) / 32);
  const int tx = threadIdx.x & 31, ty8 = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int c0 = (t % tiles_c) * 32, x0 = (t / tiles_c) * 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = ty8 + 8 * k;  // pos row for p, chain row for y
      const int pos = x0 + r, c = c0 + tx;
      tp[r][tx] = (pos < L && c < C) ? p0[pos * C + c] : ST(0);
      const int cc = c0 + r, xx = x0 + tx;
      ty[r][tx] = (cc < C && xx < L) ? y0[cc * L + xx] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = ty8 + 8 * k;
      const int cc = c0 + r, xx = x0 + tx;  // node (chain cc, pos xx)
      if (cc < C && xx < L) G[cc * L + xx] = tp[tx][r];
      const int pos = x0 + r, c = c0 + tx;  // family slot (pos, chain c)
      if (pos < L && c < C) p0[pos * C + c] = (ST)ty[tx][r];
    }
    __syncthreads();
  }
}

template <int R, class ST>
__global__ void __launch_bounds__(256) k_apply_nodes(
    const double* __restrict__ y, ST* __restrict__ p, const ST* __restrict__ G,
    double* __restrict__ cdrift, ST* __restrict__ X, const double* __restrict__ w, int n,
    int L, int D1, int C1, double* parts) {
  // rows of L nodes; 3D: row = z * D1 + y, family 1 (y lines) at [y][z][x]
  const int rows = n / L;
  ST* p1 = p + (int64_t)n;       // family 1 state
  ST* p2 = p + 2 * (int64_t)n;   // family 2 state (3D z lines: node order)
  const int lane = threadIdx.x & 31;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nwg = gridDim.x * (blockDim.x >> 5);
  double acc = 0.0;
  for (int Rr = wg; Rr < rows; Rr += nwg) {
    const int q1 = R == 3 ? (Rr % D1) * C1 + (Rr / D1) * L : Rr * L;  // family 1 row base
#pragma unroll 2
    for (int x = lane; x < L; x += 32) {
      const int i = Rr * L + x;
      double yv[R];
      ST po[R];
#pragma unroll
      for (int j = 0; j < R; ++j) yv[j] = y[(int64_t)j * n + i];
      po[0] = G[i];
      po[1] = p1[q1 + x];
      if (R == 3) po[R - 1] = p2[i];
      const double wi = w[i], ci = cdrift[i];
      double g = 0.0, sp = 0.0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const ST pn = (ST)yv[j];
        if (j == 1) p1[q1 + x] = pn;
        if (j == 2) p2[i] = pn;
        const double d = (double)pn - (double)po[j];
        g += d;
        sp += (double)pn;
        acc += d * d;
      }
      const double xn = wi - sp;
      X[i] = (ST)xn;
      const double dc = (xn - g) / (double)R;
      cdrift[i] = ci + dc;
      acc += 2.0 * dc * g + (double)R * dc * dc;
    }
  }
  __shared__ double sh[32];
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = tot;
}

constexpr int APPLY_TILE = 32;
constexpr int APPLY_THREADS = 256;  // launch with exactly this many threads

template <int R, class ST>
__global__ void __launch_bounds__(APPLY_THREADS, 3) k_apply_fast(
    const double* __restrict__ y, ST* __restrict__ p, double* __restrict__ cdrift,
    ST* __restrict__ X, const double* __restrict__ w, int64_t n,
    const __grid_constant__ FamSet FS, const __grid_constant__ Dims D, double* parts) {
  constexpr int T = APPLY_TILE, NW = APPLY_THREADS / 32;
  constexpr int CELLS = (T + 1) * T, PASSES = (CELLS + APPLY_THREADS - 1) / APPLY_THREADS;
  // chains R0-1 .. R0+T-1 (zig-zag chain c covers rows c and c+1) x T positions
  __shared__ ST tile[R][T + 1][T + 1];
  const int64_t L = D.nd == 3 ? D.d[2] : D.d[1];
  const int64_t rows = n / L;
  const int64_t D1 = D.nd == 3 ? D.d[1] : 1;
  const int64_t D0L = D.nd == 3 ? D.d[0] * L : 0;
  const int64_t tiles_x = (L + T - 1) / T;
  const int64_t tiles = ((rows + T - 1) / T) * tiles_x;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t R0 = (t / tiles_x) * T;
    const int64_t X0 = (t % tiles_x) * T;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const Fam& F = FS.f[j];
      if (!fam_rowlike(F.kind)) continue;
      ST v[PASSES];
#pragma unroll
      for (int k = 0; k < PASSES; ++k) {
        const int e = threadIdx.x + k * APPLY_THREADS;
        const int cc = e % (T + 1), xx = e / (T + 1);
        const int64_t c = R0 - 1 + cc, x = X0 + xx;
        v[k] = (e < CELLS && c >= 0 && c < F.C && x < L) ? p[j * n + x * F.C + c] : ST(0);
      }
#pragma unroll
      for (int k = 0; k < PASSES; ++k) {
        const int e = threadIdx.x + k * APPLY_THREADS;
        if (e < CELLS) tile[j][e % (T + 1)][e / (T + 1)] = v[k];
      }
    }
    __syncthreads();
    // all loads of the warp's T/NW rows first (memory-level parallelism),
    // then the arithmetic and the stores
    // rows per batch: bounded so the register file holds two blocks per SM
    // (32-bit node indices: pcb_create keeps n below 2^31; family offsets j * n
    // stay 64-bit)
    constexpr int S = 2;
#pragma unroll 1
    for (int b0 = 0; b0 < T / NW; b0 += S) {
    double yv[S][R], wv[S], cv[S];
    ST po[S][R];
    int qv[S][R];
    bool in[S][R];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int Rr = (int)R0 + wp + (b0 + s) * NW, x = (int)X0 + lane;
      const bool ok = Rr < rows && x < L;
      const int i = ok ? Rr * (int)L + x : 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const Fam& F = FS.f[j];
        yv[s][j] = ok ? y[j * n + i] : 0.0;
        if (fam_rowlike(F.kind)) {
          const int c = (F.kind == K_ZZ0 || F.kind == K_ZZ1) ? Rr - ((x + F.phase) & 1) : Rr;
          in[s][j] = ok && c >= 0 && c < F.C;  // zig-zag border node: not in this family
          qv[s][j] = c - ((int)R0 - 1);         // tile row
          po[s][j] = in[s][j] ? tile[j][qv[s][j]][lane] : ST(0);
        } else {
          // COL2 / Z3: family layout == node order; Y3: [y][z][x]
          in[s][j] = ok;
          qv[s][j] = F.kind == K_Y3 ? (Rr % (int)D1) * (int)D0L + (Rr / (int)D1) * (int)L + x : i;
          po[s][j] = ok ? p[(int64_t)j * n + qv[s][j]] : ST(0);
        }
      }
      wv[s] = ok ? w[i] : 0.0;
      cv[s] = ok ? cdrift[i] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int Rr = (int)R0 + wp + (b0 + s) * NW, x = (int)X0 + lane;
      if (Rr >= rows || x >= L) continue;
      const int i = Rr * (int)L + x;
      double g = 0.0, sp = 0.0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (!in[s][j]) continue;
        const ST pn = (ST)yv[s][j];
        if (fam_rowlike(FS.f[j].kind)) tile[j][qv[s][j]][lane] = pn;
        else p[(int64_t)j * n + qv[s][j]] = pn;
        const double d = (double)pn - (double)po[s][j];
        g += d;
        sp += (double)pn;
        acc += d * d;
      }
      const double xn = wv[s] - sp;
      X[i] = (ST)xn;
      const double dc = (xn - g) / (double)R;
      cdrift[i] = cv[s] + dc;
      acc += 2.0 * dc * g + (double)R * dc * dc;
    }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const Fam& F = FS.f[j];
      if (!fam_rowlike(F.kind)) continue;
      const bool zz = F.kind == K_ZZ0 || F.kind == K_ZZ1;
#pragma unroll
      for (int k = 0; k < PASSES; ++k) {
        const int e = threadIdx.x + k * APPLY_THREADS;
        const int cc = e % (T + 1), xx = e / (T + 1);
        const int64_t c = R0 - 1 + cc, x = X0 + xx;
        const int64_t row = zz ? c + ((x + F.phase) & 1) : c;  // the node (c, x) sits in
        if (e < CELLS && c >= 0 && c < F.C && x < L && row >= R0 && row < R0 + T && row < rows)
          p[j * n + x * F.C + c] = tile[j][cc][xx];
      }
    }
    __syncthreads();
  }
  __shared__ double sh[32];
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = tot;
}

// s = y_0 + y_1 + ... (class order), x = w - s, label bits per threshold,
// partial sums: [unary_t (T)], dual, ww, dd.
template <int TT, int R>  // threshold slots compiled in (TT = T, or MAXT generic); R families
__global__ void __launch_bounds__(RED_BLOCK) k_check_nodes(
    const double* __restrict__ y, const double* __restrict__ w, int64_t n, int64_t n_own, int T,
    const double* __restrict__ thr, uint8_t* __restrict__ bits, double* __restrict__ xcur,
    double* __restrict__ parts) {
  double un[TT], th[TT];  // register arrays: every index below is static
#pragma unroll
  for (int t = 0; t < TT; ++t) {
    un[t] = 0.0;
    th[t] = t < T ? thr[t] : 0.0;
  }
  double dual = 0.0, ww = 0.0, dd = 0.0;
  // grid-stride over nodes, U strides at a time with every load of the U
  // nodes issued before the arithmetic (the same nodes per thread, in the same
  // order, as a plain grid-stride loop: the partial sums do not change)
  constexpr int U = 4;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * step) {
    double yv[U][R], wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * step;
      const bool ok = i < n;
#pragma unroll
      for (int j = 0; j < R; ++j) yv[u][j] = ok ? y[(int64_t)j * n + i] : 0.0;
      wv[u] = ok ? w[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * step;
      if (i >= n) break;
      double s = yv[u][0];
#pragma unroll
      for (int j = 1; j < R; ++j) s = s + yv[u][j];
      const double wi = wv[u];
      const double x = wi - s;
      xcur[i] = x;
      const bool own = i < n_own;  // halo copies: labels for the cut, sums are the owner's
      unsigned b = 0;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < T && x > th[t]) {
          b |= 1u << t;
          if (own) un[t] += wi;
        }
      }
      bits[i] = (uint8_t)b;
      if (!own) continue;
      const double sw = s - wi;
      dual += fmin(sw, 0.0);
      ww += wi * wi;
      dd += sw * sw;
    }
  }
  __shared__ double sh[32];
  const int nv = T + 3;
#pragma unroll
  for (int t = 0; t < TT; ++t) {
    if (t >= T) break;
    const double v = block_sum(un[t], sh);
    if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * nv + t] = v;
  }
  double v = block_sum(dual, sh);
  if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * nv + T] = v;
  v = block_sum(ww, sh);
  if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * nv + T + 1] = v;
  v = block_sum(dd, sh);
  if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * nv + T + 2] = v;
}

struct DirGeom {
  int ndir;
  int off[4][3];  // direction offsets (graph.DIRECTIONS)
};

// cut_t = sum_edges a_e |lab_t(i) - lab_t(j)|, per direction array element.
// One block walks whole grid rows (flattened leading coordinates); per row
// and direction the edge-array row and the neighbour offset are computed
// once, and the threads stride along the last axis (coalesced a_e and bits).
template <int TT>
__global__ void k_check_edges(const __grid_constant__ Dims D, const __grid_constant__ DirGeom DG,
                              const __grid_constant__ DirPtrs dw, const uint8_t* __restrict__ bits,
                              int T, double* __restrict__ parts) {
  double cut[TT];
#pragma unroll
  for (int t = 0; t < TT; ++t) cut[t] = 0.0;
  const int nd = D.nd;
  const int64_t L = nd == 3 ? D.d[2] : D.d[1];
  const int64_t rows = nd == 3 ? D.d[0] * D.d[1] : D.d[0];
  // one warp per grid row (the rows of a block in flight together: the
  // label loads of a row are few and latency bound); lanes along the row
  const int lane = threadIdx.x & 31, nwb = blockDim.x >> 5;
  for (int64_t Rr = (int64_t)blockIdx.x * nwb + (threadIdx.x >> 5); Rr < rows;
       Rr += (int64_t)gridDim.x * nwb) {
    int64_t co[2] = {Rr, 0};
    if (nd == 3) {
      co[0] = Rr / D.d[1];
      co[1] = Rr % D.d[1];
    }
    const int64_t base = Rr * L;
    for (int k = 0; k < DG.ndir; ++k) {
      // this row holds the "sa" end of direction-k edges iff every leading
      // coordinate stays in range
      bool ok = true;
      int64_t erow = 0, joff = 0, stride = L;
#pragma unroll
      for (int a = 1; a >= 0; --a) {
        if (a > nd - 2) continue;
        joff += DG.off[k][a] * stride;
        stride *= D.d[a];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        if (a > nd - 2) continue;
        const int o = DG.off[k][a];
        const int64_t len = D.d[a] - (o < 0 ? -o : o);
        const int64_t q = co[a] - (o >= 0 ? 0 : -o);
        if (q < 0 || q >= len) ok = false;
        erow = erow * (len > 0 ? len : 1) + q;
      }
      if (!ok) continue;
      const int oL = DG.off[k][nd - 1];
      joff += oL;
      const int64_t lenL = L - (oL < 0 ? -oL : oL), loL = oL >= 0 ? 0 : -oL;
      const double* av = dw.p[k] + erow * lenL - loL;  // element (erow, x - loL)
      const uint8_t* bn = bits + base + joff;
      if ((L & 3) == 0) {
        // four positions per lane: the row's labels and the neighbours' as
        // aligned 32-bit words (the neighbour row funnel-shifted into place);
        // the weight is read only where a label differs (boundary edges)
        const uint32_t* w32 = reinterpret_cast<const uint32_t*>(bits);
        const int64_t nb0 = base + joff;  // neighbour of position 0
        const unsigned sh = (unsigned)(nb0 & 3) * 8u;
        for (int64_t x4 = (int64_t)lane * 4; x4 < L; x4 += 128) {
          const uint32_t own = w32[(base + x4) >> 2];
          const int64_t q = (nb0 + x4) >> 2;
          const uint32_t lo = w32[q];
          const uint32_t nb = sh ? __funnelshift_r(lo, w32[q + 1], sh) : lo;
          const uint32_t diff4 = own ^ nb;
          if (!diff4) continue;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int64_t x = x4 + b;
            const unsigned diff = (diff4 >> (8 * b)) & 0xffu;
            if (diff && x >= loL && x < loL + lenL) {
              const double a = av[x];
#pragma unroll
              for (int t = 0; t < TT; ++t)
                if ((diff >> t) & 1u) cut[t] += a;  // bits >= T are never set
            }
          }
        }
        continue;
      }
#pragma unroll 4
      for (int64_t x = loL + lane; x < loL + lenL; x += 32) {
        const unsigned diff = (unsigned)bits[base + x] ^ (unsigned)bn[x];
        if (diff) {
          const double a = av[x];
#pragma unroll
          for (int t = 0; t < TT; ++t)
            if ((diff >> t) & 1u) cut[t] += a;  // bits >= T are never set
        }
      }
    }
  }
  __shared__ double sh[32];
#pragma unroll
  for (int t = 0; t < TT; ++t) {
    if (t >= T) break;
    const double v = block_sum(cut[t], sh);
    if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * T + t] = v;
  }
}

__global__ void k_labels(const uint8_t* bits, int64_t n, int t, uint8_t* lab) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lab[i] = (bits[i] >> t) & 1u;
}

// Jaccard distance of every logged packed labeling (slot i at lab + i * nb)
// against ref: one block per slot, integer popcounts (exact).
// Jaccard distance of every logged labeling against ref, in two steps: blocks
// of grid (chunks, labelings) popcount one chunk of one labeling (8-byte words
// when the rows are 8-byte aligned) and add their integer counts into the
// labeling's (intersection, union) pair -- integer atomics, so the result is
// independent of the order; k_log_jaccard_fin turns the pairs into distances.
__global__ void k_log_jaccard_part(const uint8_t* __restrict__ lab, const uint8_t* __restrict__ ref,
                                   int64_t nb, unsigned long long* __restrict__ acc) {
  const uint8_t* a = lab + (int64_t)blockIdx.y * nb;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long inter = 0, uni = 0;
  if ((nb & 7) == 0) {
    const unsigned long long* a8 = reinterpret_cast<const unsigned long long*>(a);
    const unsigned long long* r8 = reinterpret_cast<const unsigned long long*>(ref);
    const int64_t nw = nb >> 3;
#pragma unroll 4
    for (int64_t q = t0; q < nw; q += stride) {
      const unsigned long long x = __ldg(a8 + q), y = __ldg(r8 + q);
      inter += __popcll(x & y);
      uni += __popcll(x | y);
    }
  } else {
    for (int64_t q = t0; q < nb; q += stride) {
      const unsigned x = a[q], y = ref[q];
      inter += __popc(x & y);
      uni += __popc(x | y);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    inter += __shfl_down_sync(0xffffffffu, inter, o);
    uni += __shfl_down_sync(0xffffffffu, uni, o);
  }
  if ((threadIdx.x & 31) == 0 && (inter | uni)) {
    atomicAdd(acc + 2 * blockIdx.y, inter);
    atomicAdd(acc + 2 * blockIdx.y + 1, uni);
  }
}

__global__ void k_log_jaccard_fin(const unsigned long long* acc, int64_t nlab, double* out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nlab;
       k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long ti = acc[2 * k], tu = acc[2 * k + 1];
    out[k] = tu == 0 ? 0.0 : 1.0 - (double)ti / (double)tu;
  }
}

// np.packbits order: byte q holds labels 8q..8q+7, label 8q in bit 7.
__global__ void k_pack(const uint8_t* bits, int64_t n, int t, uint8_t* out) {
  const int64_t nb = (n + 7) / 8;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nb;
       q += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t i = q * 8 + k;
      const unsigned l = i < n ? ((bits[i] >> t) & 1u) : 0u;
      v |= l << (7 - k);
    }
    out[q] = (uint8_t)v;
  }
}

__global__ void k_sum_classes(const double* y, int r, int64_t n, double* s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = y[i];
    for (int j = 1; j < r; ++j) v = v + y[(int64_t)j * n + i];
    s[i] = v;
  }
}

// lam_j = (v_j + corr) * support_j, corr = (w - sum_k v_k) / d on covered nodes.
__global__ void k_project_L(const double* w, const int64_t* deg, const uint8_t* sup, int r,
                            int64_t n, const double* v, double* out, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double total = v[i];
    for (int j = 1; j < r; ++j) total = total + v[(int64_t)j * n + i];
    double corr = 0.0;
    if (deg[i] == 0) {
      if (w[i] != 0.0) atomicExch(bad, 1);
    } else {
      corr = (w[i] - total) / (double)deg[i];
    }
    for (int j = 0; j < r; ++j) {
      const int64_t q = (int64_t)j * n + i;
      out[q] = (v[q] + corr) * (double)sup[q];
    }
  }
}

__global__ void k_diff_norm(const double* a, const double* b, int64_t n, double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    acc += d * d;
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

int grid_for(int64_t n, int block, int cap) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// ----------------------------------------------------------------- device buffers

// Device memory comes from a per-device stream-ordered pool that keeps what
// it has mapped (release threshold lifted): a handle created after another
// was destroyed reuses the mapped memory instead of paying cudaFree's unmap
// and cudaMalloc's remap (measured ~250 ms of create + destroy at 16.7M
// nodes with plain cudaMalloc/cudaFree).  pcb_release_memory trims it.
cudaMemPool_t g_pool[64] = {};

cudaMemPool_t device_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      (void)cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pool[dev] = pool;
  }
  return g_pool[dev];
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool pooled = false;
  // the owning handle's stream (pcb_solver binds its buffers): frees are
  // stream-ordered behind that handle's queued work instead of a device-wide
  // sync that would stall other handles' streams and break their graph captures
  cudaStream_t* owner = nullptr;
  int alloc(size_t count) {
    free();
    if (count == 0) count = 1;
    const size_t bytes = count * sizeof(T);
    cudaError_t e = cudaErrorMemoryAllocation;
    if (cudaMemPool_t pool = device_pool()) {
      // allocated in legacy-stream order, complete before any stream uses it
      e = cudaMallocFromPoolAsync((void**)&p, bytes, pool, 0);
      if (e == cudaSuccess) e = cudaStreamSynchronize(0);
      pooled = e == cudaSuccess;
    }
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      e = cudaMalloc(&p, bytes);
      pooled = false;
    }
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      p = nullptr;
      return fail(PCB_E_NOMEM, "device allocation (%zu bytes): %s", bytes, cudaGetErrorString(e));
    }
    n = count;
    return 0;
  }
  void free() {
    if (p) {
      if (pooled && owner) {
        cudaFreeAsync(p, *owner);
      } else if (pooled) {
        cudaDeviceSynchronize();  // unowned scratch: queued work on any stream may still use p
        cudaFreeAsync(p, 0);
      } else {
        cudaFree(p);
      }
    }
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
};

#include "hostio.cuh"

// grow b to hold `need` elements, keeping its first `used` (stream-ordered copy)
template <class T>
int grow_keep(DBuf<T>& b, size_t need, size_t used, cudaStream_t st, size_t min_cap = 0) {
  if (b.n >= need && b.p) return 0;
  DBuf<T> nb;
  nb.owner = b.owner;
  size_t cap = b.n * 2;
  if (cap < need) cap = need;
  if (cap < min_cap) cap = min_cap;
  if (int e = nb.alloc(cap)) return e;
  if (used > 0 && b.p) {
    cudaError_t ce = cudaMemcpyAsync(nb.p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail(PCB_E_CUDA, "log growth: %s", cudaGetErrorString(ce));
  }
  std::swap(b.p, nb.p);
  std::swap(b.n, nb.n);
  std::swap(b.pooled, nb.pooled);
  return 0;  // nb now owns (and frees) the old storage
}

}  // namespace

struct pcb_solver {
  int device = 0;
  cudaStream_t stream = 0;
  int precision = PCB_F64;
  int conn = 0;
  Dims D{};
  DirGeom DG{};
  int r = 0;
  int64_t n = 0;
  int64_t n_own = -1;  // nodes [n_own, n) are halo copies (pcb_set_owned); -1: none
  Fam fam[MAXR]{};
  int order[MAXR]{};  // fast-mode processing order (last one covers all nodes)
  int maxm = 1;
  int64_t maxC = 1;
  int64_t launches = 0;
  bool have_state = false;
  bool have_shadow = false;
  bool y_valid = false;  // y holds the last shadow (not clobbered by aar_run)
  bool have_check = false;
  bool have_best = false;
  bool x_in_best = false;  // the current check's x lives in bestx (pcb_keep_best swapped)
  int alg = 0;            // 0: AAR state; PCB_ALG_*: a dual scheme owns y/z
  double fista_t = 1.0;   // FISTA momentum parameter t_k
  int check_T = 0;

  DBuf<double> w;
  DBuf<double> dirw[4];
  DBuf<double> dirw_base[4];  // lambda = 1 weights, kept on the first pcb_scale_pairwise
  DBuf<double> wf64[MAXR];
  DBuf<float> wf32[MAXR];
  DBuf<double> z;      // F64: r*n AAR point
  DBuf<double> y;      // r*n shadow (both modes)
  DBuf<float> p32;     // F32: r*n shadow state
  pcb::fast::Maps maps[MAXR]{};  // F32: TMA descriptors of the strided families
  DBuf<double> cdrift; // F32: n drift
  DBuf<float> X32;     // F32: primal
  DBuf<float> G32;     // F32: accumulator
  DBuf<double> tmp;    // r*n scratch (project_K)
  DBuf<double> yprev;  // r*n previous shadow (dual_tol)
  DBuf<uint8_t> bits;
  DBuf<double> xcur;
  DBuf<uint8_t> bestlab;
  DBuf<double> bestx;
  DBuf<double> parts;  // reduction partials
  DBuf<double> vals;   // reduced values
  DBuf<double> norms;  // per-iteration step norms
  DBuf<int> sp_cx, sp_fx;
  DBuf<double> sp_cy, sp_fy;
  DBuf<uint8_t> packed;
  // solve log (pcb_log_*): step norms and packed check labelings stay on the
  // device until the solve ends, so check cycles need one host sync only
  bool logging = false;
  DBuf<double> normlog;
  int64_t nlog = 0;
  DBuf<uint8_t> lablog;
  int64_t nlab = 0;
  int64_t spill_per = 0;  // spill entries per thread
  unsigned fmask = 0xfu;  // families swept by this handle (sharded runs split them)
  int nbk[MAXR]{};        // fp32 path: blocks per chain (intra-chain split), 1 = whole chains
  int lbk[MAXR]{};        // block length (positions)
  DBuf<int> merge;        // merge points, family j at merge_off[j] (nbk[j] * C_j entries)
  // Double-buffered fp32 step with verified sweeps:
  // alternate state buffers (the step reads p32 / cdrift / X32 and writes
  // these, then the two sets swap), per-family segment hints and the
  // per-family device mode words {mode (1 = VER), count}.
  bool dbuf = false;
  // verify while fewer than vtheta % of a family's chains need a repair (the
  // verified sweep's break-even on cfg5 is a few %: nearly every warp then
  // holds a repairing lane)
  int vtheta = 3;
  DBuf<float> p32b, G32b, X32b;
  DBuf<double> cdriftb;
  DBuf<uint16_t> sg[MAXR];
  DBuf<int> vstate;
  pcb::fast::Maps maps2[MAXR]{};  // TMA descriptors of the alternate buffers
  // F64S (fp64 split mode): the fast path's state in fp64 (p, G, X; weights
  // wf64), the same kernels with fp64 ring slots and fp64 scans
  DBuf<double> p64, G64, X64;
  pcb::fast::Maps maps64[MAXR]{};
  // CUDA graphs of GRAPH_STEPS plain iterations (launch-bound small grids),
  // one per buffer parity of the double-buffered step
  int par = 0;  // swaps of the double-buffered state, mod 2
  cudaStream_t gstream = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t glaunches[2] = {0, 0};  // kernel launches in each graph
  // graphs are captured once the handle has run this many plain iterations
  // eagerly (capture + instantiate cost about 80 iterations' worth of the
  // replay's saving: short solves never pay it); pcb_set_graph_after
  int64_t graph_after = 64;
  int64_t plain_done = 0;  // plain (flags == 0) iterations run on this handle
  DBuf<double> gnorms;
  int64_t merge_off[MAXR]{};
  // merges of a step run on a side stream, overlapping the sweeps (they
  // depend only on the state at the start of the step)
  bool overlap_merges = true;  // PCB_OVERLAP_MERGE=0 runs them inline
  // programmatic dependent launch of the MID / LAST sweeps of a plain step
  // (PCB_PDL=0: off): their scans start in the previous sweep's tail, the
  // first read of its output waits in griddepcontrol.wait
  DBuf<unsigned long long> jacc;  // (intersection, union) per logged labeling
  bool use_pdl = true;
  bool pdl_launch = false;  // the next launch_sweep is programmatic
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_merge[MAXR] = {};
  // recorded right after the previous step's last sweep: the next step's
  // merges need only that (not the norm reduction queued behind it).  Valid
  // only between steps of one pcb_aar_step call outside graph boundaries.
  cudaEvent_t ev_sweeps = nullptr;
  bool sweeps_ev_ok = false;
  // profiling: event pairs around family launches
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_fam;
  template <class... B>
  void bind(B&... b) {
    ((b.owner = &stream), ...);
  }
  template <class T, size_t K>
  void bind_arr(DBuf<T> (&a)[K]) {
    for (auto& b : a) b.owner = &stream;
  }
  pcb_solver() {
    bind(w, z, y, p32, cdrift, X32, G32, tmp, yprev, bits, xcur, bestlab, bestx, parts, vals,
         norms, sp_cx, sp_fx, sp_cy, sp_fy, packed, normlog, lablog, merge, p32b, G32b, X32b,
         cdriftb, vstate, p64, G64, X64, gnorms, jacc);
    bind_arr(sg);
    bind_arr(dirw);
    bind_arr(dirw_base);
    bind_arr(wf64);
    bind_arr(wf32);
  }
  ~pcb_solver() {
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_sweeps) cudaEventDestroy(ev_sweeps);
    for (cudaEvent_t e : ev_merge)
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    for (cudaGraphExec_t g : gexec)
      if (g) cudaGraphExecDestroy(g);
    if (gstream) cudaStreamDestroy(gstream);
  }
};

namespace {

// The fast path's state of a handle by storage type: float for PCB_F32,
// double for PCB_F64S (same kernels, templated on the type).
template <class ST>
struct FastState;
template <>
struct FastState<float> {
  static float* p(pcb_solver* h) { return h->p32.p; }
  static float* G(pcb_solver* h) { return h->G32.p; }
  static float* X(pcb_solver* h) { return h->X32.p; }
  static const float* wf(pcb_solver* h, int j) { return h->wf32[j].p; }
  static pcb::fast::Maps* maps(pcb_solver* h) { return h->maps; }
};
template <>
struct FastState<double> {
  static double* p(pcb_solver* h) { return h->p64.p; }
  static double* G(pcb_solver* h) { return h->G64.p; }
  static double* X(pcb_solver* h) { return h->X64.p; }
  static const double* wf(pcb_solver* h, int j) { return h->wf64[j].p; }
  static pcb::fast::Maps* maps(pcb_solver* h) { return h->maps64; }
};

int set_dev(pcb_solver* h) {
  CUDA_TRY(cudaSetDevice(h->device));
  return 0;
}

// Record an event pair slot around a family launch (profiling only).
cudaEvent_t prof_event(pcb_solver* h) {
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    h->ev_pool.push_back(e);
  }
  return h->ev_pool[h->ev_used++];
}

void prof_begin(pcb_solver* h, int fam) {
  if (!h->profiling) return;
  cudaEvent_t e = prof_event(h);
  if (e) {
    cudaEventRecord(e, h->stream);
    h->ev_fam.push_back(fam);
  }
}

void prof_end(pcb_solver* h) {
  if (!h->profiling) return;
  cudaEvent_t e = prof_event(h);
  if (e) cudaEventRecord(e, h->stream);
}

FamSet famset(const pcb_solver* h) {
  FamSet FS{};
  FS.r = h->r;
  for (int j = 0; j < h->r; ++j) FS.f[j] = h->fam[j];
  return FS;
}

Spill spill_of(pcb_solver* h) {
  return Spill{h->sp_cx.p, h->sp_cy.p, h->sp_fx.p, h->sp_fy.p};
}

int setup_geometry(pcb_solver* h) {
  const int64_t* d = h->D.d;
  auto mk = [](int kind, int m, int64_t C, int64_t cdiv, int64_t chi, int64_t clo, int64_t ns,
               int64_t zz, int phase) {
    Fam F;
    F.kind = kind;
    F.m = m;
    F.C = C;
    F.cdiv = cdiv;
    F.chi = chi;
    F.clo = clo;
    F.ns = ns;
    F.zz = zz;
    F.phase = phase;
    return F;
  };
  if (h->conn == PCB_CONN_2D4 || h->conn == PCB_CONN_2D8) {
    const int64_t H = d[0], W = d[1];
    h->fam[0] = mk(K_ROW2, (int)W, H, 1, W, 0, 1, 0, 0);
    h->fam[1] = mk(K_COL2, (int)H, W, 1, 1, 0, W, 0, 0);
    h->r = 2;
    if (h->conn == PCB_CONN_2D8) {
      const int64_t C = (H >= 2 && W >= 2) ? H - 1 : 0;
      h->fam[2] = mk(K_ZZ0, (int)W, C, 1, W, 0, 1, W, 0);
      h->fam[3] = mk(K_ZZ1, (int)W, C, 1, W, 0, 1, W, 1);
      h->r = 4;
    }
  } else {
    const int64_t D0 = d[0], D1 = d[1], D2 = d[2];
    h->fam[0] = mk(K_X3, (int)D2, D0 * D1, 1, D2, 0, 1, 0, 0);
    h->fam[1] = mk(K_Y3, (int)D1, D0 * D2, D2, D1 * D2, 1, D2, 0, 0);
    h->fam[2] = mk(K_Z3, (int)D0, D1 * D2, 1, 1, 0, D1 * D2, 0, 0);
    h->r = 3;
  }
  // fast-path order: a row-like family first (its G pass is write-only), a
  // strided full-coverage family last (zig-zags leave border singletons)
  if (h->r == 4) {
    h->order[0] = 0;
    h->order[1] = 2;
    h->order[2] = 3;
    h->order[3] = 1;
  } else {
    for (int j = 0; j < h->r; ++j) h->order[j] = j;
  }
  h->maxm = 1;
  h->maxC = 1;
  for (int j = 0; j < h->r; ++j) {
    if (h->fam[j].m > h->maxm) h->maxm = h->fam[j].m;
    if (h->fam[j].C > h->maxC) h->maxC = h->fam[j].C;
  }
  // direction geometry for the certificate kernel
  static const int off2d4[2][3] = {{0, 1, 0}, {1, 0, 0}};
  static const int off2d8[4][3] = {{0, 1, 0}, {1, 0, 0}, {1, 1, 0}, {1, -1, 0}};
  static const int off3d6[3][3] = {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}};
  if (h->conn == PCB_CONN_2D4) {
    h->DG.ndir = 2;
    memcpy(h->DG.off, off2d4, sizeof(off2d4));
  } else if (h->conn == PCB_CONN_2D8) {
    h->DG.ndir = 4;
    memcpy(h->DG.off, off2d8, sizeof(off2d8));
  } else {
    h->DG.ndir = 3;
    memcpy(h->DG.off, off3d6, sizeof(off3d6));
  }
  return 0;
}

int64_t dir_size(const pcb_solver* h, int k) {
  int64_t s = 1;
  for (int a = 0; a < h->D.nd; ++a) {
    int o = h->DG.off[k][a];
    int64_t len = h->D.d[a] - (o < 0 ? -o : o);
    s *= len > 0 ? len : 0;
  }
  return s;
}

int ensure_wf64(pcb_solver* h) {
  DirPtrs dp{};
  for (int k = 0; k < h->DG.ndir; ++k) dp.p[k] = h->dirw[k].p;
  for (int j = 0; j < h->r; ++j) {
    if (h->wf64[j].p) continue;
    const Fam& F = h->fam[j];
    const int64_t cnt = F.C * (int64_t)(F.m > 1 ? F.m - 1 : 0);
    if (int e = h->wf64[j].alloc((size_t)cnt)) return e;
    if (cnt > 0) {
      k_build_family_weights<double><<<grid_for(cnt, 256, 148 * 16), 256, 0, h->stream>>>(
          F, h->D, dp, h->wf64[j].p);
      LAUNCH_CHECK(h);
    }
  }
  return 0;
}

int ensure_wf32(pcb_solver* h) {
  DirPtrs dp{};
  for (int k = 0; k < h->DG.ndir; ++k) dp.p[k] = h->dirw[k].p;
  for (int j = 0; j < h->r; ++j) {
    if (h->wf32[j].p) continue;
    const Fam& F = h->fam[j];
    const int64_t cnt = F.C * (int64_t)(F.m > 1 ? F.m - 1 : 0);
    if (int e = h->wf32[j].alloc((size_t)cnt)) return e;
    if (cnt > 0) {
      k_build_family_weights<float><<<grid_for(cnt, 256, 148 * 16), 256, 0, h->stream>>>(
          F, h->D, dp, h->wf32[j].p);
      LAUNCH_CHECK(h);
    }
  }
  return 0;
}

__global__ void k_scale(const double* base, double* out, int64_t n, double f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = base[i] * f;  // graph.py:182-187: edge_a * factor
}

int ensure_spill(pcb_solver* h) {
  if (h->sp_cx.p) return 0;
  const int64_t per = h->maxm + 1 > HC ? h->maxm + 1 - HC : 1;
  const int64_t threads = ((h->maxC + FAM_BLOCK - 1) / FAM_BLOCK) * FAM_BLOCK;
  const size_t cnt = (size_t)(per * threads);
  if (int e = h->sp_cx.alloc(cnt)) return e;
  if (int e = h->sp_fx.alloc(cnt)) return e;
  if (int e = h->sp_cy.alloc(cnt)) return e;
  if (int e = h->sp_fy.alloc(cnt)) return e;
  h->spill_per = per;
  return 0;
}

template <int RL>
int launch_exact_sweep(pcb_solver* h, const pcb::exact::ArgSet& S, int nfam, int64_t maxC) {
  constexpr int bytes = pcb::exact::WARPS * pcb::exact::warp_bytes<RL>();
  static unsigned set_mask = 0;
  const unsigned bit = 1u << (h->device & 31);
  if (!(set_mask & bit)) {
    CUDA_TRY(cudaFuncSetAttribute(pcb::exact::k_sweep_exact<RL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    set_mask |= bit;
  }
  const int per = pcb::exact::WARPS * 32;
  const dim3 g((unsigned)((maxC + per - 1) / per), (unsigned)nfam);
  pcb::exact::k_sweep_exact<RL><<<g, per, bytes, h->stream>>>(S);
  return 0;
}

// PCB_EXACT_THREAD=1 selects the thread-per-chain kernel (A/B comparisons)
bool exact_thread_kernel() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PCB_EXACT_THREAD");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// exact prox of families j0..j1-1: srcs[j-j0] -> dsts[j-j0] (n each).  The
// families are independent and go out as one launch (blockIdx.y = family);
// under profiling that launch is timed as family j0.
int sweep_exact_sel(pcb_solver* h, int j0, int j1, const double* const* srcs,
                    double* const* dsts, bool zero_singletons = false) {
  const Spill sp = spill_of(h);
  // a zig-zag family leaves border nodes as one-node chains (y = 0 there,
  // decompose.py:153-183) that no kernel writes: clear them in a fresh dst
  if (zero_singletons)
    for (int j = j0; j < j1; ++j)
      if (h->fam[j].kind == K_ZZ0 || h->fam[j].kind == K_ZZ1)
        CUDA_TRY(cudaMemsetAsync(dsts[j - j0], 0, h->n * sizeof(double), h->stream));
  if (exact_thread_kernel()) {
    for (int j = j0; j < j1; ++j) {
      const Fam& F = h->fam[j];
      if (F.C == 0) continue;
      const int g = (int)((F.C + FAM_BLOCK - 1) / FAM_BLOCK);
      prof_begin(h, j);
      k_family_exact<<<g, FAM_BLOCK, 0, h->stream>>>(F, srcs[j - j0], dsts[j - j0], h->wf64[j].p,
                                                      sp);
      prof_end(h);
      LAUNCH_CHECK(h);
    }
    return 0;
  }
  const int64_t gs = ((h->maxC + FAM_BLOCK - 1) / FAM_BLOCK) * FAM_BLOCK;
  auto args_of = [&](int j) {
    return pcb::exact::Args{h->fam[j],   srcs[j - j0], dsts[j - j0], h->wf64[j].p,
                            sp.cx,       sp.cy,        sp.fx,        sp.fy,
                            gs};
  };
  // ring depth from the parallelism on offer (warps per SM over the sweep)
  int64_t warps = 0;
  for (int j = j0; j < j1; ++j) warps += (h->fam[j].C + 31) / 32;
  const bool deep = warps < 148 * 12;
  auto launch = [&](const pcb::exact::ArgSet& S, int nfam, int64_t maxC) {
    return deep ? launch_exact_sweep<32>(h, S, nfam, maxC)
                : launch_exact_sweep<16>(h, S, nfam, maxC);
  };
  pcb::exact::ArgSet S{};
  int64_t maxC = 0;
  for (int j = j0; j < j1; ++j) {
    S.f[j - j0] = args_of(j);
    maxC = h->fam[j].C > maxC ? h->fam[j].C : maxC;
  }
  if (maxC == 0) return 0;
  prof_begin(h, j0);  // one launch for all families: timed as family j0
  if (int e = launch(S, j1 - j0, maxC)) return e;
  prof_end(h);
  LAUNCH_CHECK(h);
  return 0;
}

// exact prox of every family: src (r*n) -> dst (r*n), y_j = z_j - prox(z_j)
int sweep_exact(pcb_solver* h, const double* src, double* dst, bool zero_singletons = false) {
  const double* srcs[MAXR];
  double* dsts[MAXR];
  for (int j = 0; j < h->r; ++j) {
    srcs[j] = src + (int64_t)j * h->n;
    dsts[j] = dst + (int64_t)j * h->n;
  }
  return sweep_exact_sel(h, 0, h->r, srcs, dsts, zero_singletons);
}

constexpr int NODE_GRID = 148 * 8;

int update_exact(pcb_solver* h, double* norm_slot) {
  const int g = grid_for(h->n, RED_BLOCK, NODE_GRID);
  switch (h->r) {
    case 2:
      k_update_exact<2><<<g, RED_BLOCK, 0, h->stream>>>(h->z.p, h->y.p, h->w.p, h->n, h->parts.p);
      break;
    case 3:
      k_update_exact<3><<<g, RED_BLOCK, 0, h->stream>>>(h->z.p, h->y.p, h->w.p, h->n, h->parts.p);
      break;
    default:
      k_update_exact<4><<<g, RED_BLOCK, 0, h->stream>>>(h->z.p, h->y.p, h->w.p, h->n, h->parts.p);
      break;
  }
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, norm_slot, 1);
  LAUNCH_CHECK(h);
  return 0;
}

template <class ST>
int apply_fast(pcb_solver* h, double* norm_slot) {
  ST* const P = FastState<ST>::p(h);
  ST* const Gb = FastState<ST>::G(h);
  ST* const Xb = FastState<ST>::X(h);
  const int g = grid_for(h->n, RED_BLOCK, NODE_GRID);
  const Fam* F = h->fam;
  const unsigned all = (1u << h->r) - 1u;
  const bool two_pass = (h->fmask & all) == all &&
                        ((h->r == 2 && F[0].kind == K_ROW2 && F[1].kind == K_COL2) ||
                         (h->r == 3 && F[0].kind == K_X3 && F[1].kind == K_Y3 && F[2].kind == K_Z3));
  if (two_pass && getenv("PCB_APPLY_TILED") == nullptr) {
    const int C0 = (int)F[0].C, L = (int)F[0].m;  // rows of L nodes
    k_apply_rows<<<NODE_GRID, 256, 0, h->stream>>>(h->y.p, P, Gb, C0, L);
    LAUNCH_CHECK(h);
    const int n = (int)h->n;
    const int D1 = h->r == 3 ? (int)h->D.d[1] : 1;
    const int C1 = h->r == 3 ? (int)(h->D.d[0] * h->D.d[2]) : 0;  // y family: [y][z][x]
    if (h->r == 2)
      k_apply_nodes<2, ST><<<g, 256, 0, h->stream>>>(h->y.p, P, Gb, h->cdrift.p, Xb,
                                                h->w.p, n, L, D1, C1, h->parts.p);
    else
      k_apply_nodes<3, ST><<<g, 256, 0, h->stream>>>(h->y.p, P, Gb, h->cdrift.p, Xb,
                                                h->w.p, n, L, D1, C1, h->parts.p);
    LAUNCH_CHECK(h);
    k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, norm_slot, 1);
    LAUNCH_CHECK(h);
    return 0;
  }
  switch (h->r) {
    case 2:
      k_apply_fast<2, ST><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, P, h->cdrift.p, Xb,
                                                      h->w.p, h->n, famset(h), h->D, h->parts.p);
      break;
    case 3:
      k_apply_fast<3, ST><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, P, h->cdrift.p, Xb,
                                                      h->w.p, h->n, famset(h), h->D, h->parts.p);
      break;
    default:
      k_apply_fast<4, ST><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, P, h->cdrift.p, Xb,
                                                      h->w.p, h->n, famset(h), h->D, h->parts.p);
      break;
  }
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, norm_slot, 1);
  LAUNCH_CHECK(h);
  return 0;
}

template <int ROLE, bool ROWLIKE, bool VER = false, class ST = float, bool RT = false,
          bool XG = false>
int launch_sweep(pcb_solver* h, const pcb::fast::ArgsT<ST>& a_in, const pcb::fast::Maps& M) {
  if constexpr (ROLE == pcb::fast::LAST && !XG && !VER) {  // the exporting variant of LAST
    if (a_in.export_g) return launch_sweep<ROLE, ROWLIKE, VER, ST, RT, true>(h, a_in, M);
  }
  pcb::fast::ArgsT<ST> a = a_in;
  pcb::fast::args_inplace(a);
#ifndef PCB_RING_PAD
#define PCB_RING_PAD 0  // experiment knob: extra dynamic smem per block (occupancy probes)
#endif
  const int bytes = pcb::fast::WARPS * pcb::fast::ring_bytes_host<ROLE, ST>() + PCB_RING_PAD;
  // set once per device (outside any later CUDA-graph capture of the sweep)
  static unsigned set_mask = 0;
  const unsigned bit = 1u << (h->device & 31);
  if (!(set_mask & bit)) {
    CUDA_TRY(cudaFuncSetAttribute(pcb::fast::k_sweep<ROLE, ROWLIKE, VER, ST, RT, XG>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    set_mask |= bit;
  }
  const int per = pcb::fast::WARPS * 32;
  const dim3 g((unsigned)((a.F.C + per - 1) / per), (unsigned)(a.merge ? a.nb : 1));
  if (h->pdl_launch) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = dim3(per);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, pcb::fast::k_sweep<ROLE, ROWLIKE, VER, ST, RT, XG>, a, M));
  } else {
    pcb::fast::k_sweep<ROLE, ROWLIKE, VER, ST, RT, XG><<<g, per, bytes, h->stream>>>(a, M);
  }
  LAUNCH_CHECK(h);
  return 0;
}

// a row family with a row map (Maps::row) in the first or shadow role runs
// the row-TMA sweep; other row-like families (zig-zags, later roles) the
// per-lane cp.async one
template <int ROLE, class ST>
int launch_rowlike(pcb_solver* h, const pcb::fast::ArgsT<ST>& a, const pcb::fast::Maps& M) {
  if constexpr (ROLE == pcb::fast::FIRST || ROLE == pcb::fast::SHADOW) {
    if (M.row && M.tma) return launch_sweep<ROLE, false, false, ST, true>(h, a, M);
  }
  return launch_sweep<ROLE, true, false, ST>(h, a, M);
}

template <int ROLE, class ST>
int launch_role(pcb_solver* h, const pcb::fast::ArgsT<ST>& a, int j) {
  pcb::fast::Maps* M = FastState<ST>::maps(h);
  return fam_rowlike(a.F.kind) ? launch_rowlike<ROLE, ST>(h, a, M[j])
                               : launch_sweep<ROLE, false, false, ST>(h, a, M[j]);
}

// SCAN and VER sweeps of one family in the double-buffered step: both are
// launched, the device mode word picks the one that runs
template <int ROLE, bool ROWLIKE>
int launch_verify(pcb_solver* h, const pcb::fast::Args& a_in) {
  pcb::fast::Args a = a_in;
  pcb::fast::args_inplace(a);
  constexpr int per = pcb::fast::LV_WARPS * 32;
  const unsigned g = (unsigned)((a.F.C + per - 1) / per);
  pcb::fast::k_verify<ROLE, ROWLIKE><<<g, per, 0, h->stream>>>(a);
  LAUNCH_CHECK(h);
  return 0;
}

// PCB_VERIFY_RING=1: the verified sweep inside the ring kernel (A/B experiments)
bool verify_ring() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PCB_VERIFY_RING");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int ROLE, class ST>
int launch_role_v(pcb_solver* h, const pcb::fast::ArgsT<ST>& a, int j) {
  if constexpr (!std::is_same<ST, float>::value) {
    return launch_role<ROLE, ST>(h, a, j);
  } else {
  const bool rl = fam_rowlike(a.F.kind);
  if (int e = rl ? launch_rowlike<ROLE, float>(h, a, h->maps[j]) : launch_sweep<ROLE, false>(h, a, h->maps[j]))
    return e;
  if (!a.vmode) return 0;
  if (verify_ring())
    return rl ? launch_sweep<ROLE, true, true>(h, a, h->maps[j])
              : launch_sweep<ROLE, false, true>(h, a, h->maps[j]);
  return rl ? launch_verify<ROLE, true>(h, a) : launch_verify<ROLE, false>(h, a);
  }
}

// merge points of family j for the current state (before its sweep), on
// stream st; a.merge / a.nb point the sweep at them
template <class ST>
int launch_merge(pcb_solver* h, int j, pcb::fast::ArgsT<ST>& a, cudaStream_t st) {
  a.merge = nullptr;
  a.nb = 1;
  if (h->nbk[j] <= 1) return 0;
  const Fam& F = h->fam[j];
  const int per = pcb::fast::MWARPS * 32;
  const dim3 g((unsigned)((F.C + per - 1) / per), (unsigned)(h->nbk[j] - 1));
  int* out = h->merge.p + h->merge_off[j];
  if (fam_rowlike(F.kind))
    pcb::fast::k_merge<true, ST><<<g, per, 0, st>>>(F, a.p, a.wf, a.c, h->lbk[j], h->nbk[j],
                                                4 * h->lbk[j], out);
  else
    pcb::fast::k_merge<false, ST><<<g, per, 0, st>>>(F, a.p, a.wf, a.c, h->lbk[j], h->nbk[j],
                                                 4 * h->lbk[j], out);
  LAUNCH_CHECK(h);
  a.merge = out;
  a.nb = h->nbk[j];
  return 0;
}

template <class ST>
int launch_merge(pcb_solver* h, int j, pcb::fast::ArgsT<ST>& a) { return launch_merge(h, j, a, h->stream); }

// side stream + events for the overlapped merges (created on first use)
int ensure_side(pcb_solver* h) {
  if (h->side) return 0;
  CUDA_TRY(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&h->ev_sweeps, cudaEventDisableTiming));
  for (int j = 0; j < MAXR; ++j)
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_merge[j], cudaEventDisableTiming));
  return 0;
}

// cuTensorMapEncodeTiled from the driver (no -lcuda link needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    else
      (void)cudaGetLastError();
  }
  return fn;
}

// A row family (chain c is the node row [c*m, (c+1)*m)) that gets the row map
// of the TMA-fed sweep (k_sweep<..., RT>): full warps, and 16-B aligned row
// starts for the retire's vector stores (m % 4 == 0).  PCB_TMA=0 /
// PCB_ROW_TMA=0 keep it on per-lane cp.async.
bool row_tma_family(const Fam& F) {
  const char* env = getenv("PCB_TMA");
  if (env && env[0] == '0') return false;
  const char* renv = getenv("PCB_ROW_TMA");
  if (renv && renv[0] == '0') return false;
  if (!encode_tiled()) return false;
  return (F.kind == K_ROW2 || F.kind == K_X3) && F.zz == 0 && F.ns == 1 && F.cdiv == 1 &&
         F.clo == 0 && F.chi == F.m && F.C % 32 == 0 && F.m % 4 == 0;
}

// TMA maps for the strided families whose warps cover 32 consecutive nodes
// (cols; 3D y with D2 % 32 == 0; 3D z).  Others keep the per-lane cp.async.
// PCB_TMA=0 disables them.
template <class ST>
void build_maps_for(pcb_solver* h, ST* pbuf, double* cbuf, pcb::fast::Maps* maps) {
  constexpr CUtensorMapDataType ET =
      sizeof(ST) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  for (int j = 0; j < MAXR; ++j) maps[j] = pcb::fast::Maps{};
  const char* env = getenv("PCB_TMA");
  if (env && env[0] == '0') return;
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return;
  using pcb::fast::TP;
  for (int j = 0; j < h->r; ++j) {
    const Fam& F = h->fam[j];
    if (row_tma_family(F)) {
      pcb::fast::Maps M{};
      const cuuint32_t box2[2] = {32, (cuuint32_t)TP}, es2[2] = {1, 1};
      const cuuint64_t dp[2] = {(cuuint64_t)F.C, (cuuint64_t)F.m};
      const cuuint64_t da[2] = {(cuuint64_t)F.C, (cuuint64_t)(F.m - 1)};
      const cuuint64_t sp[1] = {(cuuint64_t)F.C * sizeof(ST)};
      CUresult r1 = fn(&M.p, ET, 2, (void*)(pbuf + (int64_t)j * h->n), dp, sp, box2, es2,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      CUresult r2 = fn(&M.a, ET, 2, (void*)FastState<ST>::wf(h, j), da, sp, box2, es2,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const cuuint64_t dc[2] = {(cuuint64_t)F.m, (cuuint64_t)F.C};
      const cuuint64_t sc[1] = {(cuuint64_t)F.m * 8};
      const cuuint32_t boxc[2] = {(cuuint32_t)TP, 32};
      CUresult r3 = fn(&M.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)cbuf, dc, sc, boxc, es2,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS) continue;
      M.tma = 1;
      M.row = 1;
      maps[j] = M;
      continue;
    }
    if (fam_rowlike(F.kind) || F.zz != 0 || F.C % 32 != 0 || F.m < 2) continue;
    bool c3;
    if (F.cdiv == 1 && F.chi == 1 && F.clo == 0)
      c3 = false;  // node = c + i * ns
    else if (F.clo == 1 && F.cdiv % 32 == 0)
      c3 = true;  // node = (c / cdiv) * chi + c % cdiv + i * ns
    else
      continue;
    pcb::fast::Maps M{};
    const cuuint32_t box2[2] = {32, (cuuint32_t)TP}, es2[2] = {1, 1};
    const cuuint64_t dp[2] = {(cuuint64_t)F.C, (cuuint64_t)F.m};
    const cuuint64_t da[2] = {(cuuint64_t)F.C, (cuuint64_t)(F.m - 1)};
    const cuuint64_t sp[1] = {(cuuint64_t)F.C * sizeof(ST)};
    CUresult r1 = fn(&M.p, ET, 2, (void*)(pbuf + (int64_t)j * h->n), dp, sp, box2, es2,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = fn(&M.a, ET, 2, (void*)FastState<ST>::wf(h, j), da, sp, box2,
                     es2, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r3;
    if (!c3) {
      const cuuint64_t dc[2] = {(cuuint64_t)F.C, (cuuint64_t)F.m};
      const cuuint64_t sc[1] = {(cuuint64_t)F.ns * 8};
      r3 = fn(&M.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)cbuf, dc, sc, box2, es2,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t dc[3] = {(cuuint64_t)F.cdiv, (cuuint64_t)F.m, (cuuint64_t)(F.C / F.cdiv)};
      const cuuint64_t sc[2] = {(cuuint64_t)F.ns * 8, (cuuint64_t)F.chi * 8};
      const cuuint32_t box3[3] = {32, (cuuint32_t)TP, 1}, es3[3] = {1, 1, 1};
      r3 = fn(&M.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)cbuf, dc, sc, box3, es3,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS) continue;
    M.tma = 1;
    M.c3 = c3 ? 1 : 0;
    maps[j] = M;
  }
}

void build_maps(pcb_solver* h) {
  if (h->precision == PCB_F64S) {
    build_maps_for(h, h->p64.p, h->cdrift.p, h->maps64);
    return;
  }
  build_maps_for(h, h->p32.p, h->cdrift.p, h->maps);
  if (h->dbuf) build_maps_for(h, h->p32b.p, h->cdriftb.p, h->maps2);
}

// step-norm partial slots of a family sweep: one per warp (and unit)
int fam_units(const pcb_solver* h, int j) {
  const int per = pcb::fast::WARPS * 32;
  return (int)((h->fam[j].C + per - 1) / per) * pcb::fast::WARPS * (h->nbk[j] > 1 ? h->nbk[j] : 1);
}

// Per family {mode, count, cool, backoff}, then {verified sweeps, repaired
// chains, scan sweeps, changed chains} (int64) per family.
constexpr int VS_FAM = 4;
constexpr int VSTATE_INTS = VS_FAM * MAXR + 8 * MAXR;
constexpr int VS_COOL0 = 64;  // plain iterations before the first verified probe

// Mode policy of the verified sweeps, once per double-buffered step (device
// side, so graph-capturable and deterministic: it depends only on integer
// counts).  Modes: 0 scan, 2 scan that writes segment hints (the iteration
// before a probe), 1 verify.  A family verifies while fewer than theta % of
// its chains needed a repair; otherwise it scans for `backoff` iterations
// (doubling, up to 256) before the next probe.
struct VModeArgs {
  int r;
  int64_t C[MAXR];  // 0: family without hints (always scans)
  int theta_pct;
};

__global__ void k_vmode(int* vs, VModeArgs va) {
  const int j = threadIdx.x;
  if (j >= va.r || va.C[j] == 0) return;
  int* f = vs + VS_FAM * j;
  const int64_t cnt = f[1];
  long long* st = reinterpret_cast<long long*>(vs + VS_FAM * MAXR) + 4 * j;
  const int mode = f[0];
  st[mode == 1 ? 0 : 2] += 1;
  st[mode == 1 ? 1 : 3] += cnt;
  if (mode == 1) {
    if (cnt * 100 >= va.C[j] * (int64_t)va.theta_pct) {
      f[3] = min(2 * f[3], 256);
      f[2] = f[3];
      f[0] = 0;
    }
  } else if (mode == 2) {
    f[0] = 1;
  } else if (--f[2] <= 0) {
    f[0] = 2;
  }
  f[1] = 0;
}

template <class T>
void swap_buf(DBuf<T>& a, DBuf<T>& b) {
  std::swap(a.p, b.p);
  std::swap(a.n, b.n);
  std::swap(a.pooled, b.pooled);
}

// after a double-buffered step the alternate buffers hold the state
void swap_state(pcb_solver* h) {
  h->par ^= 1;
  swap_buf(h->p32, h->p32b);
  swap_buf(h->cdrift, h->cdriftb);
  swap_buf(h->X32, h->X32b);
  for (int j = 0; j < MAXR; ++j) std::swap(h->maps[j], h->maps2[j]);
}

// one fused fp32 iteration over the handle's active families; partials of
// every family land in parts[], reduced in order.  flags: PCB_STEP_G_PRESET
// (G already holds other families' d: no FIRST role), PCB_STEP_NO_UPDATE (no
// LAST role: the drift/primal update happens on another handle),
// PCB_STEP_EXPORT_G (LAST stores its per-node g in G), PCB_STEP_NORM_RAW
// (store the sum of squares, not its square root).
template <class ST>
int step_fast(pcb_solver* h, double* norm_slot, int flags) {
  ST* const P = FastState<ST>::p(h);
  ST* const G = FastState<ST>::G(h);
  ST* const X = FastState<ST>::X(h);
  constexpr bool F32 = std::is_same<ST, float>::value;
  const double inv_r = 1.0 / (double)h->r, rd = (double)h->r;
  int act[MAXR], na = 0;
  for (int q = 0; q < h->r; ++q) {
    const int j = h->order[q];
    if (((h->fmask >> j) & 1u) && h->fam[j].C > 0) act[na++] = j;
  }
  const bool preset = flags & PCB_STEP_G_PRESET;
  const bool noupd = flags & PCB_STEP_NO_UPDATE;
  if (na == 1 && !preset && !noupd) CUDA_TRY(cudaMemsetAsync(G, 0, h->n * sizeof(ST), h->stream));
  // Every merge depends only on the state at the start of the step (p_j, the
  // drift c, the weights): launch them all on the side stream now, so they
  // run in the earlier sweeps' tails; sweep j waits for merge j only.
  bool side_merge[MAXR] = {};
  if (h->overlap_merges) {
    bool any = false;
    for (int q = 0; q < na; ++q) any = any || h->nbk[act[q]] > 1;
    if (any) {
      if (int e = ensure_side(h)) return e;
      if (h->sweeps_ev_ok) {  // the previous step's sweeps only
        CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_sweeps, 0));
      } else {
        CUDA_TRY(cudaEventRecord(h->ev_start, h->stream));
        CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_start, 0));
      }
      for (int q = 0; q < na; ++q) {
        const int j = act[q];
        if (h->nbk[j] <= 1) continue;
        pcb::fast::ArgsT<ST> m{h->fam[j], P + (int64_t)j * h->n, FastState<ST>::wf(h, j), h->cdrift.p};
        if (int rc = launch_merge(h, j, m, h->side)) return rc;
        CUDA_TRY(cudaEventRecord(h->ev_merge[j], h->side));
        side_merge[j] = true;
      }
    }
  }
  // double-buffered step (plain single-handle iterations): read the current
  // state, write the alternate buffers, swap at the end; families with segment
  // hints launch both the SCAN and the verified sweep (device mode word)
  const unsigned all = (1u << h->r) - 1u;
  const bool dbuf = F32 && h->dbuf && flags == 0 && (h->fmask & all) == all && na == h->r && na >= 2;
  ST* Gb[2] = {G, (ST*)h->G32b.p};
  int gcur = 0;  // Gb[gcur]: the accumulator the previous role wrote
  int64_t off = 0;
  for (int q = 0; q < na; ++q) {
    const int j = act[q];
    const Fam& F = h->fam[j];
    int role;
    if (q == na - 1 && !noupd) role = pcb::fast::LAST;
    else if (q == 0 && !preset && !(na == 1 && !noupd)) role = pcb::fast::FIRST;
    else role = pcb::fast::MID;
    pcb::fast::ArgsT<ST> a{F, P + (int64_t)j * h->n, FastState<ST>::wf(h, j), h->cdrift.p, G,
                           X, nullptr, inv_r, rd, h->parts.p + off, nullptr, 1,
                           (flags & PCB_STEP_EXPORT_G) ? 1 : 0};
    if (dbuf) {
      a.po = (ST*)h->p32b.p + (int64_t)j * h->n;
      a.co = h->cdriftb.p;
      a.Xo = (ST*)h->X32b.p;
      if (role == pcb::fast::FIRST) {  // G = d
        a.G = Gb[0];
        a.Gi = Gb[0];
        gcur = 0;
      } else if (role == pcb::fast::MID && (F.kind == K_ZZ0 || F.kind == K_ZZ1)) {
        // a zig-zag family leaves border nodes out: its G += d stays in place
        // (those nodes keep G), and it gets no hints (no verified sweep)
        a.G = Gb[gcur];
        a.Gi = Gb[gcur];
      } else if (role == pcb::fast::MID) {  // G' = G + d into the other buffer
        a.Gi = Gb[gcur];
        a.G = Gb[gcur ^ 1];
        gcur ^= 1;
      } else {  // LAST reads the final accumulator
        a.G = Gb[gcur];
        a.Gi = Gb[gcur];
      }
      if (h->sg[j].p) {
        a.sg = h->sg[j].p;
        a.vmode = h->vstate.p + VS_FAM * j;
        a.vcount = h->vstate.p + VS_FAM * j + 1;
      }
    }
    int rc = 0;
    if (side_merge[j]) {
      CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_merge[j], 0));
      a.merge = h->merge.p + h->merge_off[j];
      a.nb = h->nbk[j];
    }
    prof_begin(h, j);
    if (!side_merge[j]) rc = launch_merge(h, j, a);
    // MID / LAST of a plain single-buffer step: programmatic launch (their
    // scans read only p_j, the weights and the drift, none of which the
    // previous sweep writes; k_sweep waits before reading G / X).  Not when
    // per-family events are recorded in between or a merge ran inline.
    h->pdl_launch = h->use_pdl && flags == 0 && !dbuf && role != pcb::fast::FIRST &&
                    !h->profiling && (side_merge[j] || h->nbk[j] <= 1);
    if (!rc) {
      if (role == pcb::fast::FIRST) rc = launch_role_v<pcb::fast::FIRST, ST>(h, a, j);
      else if (role == pcb::fast::MID) rc = launch_role_v<pcb::fast::MID, ST>(h, a, j);
      else rc = launch_role_v<pcb::fast::LAST, ST>(h, a, j);
    }
    h->pdl_launch = false;
    prof_end(h);
    if (rc) return rc;
    off += fam_units(h, j);
  }
  if (h->side && h->ev_sweeps) {  // the next step's merges may start here
    CUDA_TRY(cudaEventRecord(h->ev_sweeps, h->stream));
    h->sweeps_ev_ok = true;
  }
  if (dbuf) {
    VModeArgs va{};
    va.r = h->r;
    for (int j = 0; j < h->r; ++j) va.C[j] = h->sg[j].p ? h->fam[j].C : 0;
    va.theta_pct = h->vtheta;
    k_vmode<<<1, 32, 0, h->stream>>>(h->vstate.p, va);
    LAUNCH_CHECK(h);
    swap_state(h);
  }
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, off, norm_slot,
                                            (flags & PCB_STEP_NORM_RAW) ? 0 : 1);
  LAUNCH_CHECK(h);
  return 0;
}

// x -= g; c += (x - g) / r on this handle's nodes (the pencil copy of the
// drift in a sharded run), with g exported by the slab side's LAST family
__global__ void k_apply_g(const float* g, float* X, double* cdr, int64_t n, int64_t n_own,
                          double inv_r, double rd, double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gv = (double)g[i];
    const double xn = (double)X[i] - gv;
    X[i] = (float)xn;
    const double dcv = (xn - gv) * inv_r;
    cdr[i] += dcv;
    if (i < n_own) acc += 2.0 * dcv * gv + rd * dcv * dcv;  // the LAST role's norm term
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

template <class ST>
int shadow_fast(pcb_solver* h) {
  for (int j = 0; j < h->r; ++j) {
    const Fam& F = h->fam[j];
    if (F.C == 0 || !((h->fmask >> j) & 1u)) continue;
    pcb::fast::ArgsT<ST> a{F, FastState<ST>::p(h) + (int64_t)j * h->n, FastState<ST>::wf(h, j),
                           h->cdrift.p, nullptr,
                      nullptr, h->y.p + (int64_t)j * h->n, 0.0, 0.0, h->parts.p, nullptr, 1, 0};
    if (int rc = launch_merge(h, j, a)) return rc;
    if (int rc = launch_role<pcb::fast::SHADOW, ST>(h, a, j)) return rc;
  }
  return 0;
}

// Blocks per chain for the fp32 sweep: enough (chain group x block) units to
// fill the machine ~4 times over, blocks of at least 32 positions.
int choose_split(pcb_solver* h) {
  int64_t need = 0;
  const char* env = getenv("PCB_SPLIT_TARGET");  // tuning knob (warps)
  const int64_t target = env ? atoll(env) : 4096;
  // shortest unit (positions): 16 for the fp64 split mode (its fp64 scan
  // keeps merges reliable on short windows; measured on cfg1), 32 for fp32
  const char* um = getenv("PCB_SPLIT_MIN");  // tuning knob
  const int unit_min = um ? atoi(um) : (h->precision == PCB_F64S ? 16 : 32);
  for (int j = 0; j < h->r; ++j) {
    const Fam& F = h->fam[j];
    const int64_t warps = (F.C + 31) / 32;
    int nb = 1;
    if (F.C > 0 && warps < target && F.m >= 2 * unit_min) {
      nb = (int)((target + warps - 1) / warps);
      const int maxb = F.m / unit_min;
      if (nb > maxb) nb = maxb;
      if (nb < 1) nb = 1;
    }
    int lb = (F.m + nb - 1) / nb;
    lb = (lb + 7) & ~7;
    nb = (F.m + lb - 1) / lb;
    h->nbk[j] = nb;
    h->lbk[j] = lb;
    h->merge_off[j] = need;
    if (nb > 1) need += (int64_t)nb * F.C;
  }
  if (need > 0)
    if (int e = h->merge.alloc(need)) return e;
  const char* ov = getenv("PCB_OVERLAP_MERGE");
  h->overlap_merges = !(ov && ov[0] == '0');
  const char* pd = getenv("PCB_PDL");
  h->use_pdl = !(pd && pd[0] == '0');
  return 0;
}

// Double buffers, segment hints and mode words of the verified sweeps
// (PCB_VERIFY=0 keeps the single-buffer SCAN step).  Hints only for families
// swept as whole chains (a split family keeps its merge-point units).
int reset_verify(pcb_solver* h);

int setup_verify(pcb_solver* h) {
  const char* env = getenv("PCB_VERIFY");
  h->dbuf = false;
  if ((env && env[0] == '0') || h->r < 2) return 0;
  const char* th = getenv("PCB_VERIFY_THETA");  // tuning / test knob (percent of chains)
  h->vtheta = th ? atoi(th) : 3;
  bool any = false;
  for (int j = 0; j < h->r; ++j) {
    const Fam& F = h->fam[j];
    // row families on per-lane cp.async only: there the verified sweep's
    // contiguous vector loads win; the TMA-fed scans (strided families, and
    // row families with a row map) are as fast as a verified sweep or faster
    // (cfg5 x family: 0.96 ms verified, 0.92 ms row-TMA scan), and a step
    // without verified families keeps its programmatic launches
    if (F.C == 0 || F.m < 2 || h->nbk[j] > 1 || !fam_rowlike(F.kind) || F.kind == K_ZZ0 ||
        F.kind == K_ZZ1 || F.m >= (1 << 16) || row_tma_family(F))
      continue;
    const int64_t cnt = (int64_t)((F.m + pcb::fast::TP - 1) / pcb::fast::TP) * F.C;
    if (int e = h->sg[j].alloc(cnt)) return e;
    CUDA_TRY(cudaMemset(h->sg[j].p, 0, cnt * sizeof(uint16_t)));
    any = true;
  }
  if (!any) return 0;  // nothing to verify: the single-buffer scan step
  h->dbuf = true;
  const int64_t rn = (int64_t)h->r * h->n;
  if (int e = h->p32b.alloc(rn)) return e;
  if (int e = h->cdriftb.alloc(h->n)) return e;
  if (int e = h->X32b.alloc(h->n)) return e;
  if (int e = h->G32b.alloc(h->n)) return e;
  CUDA_TRY(cudaMemset(h->p32b.p, 0, rn * sizeof(float)));
  if (int e = h->vstate.alloc(VSTATE_INTS)) return e;
  CUDA_TRY(cudaMemset(h->vstate.p, 0, VSTATE_INTS * sizeof(int)));
  return reset_verify(h);
}

// scan first after a new state (the hints describe the old one)
int reset_verify(pcb_solver* h) {
  if (!h->vstate.p) return 0;
  static const int init[VS_FAM * MAXR] = {0, 0, VS_COOL0, VS_COOL0, 0, 0, VS_COOL0, VS_COOL0,
                                          0, 0, VS_COOL0, VS_COOL0, 0, 0, VS_COOL0, VS_COOL0};
  CUDA_TRY(cudaMemcpyAsync(h->vstate.p, init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));  // (init is pageable host memory)
  return 0;
}

int parts_needed(const pcb_solver* h) {
  int64_t fam_blocks = 0;
  for (int j = 0; j < h->r; ++j) fam_blocks += fam_units(h, j) + (h->fam[j].C + FAM_BLOCK - 1) / FAM_BLOCK;
  int64_t need = fam_blocks;
  const int64_t node = (int64_t)NODE_GRID * (MAXT + 3);
  if (node > need) need = node;
  return (int)need;
}

#include "dual_schemes.cuh"

}  // namespace

#include "level_sets.cuh"

// =================================================================== C ABI

extern "C" {

const char* pcb_last_error(void) { return g_err.c_str(); }

int pcb_version(void) { return PCB_VERSION; }

__attribute__((target("popcnt")))  // hardware POPCNT (x86-64 hosts of this image)
int pcb_jaccard_packed(const uint8_t* a, const uint8_t* b, int64_t nbytes, double* out) {
  if ((!a || !b) && nbytes > 0) return fail(PCB_E_ARG, "null argument");
  if (!out || nbytes < 0) return fail(PCB_E_ARG, "bad argument");
  uint64_t inter = 0, uni = 0;
  int64_t i = 0;
  for (; i + 8 <= nbytes; i += 8) {
    uint64_t x, y;
    memcpy(&x, a + i, 8);
    memcpy(&y, b + i, 8);
    inter += (uint64_t)__builtin_popcountll(x & y);
    uni += (uint64_t)__builtin_popcountll(x | y);
  }
  for (; i < nbytes; ++i) {
    inter += (uint64_t)__builtin_popcount((unsigned)(a[i] & b[i]));
    uni += (uint64_t)__builtin_popcount((unsigned)(a[i] | b[i]));
  }
  *out = uni == 0 ? 0.0 : 1.0 - (double)inter / (double)uni;
  return 0;
}

int pcb_device_count(int* count) {
  if (!count) return fail(PCB_E_ARG, "count is null");
  CUDA_TRY(cudaGetDeviceCount(count));
  return 0;
}

}  // extern "C"

namespace {

// Weights source of a handle build: host arrays, a PCUT1B file, or the
// synthetic generator (built in HBM, generator.cuh).
struct SynthSpec {
  int nshapes = 0;
  const double* centres = nullptr;  // nshapes x ndim
  const double* radii = nullptr;
  uint64_t seed = 0;
  double lam = 1.0, sigma = 0.15, inv2s2 = 50.0, diag = 1.0;
  int integer = 0;
  // the generated box of the global grid (default: the whole handle grid);
  // dir_mask: directions generated (others zero, e.g. a pencil's non-cross ones)
  bool box = false;
  int64_t gdims[3] = {1, 1, 1}, origin[3] = {0, 0, 0}, extent[3] = {1, 1, 1};
  unsigned dir_mask = 0xfu;
};
struct WeightSource {
  const double* w = nullptr;
  const double* const* dirw = nullptr;
  int fd = -1;            // file: payload at `off` (w, then each direction array)
  int64_t off = 0;
  const SynthSpec* syn = nullptr;
  bool dev = false;       // w / dirw are device arrays on the same device (pcb_clone)
};

// the instance of a SynthSpec into h->w / h->dirw (stream 0, synchronous)
int synth_build(pcb_solver* h, const SynthSpec& S) {
  const int nd = h->D.nd;
  pcb::gen::Box B{};
  B.G = h->D;
  B.nb = 1;
  for (int a = 0; a < 3; ++a) {
    B.G.d[a] = S.box ? S.gdims[a] : h->D.d[a];
    B.o[a] = S.box ? S.origin[a] : 0;
    B.e[a] = S.box ? S.extent[a] : h->D.d[a];
    if (a < nd) B.nb *= B.e[a];
  }
  if (B.nb != h->n) return fail(PCB_E_ARG, "generated box does not match the handle's nodes");
  DBuf<pcb::gen::Shape> shapes;
  DBuf<uint8_t> mask;
  if (int e = mask.alloc(h->n)) return e;
  CUDA_TRY(cudaMemset(mask.p, 0, h->n));
  if (S.nshapes > 0) {
    std::vector<pcb::gen::Shape> hs(S.nshapes);
    for (int b = 0; b < S.nshapes; ++b) {
      for (int a = 0; a < 3; ++a) hs[b].c[a] = a < nd ? S.centres[b * nd + a] : 0.0;
      hs[b].r = S.radii[b];
    }
    if (int e = shapes.alloc(S.nshapes)) return e;
    CUDA_TRY(cudaMemcpy(shapes.p, hs.data(), hs.size() * sizeof(pcb::gen::Shape),
                        cudaMemcpyHostToDevice));
    pcb::gen::k_paint<<<S.nshapes, 256>>>(shapes.p, B, mask.p);
    LAUNCH_CHECK(h);
  }
  const int g = grid_for(h->n, 256, 148 * 16);
  pcb::gen::k_image<<<g, 256>>>(mask.p, B, S.seed, S.sigma, h->w.p);
  LAUNCH_CHECK(h);
  for (int k = 0; k < h->DG.ndir; ++k) {
    const int64_t cnt = dir_size(h, k);
    if (cnt <= 0) continue;
    if (!((S.dir_mask >> k) & 1u)) {
      CUDA_TRY(cudaMemset(h->dirw[k].p, 0, cnt * sizeof(double)));
      continue;
    }
    pcb::gen::EdgeArgs E{};
    int64_t bcnt = 1;  // the direction's edges inside the box
    for (int a = 0; a < 3; ++a) {
      E.off[a] = h->DG.off[k][a];
      if (a < nd) bcnt *= std::max<int64_t>(B.e[a] - (E.off[a] < 0 ? -E.off[a] : E.off[a]), 0);
    }
    if (bcnt != cnt) return fail(PCB_E_ARG, "generated box edges do not match direction %d", k);
    E.count = cnt;
    E.inv2s2 = S.inv2s2;
    E.scale = (h->conn == PCB_CONN_2D8 && k >= 2) ? S.diag : 1.0;
    E.lam = S.lam;
    E.integer = S.integer;
    pcb::gen::k_edges<<<grid_for(cnt, 256, 148 * 16), 256>>>(h->w.p, B, E, h->dirw[k].p);
    LAUNCH_CHECK(h);
  }
  pcb::gen::k_unaries<<<g, 256>>>(h->w.p, h->n, S.integer);
  LAUNCH_CHECK(h);
  CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

// pread `bytes` at `off` of fd into device memory through the pinned ring
// (reads of chunk i+1 overlap the copy engine's chunk i).  nonneg: the payload
// is fp64 edge weights; a negative one sets *negative (GridEnergy's
// "edge weights must be nonnegative", graph.py) and stops the upload.
cudaError_t file_h2d(void* dst, int fd, int64_t off, size_t bytes, cudaStream_t st,
                     bool nonneg = false, bool* negative = nullptr) {
  if (bytes == 0) return cudaSuccess;
  hostio::Stage& S = hostio::stage();
  std::lock_guard<std::mutex> lk(S.m);
  if (!S.init()) return cudaErrorMemoryAllocation;
  cudaEvent_t ev[hostio::SLOTS] = {};
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < hostio::SLOTS && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
  bool used[hostio::SLOTS] = {};
  size_t i = 0;
  for (size_t done = 0; done < bytes && e == cudaSuccess; done += hostio::CHUNK, ++i) {
    const int slot = (int)(i % hostio::SLOTS);
    const size_t len = bytes - done < hostio::CHUNK ? bytes - done : hostio::CHUNK;
    if (used[slot]) e = cudaEventSynchronize(ev[slot]);
    if (e != cudaSuccess) break;
    size_t got = 0;
    while (got < len) {
      const ssize_t r = pread(fd, (char*)S.slot[slot] + got, len - got, (off_t)(off + done + got));
      if (r <= 0) {
        e = cudaErrorUnknown;
        break;
      }
      got += (size_t)r;
    }
    if (e != cudaSuccess) break;
    if (nonneg) {
      const double* v = (const double*)S.slot[slot];
      bool neg = false;
      for (size_t q = 0; q < len / sizeof(double); ++q) neg |= v[q] < 0.0;
      if (neg) {
        *negative = true;
        break;
      }
    }
    e = cudaMemcpyAsync((char*)dst + done, S.slot[slot], len, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(ev[slot], st);
    used[slot] = true;
  }
  const cudaError_t e2 = cudaStreamSynchronize(st);
  for (int k = 0; k < hostio::SLOTS; ++k)
    if (ev[k]) cudaEventDestroy(ev[k]);
  return e != cudaSuccess ? e : e2;
}

int create_impl(const int64_t* dims, int ndim, int conn, int precision, const WeightSource& src,
                int device, pcb_solver** out) {
  *out = nullptr;
  if (conn < 0 || conn > 2) return fail(PCB_E_ARG, "unsupported connectivity code %d", conn);
  const int want_nd = conn == PCB_CONN_3D6 ? 3 : 2;
  if (ndim != want_nd) return fail(PCB_E_ARG, "dims rank does not match connectivity");
  if (precision != PCB_F64 && precision != PCB_F32 && precision != PCB_F64S)
    return fail(PCB_E_ARG, "unknown precision %d", precision);
  // n < 2^31 is what the sweeps' 32-bit index math relies on; checked before
  // every multiply so a product of large dims cannot wrap first
  const int64_t nmax = ((int64_t)1 << 31) - 1;
  int64_t n = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return fail(PCB_E_ARG, "dims must be positive");
    if (dims[a] > (int64_t)1 << 30) return fail(PCB_E_ARG, "dimension too large");
    if (n > nmax / dims[a]) return fail(PCB_E_ARG, "grid too large for one device");
    n *= dims[a];
  }
  pcb_solver* h = new pcb_solver();
  h->device = device;
  h->precision = precision;
  h->conn = conn;
  h->D.nd = ndim;
  h->D.conn = conn;
  for (int a = 0; a < 3; ++a) h->D.d[a] = a < ndim ? dims[a] : 1;
  h->n = n;
  int rc = 0;
  auto bail = [&](int code) {
    delete h;
    return code;
  };
  if ((rc = set_dev(h))) return bail(rc);
  // PCB_TRACE=1: phase timings of the setup on stderr (diagnostics)
  static const bool trace = getenv("PCB_TRACE") && getenv("PCB_TRACE")[0] == '1';
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    cudaDeviceSynchronize();
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[pcb_create] %-14s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  phase("set_dev");
  setup_geometry(h);
  if ((rc = h->w.alloc(n))) return bail(rc);
  int64_t foff = src.off;
  cudaError_t e = cudaSuccess;
  if (src.dev)
    e = cudaMemcpy(h->w.p, src.w, n * sizeof(double), cudaMemcpyDeviceToDevice);
  else if (!src.syn)
    e = src.fd >= 0 ? file_h2d(h->w.p, src.fd, foff, n * sizeof(double), 0)
                    : hostio::h2d(h->w.p, src.w, n * sizeof(double), 0);
  if (e != cudaSuccess) return bail(fail(PCB_E_CUDA, "upload w: %s", cudaGetErrorString(e)));
  foff += n * (int64_t)sizeof(double);
  for (int k = 0; k < h->DG.ndir; ++k) {
    const int64_t cnt = dir_size(h, k);
    if ((rc = h->dirw[k].alloc(cnt))) return bail(rc);
    if (cnt > 0 && src.dev) {
      e = cudaMemcpy(h->dirw[k].p, src.dirw[k], cnt * sizeof(double), cudaMemcpyDeviceToDevice);
      if (e != cudaSuccess)
        return bail(fail(PCB_E_CUDA, "copy weights: %s", cudaGetErrorString(e)));
    } else if (cnt > 0 && !src.syn) {
      if (src.fd >= 0) {
        bool neg = false;
        e = file_h2d(h->dirw[k].p, src.fd, foff, cnt * sizeof(double), 0, true, &neg);
        if (neg) return bail(fail(PCB_E_ARG, "edge weights must be nonnegative"));
      } else {
        if (!src.dirw[k]) return bail(fail(PCB_E_ARG, "direction %d weights are null", k));
        e = hostio::h2d(h->dirw[k].p, src.dirw[k], cnt * sizeof(double), 0);
      }
      if (e != cudaSuccess)
        return bail(fail(PCB_E_CUDA, "upload weights: %s", cudaGetErrorString(e)));
      foff += cnt * (int64_t)sizeof(double);
    }
  }
  if (src.syn)
    if ((rc = synth_build(h, *src.syn))) return bail(rc);
  phase("upload");
  const int64_t rn = (int64_t)h->r * n;
  if ((rc = h->y.alloc(rn))) return bail(rc);
  e = cudaMemset(h->y.p, 0, rn * sizeof(double));
  if (e != cudaSuccess) return bail(fail(PCB_E_CUDA, "memset: %s", cudaGetErrorString(e)));
  if (precision == PCB_F64) {
    if ((rc = h->z.alloc(rn))) return bail(rc);
    if ((rc = ensure_wf64(h))) return bail(rc);
  } else if (precision == PCB_F64S) {  // the fast path in fp64 (no verified sweeps)
    if ((rc = h->p64.alloc(rn))) return bail(rc);
    if ((rc = h->cdrift.alloc(n))) return bail(rc);
    if ((rc = h->X64.alloc(n))) return bail(rc);
    if ((rc = h->G64.alloc(n))) return bail(rc);
    if ((rc = ensure_wf64(h))) return bail(rc);
    if ((rc = choose_split(h))) return bail(rc);
    build_maps(h);
  } else {
    if ((rc = h->p32.alloc(rn))) return bail(rc);
    if ((rc = h->cdrift.alloc(n))) return bail(rc);
    if ((rc = h->X32.alloc(n))) return bail(rc);
    if ((rc = h->G32.alloc(n))) return bail(rc);
    phase("alloc");
    if ((rc = ensure_wf32(h))) return bail(rc);
    if ((rc = choose_split(h))) return bail(rc);
    phase("split");
    if ((rc = setup_verify(h))) return bail(rc);
    build_maps(h);
    phase("family weights");
  }
  if (precision == PCB_F64)  // hull spill for the exact kernels (f32 path: lazily, project_K only)
    if ((rc = ensure_spill(h))) return bail(rc);
  if ((rc = h->bits.alloc(n + 8))) return bail(rc);  // (+8: the cut kernel's word reads)
  e = cudaMemset(h->bits.p, 0, n + 8);
  if (e != cudaSuccess) return bail(fail(PCB_E_CUDA, "memset: %s", cudaGetErrorString(e)));
  if ((rc = h->xcur.alloc(n))) return bail(rc);
  if ((rc = h->parts.alloc(parts_needed(h)))) return bail(rc);
  if ((rc = h->vals.alloc(64))) return bail(rc);
  if ((rc = h->norms.alloc(2))) return bail(rc);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(PCB_E_CUDA, "setup: %s", cudaGetErrorString(e)));
  phase("rest");
  *out = h;
  return 0;
}

}  // namespace

extern "C" {

int pcb_create(const int64_t* dims, int ndim, int conn, int precision, const double* w,
               const double* const* dir_weights, int device, pcb_solver** out) {
  if (!out || !dims || !w || !dir_weights) return fail(PCB_E_ARG, "null argument");
  WeightSource src;
  src.w = w;
  src.dirw = dir_weights;
  return create_impl(dims, ndim, conn, precision, src, device, out);
}

int pcb_clone(const pcb_solver* src, int precision, pcb_solver** out) {
  if (!src || !out) return fail(PCB_E_ARG, "null argument");
  const double* dw[4] = {};
  for (int k = 0; k < src->DG.ndir; ++k) dw[k] = src->dirw[k].p;
  WeightSource ws;
  ws.w = src->w.p;
  ws.dirw = dw;
  ws.dev = true;
  int64_t dims[3];
  for (int a = 0; a < src->D.nd; ++a) dims[a] = src->D.d[a];
  if (int e = create_impl(dims, src->D.nd, src->conn, precision, ws, src->device, out)) return e;
  pcb_solver* h = *out;
  // a rescaled source keeps its lambda = 1 weights: so does the clone
  for (int k = 0; k < src->DG.ndir; ++k) {
    if (!src->dirw_base[k].p) continue;
    const int64_t cnt = dir_size(h, k);
    int e = h->dirw_base[k].alloc(cnt);
    if (!e && cudaMemcpy(h->dirw_base[k].p, src->dirw_base[k].p, cnt * sizeof(double),
                         cudaMemcpyDeviceToDevice) != cudaSuccess)
      e = fail(PCB_E_CUDA, "copy base weights");
    if (e) {
      delete h;
      *out = nullptr;
      return e;
    }
  }
  return 0;
}

int pcb_copy_state(pcb_solver* dst, const pcb_solver* src) {
  if (!dst || !src) return fail(PCB_E_ARG, "null argument");
  if (dst->n != src->n || dst->r != src->r || dst->conn != src->conn || dst->device != src->device)
    return fail(PCB_E_ARG, "handles of different instances or devices");
  const bool sf = src->precision == PCB_F32 || src->precision == PCB_F64S;
  const bool df = dst->precision == PCB_F32 || dst->precision == PCB_F64S;
  if (!sf || !df) return fail(PCB_E_ARG, "copy_state moves the fused-form state (f32 / f64s)");
  if (!src->have_state) return fail(PCB_E_STATE, "no AAR state in the source");
  if (int e = set_dev(dst)) return e;
  CUDA_TRY(cudaStreamSynchronize(src->stream));  // the source's queued work first
  const int g = grid_for(dst->n, 256, NODE_GRID);
  const FamSet fs = famset(dst);
  if (src->precision == PCB_F32 && dst->precision == PCB_F64S)
    k_copy_fast<float, double><<<g, 256, 0, dst->stream>>>(src->p32.p, src->cdrift.p, dst->p64.p,
        dst->cdrift.p, dst->X64.p, dst->w.p, dst->n, fs, dst->D);
  else if (src->precision == PCB_F32)
    k_copy_fast<float, float><<<g, 256, 0, dst->stream>>>(src->p32.p, src->cdrift.p, dst->p32.p,
        dst->cdrift.p, dst->X32.p, dst->w.p, dst->n, fs, dst->D);
  else if (dst->precision == PCB_F64S)
    k_copy_fast<double, double><<<g, 256, 0, dst->stream>>>(src->p64.p, src->cdrift.p,
        dst->p64.p, dst->cdrift.p, dst->X64.p, dst->w.p, dst->n, fs, dst->D);
  else
    k_copy_fast<double, float><<<g, 256, 0, dst->stream>>>(src->p64.p, src->cdrift.p,
        dst->p32.p, dst->cdrift.p, dst->X32.p, dst->w.p, dst->n, fs, dst->D);
  LAUNCH_CHECK(dst);
  if (dst->precision == PCB_F32)
    if (int e = reset_verify(dst)) return e;
  CUDA_TRY(cudaStreamSynchronize(dst->stream));
  dst->have_state = true;
  dst->have_shadow = false;
  dst->alg = 0;
  return 0;
}

int pcb_create_from_file(const char* path, int precision, int device, pcb_solver** out,
                         int64_t* dims_out, int* ndim_out, int* conn_out) {
  if (!path || !out) return fail(PCB_E_ARG, "null argument");
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(PCB_E_ARG, "%s: cannot open (%s)", path, strerror(errno));
  struct Closer {
    int fd;
    ~Closer() { close(fd); }
  } closer{fd};
  unsigned char head[8];
  if (pread(fd, head, 8, 0) != 8) return fail(PCB_E_ARG, "%s: truncated header", path);
  if (memcmp(head, "PCUT1B", 6) != 0) return fail(PCB_E_ARG, "%s: not a binary grid file", path);
  const int code = head[6], ndim = head[7];
  if (code > 2) return fail(PCB_E_ARG, "%s: unknown connectivity code %d", path, code);
  if (ndim != (code == PCB_CONN_3D6 ? 3 : 2))
    return fail(PCB_E_ARG, "%s: dimension count does not match connectivity", path);
  uint64_t d64[3] = {1, 1, 1};
  if (pread(fd, d64, 8 * ndim, 8) != 8 * ndim) return fail(PCB_E_ARG, "%s: truncated header", path);
  int64_t dims[3] = {1, 1, 1};
  int64_t nodes = 1;
  for (int a = 0; a < ndim; ++a) {  // little-endian u64 (x86 / Grace hosts)
    if (d64[a] < 1 || d64[a] > ((uint64_t)1 << 30)) return fail(PCB_E_ARG, "%s: bad dimension", path);
    dims[a] = (int64_t)d64[a];
    if (nodes > (((int64_t)1 << 31) - 1) / dims[a])
      return fail(PCB_E_ARG, "%s: grid too large for one device", path);
    nodes *= dims[a];  // < 2^31, so the payload count below cannot overflow
  }
  // payload size: w plus every direction array (sizes as direction_shape)
  static const int offs[3][4][3] = {{{0, 1, 0}, {1, 0, 0}, {0, 0, 0}, {0, 0, 0}},
                                    {{0, 1, 0}, {1, 0, 0}, {1, 1, 0}, {1, 1, 0}},
                                    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {0, 0, 0}}};
  const int ndir = code == 1 ? 4 : (code == 0 ? 2 : 3);
  int64_t count = nodes;
  for (int k = 0; k < ndir; ++k) {
    int64_t c = 1;
    for (int a = 0; a < ndim; ++a) {
      const int64_t len = dims[a] - offs[code][k][a];
      c *= len > 0 ? len : 0;
    }
    count += c;
  }
  struct stat st;
  if (fstat(fd, &st) != 0) return fail(PCB_E_ARG, "%s: cannot stat", path);
  const int64_t off = 8 + 8 * (int64_t)ndim;
  if ((int64_t)st.st_size != off + 8 * count) return fail(PCB_E_ARG, "%s: truncated payload", path);
  WeightSource src;
  src.fd = fd;
  src.off = off;
  if (dims_out)
    for (int a = 0; a < ndim; ++a) dims_out[a] = dims[a];
  if (ndim_out) *ndim_out = ndim;
  if (conn_out) *conn_out = code;
  return create_impl(dims, ndim, code, precision, src, device, out);
}

int pcb_create_synthetic(const int64_t* dims, int ndim, int conn, int nshapes,
                         const double* centres, const double* radii, uint64_t seed, double lam,
                         int integer, int precision, int device, pcb_solver** out) {
  if (!out || !dims || (nshapes > 0 && (!centres || !radii))) return fail(PCB_E_ARG, "null argument");
  if (nshapes < 0) return fail(PCB_E_ARG, "negative shape count");
  if (!(lam >= 0.0)) return fail(PCB_E_ARG, "scale factor must be nonnegative");
  SynthSpec S;
  S.nshapes = nshapes;
  S.centres = centres;
  S.radii = radii;
  S.seed = seed;
  S.lam = lam;
  S.integer = integer ? 1 : 0;
  S.sigma = 0.15;
  S.inv2s2 = 1.0 / (2.0 * 0.1 * 0.1);  // instances.INV2S2
  S.diag = 1.0 / sqrt(2.0);
  WeightSource src;
  src.syn = &S;
  return create_impl(dims, ndim, conn, precision, src, device, out);
}

int pcb_create_synthetic_box(const int64_t* gdims, int ndim, int conn, const int64_t* origin,
                             const int64_t* extent, const int64_t* dims, unsigned dir_mask,
                             int nshapes, const double* centres, const double* radii,
                             uint64_t seed, double lam, int integer, int precision, int device,
                             pcb_solver** out) {
  if (!out || !gdims || !origin || !extent || !dims || (nshapes > 0 && (!centres || !radii)))
    return fail(PCB_E_ARG, "null argument");
  if (ndim < 2 || ndim > 3) return fail(PCB_E_ARG, "dims rank must be 2 or 3");
  SynthSpec S;
  for (int a = 0; a < ndim; ++a) {
    if (origin[a] < 0 || extent[a] < 1 || origin[a] + extent[a] > gdims[a])
      return fail(PCB_E_ARG, "box [origin, origin + extent) outside the grid on axis %d", a);
    S.gdims[a] = gdims[a];
    S.origin[a] = origin[a];
    S.extent[a] = extent[a];
  }
  S.box = true;
  S.dir_mask = dir_mask;
  S.nshapes = nshapes;
  S.centres = centres;
  S.radii = radii;
  S.seed = seed;
  S.lam = lam;
  S.integer = integer ? 1 : 0;
  S.sigma = 0.15;
  S.inv2s2 = 1.0 / (2.0 * 0.1 * 0.1);
  S.diag = 1.0 / sqrt(2.0);
  WeightSource src;
  src.syn = &S;
  return create_impl(dims, ndim, conn, precision, src, device, out);
}

int pcb_get_instance(pcb_solver* h, double* w, double* const* dir_weights) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (int e = set_dev(h)) return e;
  if (w) CUDA_TRY(hostio::d2h(w, h->w.p, h->n * sizeof(double), h->stream));
  for (int k = 0; k < h->DG.ndir; ++k) {
    const int64_t cnt = dir_size(h, k);
    if (dir_weights && dir_weights[k] && cnt > 0)
      CUDA_TRY(hostio::d2h(dir_weights[k], h->dirw[k].p, cnt * sizeof(double), h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_debug_counters(uint64_t* out, int reset) {
  if (!out) return fail(PCB_E_ARG, "null argument");
#ifdef PCB_COUNT
  unsigned long long v[8];
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(v, pcb::fast::g_count, sizeof(v)));
  for (int i = 0; i < 8; ++i) out[i] = v[i];
  if (reset) {
    unsigned long long z[8] = {};
    CUDA_TRY(cudaMemcpyToSymbol(pcb::fast::g_count, z, sizeof(z)));
  }
#else
  unsigned long long v[8];
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(v, pcb::fast::g_rep, sizeof(v)));
  for (int i = 0; i < 8; ++i) out[i] = v[i];
  if (reset) {
    unsigned long long z[8] = {};
    CUDA_TRY(cudaMemcpyToSymbol(pcb::fast::g_rep, z, sizeof(z)));
  }
#endif
  return 0;
}

int pcb_scale_pairwise(pcb_solver* h, double factor) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!(factor >= 0.0)) return fail(PCB_E_ARG, "scale factor must be nonnegative");
  if (int e = set_dev(h)) return e;
  DirPtrs dp{};
  for (int k = 0; k < h->DG.ndir; ++k) {
    const int64_t cnt = dir_size(h, k);
    if (!h->dirw_base[k].p) {
      if (int e = h->dirw_base[k].alloc(cnt)) return e;
      if (cnt > 0)
        CUDA_TRY(cudaMemcpyAsync(h->dirw_base[k].p, h->dirw[k].p, cnt * sizeof(double),
                                 cudaMemcpyDeviceToDevice, h->stream));
    }
    if (cnt > 0) {
      k_scale<<<grid_for(cnt, 256, NODE_GRID), 256, 0, h->stream>>>(h->dirw_base[k].p,
                                                                     h->dirw[k].p, cnt, factor);
      LAUNCH_CHECK(h);
    }
    dp.p[k] = h->dirw[k].p;
  }
  // family weights of both precisions from the rescaled direction arrays
  for (int j = 0; j < h->r; ++j) {
    const Fam& F = h->fam[j];
    const int64_t cnt = F.C * (int64_t)(F.m > 1 ? F.m - 1 : 0);
    if (cnt == 0) continue;
    if (h->wf64[j].p) {
      k_build_family_weights<double><<<grid_for(cnt, 256, 148 * 16), 256, 0, h->stream>>>(
          F, h->D, dp, h->wf64[j].p);
      LAUNCH_CHECK(h);
    }
    if (h->wf32[j].p) {
      k_build_family_weights<float><<<grid_for(cnt, 256, 148 * 16), 256, 0, h->stream>>>(
          F, h->D, dp, h->wf32[j].p);
      LAUNCH_CHECK(h);
    }
  }
  h->have_shadow = false;
  h->y_valid = false;
  h->have_check = false;
  return 0;
}

int pcb_release_memory(int device) {
  if (device < 0 || device >= 64) return fail(PCB_E_ARG, "bad device %d", device);
  if (!g_pool[device]) return 0;
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaDeviceSynchronize());
  const cudaError_t e = cudaMemPoolTrimTo(g_pool[device], 0);
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(PCB_E_CUDA, "cudaMemPoolTrimTo: %s", cudaGetErrorString(e));
  return 0;
}

int pcb_destroy(pcb_solver* h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  delete h;
  return 0;
}

int pcb_shape(const pcb_solver* h, int* r, int64_t* n) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (r) *r = h->r;
  if (n) *n = h->n;
  return 0;
}

int pcb_set_stream(pcb_solver* h, uintptr_t stream) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  // buffer frees are ordered on the handle's stream: drain the old one first
  // (not while either stream is being captured into a graph: a sync would
  // invalidate the capture, and captured work is not queued work)
  if ((cudaStream_t)stream != h->stream) {
    cudaSetDevice(h->device);
    cudaStreamCaptureStatus c_old = cudaStreamCaptureStatusNone, c_new = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(h->stream, &c_old));
    CUDA_TRY(cudaStreamIsCapturing((cudaStream_t)stream, &c_new));
    if (c_old == cudaStreamCaptureStatusNone && c_new == cudaStreamCaptureStatusNone)
      CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  h->stream = (cudaStream_t)stream;
  return 0;
}

int pcb_synchronize(pcb_solver* h) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (int e = set_dev(h)) return e;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_init_cold(pcb_solver* h) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (int e = set_dev(h)) return e;
  const int g = grid_for(h->n, 256, NODE_GRID);
  if (h->precision == PCB_F64) {
    k_init_exact<<<g, 256, 0, h->stream>>>(h->z.p, h->w.p, h->n, h->r);
  } else if (h->precision == PCB_F64S) {
    k_init_fast<<<g, 256, 0, h->stream>>>(h->p64.p, h->cdrift.p, h->X64.p, h->w.p, h->n, h->r);
  } else {
    k_init_fast<<<g, 256, 0, h->stream>>>(h->p32.p, h->cdrift.p, h->X32.p, h->w.p, h->n, h->r);
    if (int e = reset_verify(h)) return e;
  }
  LAUNCH_CHECK(h);
  h->have_state = true;
  h->have_shadow = false;
  h->alg = 0;
  return 0;
}

int pcb_set_z(pcb_solver* h, const double* z) {
  if (!h || !z) return fail(PCB_E_ARG, "null argument");
  if (int e = set_dev(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  if (h->precision == PCB_F64) {
    CUDA_TRY(hostio::h2d(h->z.p, z, rn * sizeof(double), h->stream));
  } else {
    if (int e = h->tmp.alloc(rn)) return e;
    CUDA_TRY(hostio::h2d(h->tmp.p, z, rn * sizeof(double), h->stream));
    if (h->precision == PCB_F64S)
      k_set_fast<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(
          h->tmp.p, h->p64.p, h->cdrift.p, h->X64.p, h->w.p, h->n, famset(h), h->D);
    else
      k_set_fast<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(
          h->tmp.p, h->p32.p, h->cdrift.p, h->X32.p, h->w.p, h->n, famset(h), h->D);
    LAUNCH_CHECK(h);
    if (int e = reset_verify(h)) return e;
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->have_state = true;
  h->have_shadow = false;
  h->alg = 0;
  return 0;
}

int pcb_get_z(pcb_solver* h, double* z) {
  if (!h || !z) return fail(PCB_E_ARG, "null argument");
  if (!h->have_state) return fail(PCB_E_STATE, "no AAR state (call init_cold or set_z)");
  if (int e = set_dev(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  if (h->precision == PCB_F64) {
    CUDA_TRY(hostio::d2h(z, h->z.p, rn * sizeof(double), h->stream));
  } else {
    if (int e = h->tmp.alloc(rn)) return e;
    if (h->precision == PCB_F64S)
      k_get_fast<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(
          h->p64.p, h->cdrift.p, h->tmp.p, h->n, famset(h), h->D);
    else
      k_get_fast<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(
          h->p32.p, h->cdrift.p, h->tmp.p, h->n, famset(h), h->D);
    LAUNCH_CHECK(h);
    CUDA_TRY(hostio::d2h(z, h->tmp.p, rn * sizeof(double), h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_aar_run(pcb_solver* h, int64_t iters, double* step_norms) {
  return pcb_aar_step(h, iters, 0, step_norms);
}

namespace {

// one plain AAR iteration of any precision; its step norm into *slot
int one_step(pcb_solver* h, double* slot, int flags) {
  if (h->precision == PCB_F64) {
    if (int rc = sweep_exact(h, h->z.p, h->y.p)) return rc;
    return update_exact(h, slot);
  }
  if (h->precision == PCB_F64S) return step_fast<double>(h, slot, flags);
  return step_fast<float>(h, slot, flags);
}

constexpr int GRAPH_STEPS = 8;  // even: the double-buffered state returns to its parity

bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PCB_GRAPH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// PCB_GRAPH_AFTER=N overrides every handle's capture threshold (experiments)
int64_t graph_after_env() {
  static int64_t v = -2;
  if (v == -2) {
    const char* e = getenv("PCB_GRAPH_AFTER");
    v = (e && e[0]) ? (int64_t)atoll(e) : -1;
  }
  return v;
}

// GRAPH_STEPS iterations replayed from a CUDA graph captured on first use (the
// step's launches -- sweeps, merges on the side stream, reductions, mode
// words -- become one graph launch); norms land in h->gnorms.
int graph_steps(pcb_solver* h) {
  cudaGraphExec_t& ex = h->gexec[h->par];
  if (!ex) {
    if (!h->gstream) CUDA_TRY(cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
    if (!h->gnorms.p)
      if (int e = h->gnorms.alloc(GRAPH_STEPS)) return e;
    CUDA_TRY(cudaStreamSynchronize(h->stream));  // (capture runs nothing; order by sync)
    const cudaStream_t keep = h->stream;
    const int64_t launches = h->launches;
    h->stream = h->gstream;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal));
    h->sweeps_ev_ok = false;  // the graph's first step orders on its own start
    int rc = 0;
    const int par0 = h->par;
    for (int k = 0; k < GRAPH_STEPS && !rc; ++k) rc = one_step(h, h->gnorms.p + k, 0);
    const cudaError_t ce = cudaStreamEndCapture(h->gstream, &graph);
    h->stream = keep;
    // capture swapped the host-side buffer roles GRAPH_STEPS times: back to par0
    if (h->par != par0) return fail(PCB_E_STATE, "graph capture left the buffer parity");
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(PCB_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      ex = nullptr;
      return fail(PCB_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ie));
    }
    h->glaunches[h->par] = h->launches - launches;
    h->launches = launches;  // (counted per replay below)
  }
  CUDA_TRY(cudaGraphLaunch(ex, h->stream));
  h->launches += h->glaunches[h->par];
  // the replay swapped the device buffers GRAPH_STEPS times (even): parity unchanged
  return 0;
}

}  // namespace

int pcb_aar_step(pcb_solver* h, int64_t iters, int flags, double* step_norms) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (h->alg) return fail(PCB_E_STATE, "handle holds a dual-scheme state (init_cold/set_z for AAR)");
  if (flags && h->precision != PCB_F32) return fail(PCB_E_ARG, "step flags need the f32 path");
  if (iters < 0) return fail(PCB_E_ARG, "iters must be >= 0");
  if (!h->have_state) return fail(PCB_E_STATE, "no AAR state (call init_cold or set_z)");
  if (iters == 0) return 0;
  if (int e = set_dev(h)) return e;
  if ((int64_t)h->norms.n < iters)
    if (int e = h->norms.alloc(iters)) return e;
  const bool to_log = h->logging && !step_norms;
  if (to_log)
    if (int e = grow_keep(h->normlog, (size_t)(h->nlog + iters), (size_t)h->nlog, h->stream, 4096))
      return e;
  double* nout = to_log ? h->normlog.p + h->nlog : h->norms.p;
  h->sweeps_ev_ok = false;  // other work may have touched the state since the last step
  const bool use_graph = flags == 0 && !h->profiling && graphs_enabled() && h->precision != PCB_F64;
  int64_t k = 0;
  if (use_graph) {
    // eager until the handle has run graph_after plain iterations (a graph
    // that exists already is replayed at once)
    const int64_t after = graph_after_env() >= 0 ? graph_after_env() : h->graph_after;
    if (!h->gexec[h->par] && h->plain_done < after) {
      // (whole blocks of the eager part keep the double-buffered parity)
      const int64_t need = after - h->plain_done;
      const int64_t eager = std::min(iters, (need + GRAPH_STEPS - 1) / GRAPH_STEPS * GRAPH_STEPS);
      for (; k < eager; ++k)
        if (int rc = one_step(h, nout + k, flags)) return rc;
    }
    for (; k + GRAPH_STEPS <= iters; k += GRAPH_STEPS) {
      if (int rc = graph_steps(h)) return rc;
      h->sweeps_ev_ok = false;  // (recorded inside the capture, not at this replay)
      CUDA_TRY(cudaMemcpyAsync(nout + k, h->gnorms.p, GRAPH_STEPS * sizeof(double),
                               cudaMemcpyDeviceToDevice, h->stream));
    }
  }
  for (; k < iters; ++k)
    if (int rc = one_step(h, nout + k, flags)) return rc;
  if (flags == 0) h->plain_done += iters;
  if (to_log) h->nlog += iters;
  h->have_shadow = false;
  h->y_valid = false;
  if (step_norms) {
    CUDA_TRY(hostio::d2h(step_norms, h->norms.p, iters * sizeof(double), h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  return 0;
}

int pcb_shadow(pcb_solver* h, double* y_out, double* s_out) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (h->alg) return fail(PCB_E_STATE, "handle holds a dual-scheme state (init_cold/set_z for AAR)");
  if (!h->have_state) return fail(PCB_E_STATE, "no AAR state (call init_cold or set_z)");
  if (int e = set_dev(h)) return e;
  int rc;
  if (h->precision == PCB_F64) {
    if ((rc = sweep_exact(h, h->z.p, h->y.p))) return rc;
  } else if (h->precision == PCB_F64S) {
    if ((rc = shadow_fast<double>(h))) return rc;
  } else {
    if ((rc = shadow_fast<float>(h))) return rc;
  }
  h->have_shadow = true;
  h->y_valid = true;
  const int64_t rn = (int64_t)h->r * h->n;
  if (y_out)
    CUDA_TRY(hostio::d2h(y_out, h->y.p, rn * sizeof(double), h->stream));
  if (s_out) {
    k_sum_classes<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(h->y.p, h->r, h->n,
                                                                        h->xcur.p);
    LAUNCH_CHECK(h);
    CUDA_TRY(hostio::d2h(s_out, h->xcur.p, h->n * sizeof(double), h->stream));
    h->have_check = false;
  }
  if (y_out || s_out) CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_shadow_get(pcb_solver* h, double* y_out) {
  if (!h || !y_out) return fail(PCB_E_ARG, "null argument");
  if (!h->y_valid) return fail(PCB_E_STATE, "no current shadow");
  if (int e = set_dev(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  CUDA_TRY(hostio::d2h(y_out, h->y.p, rn * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_shadow_delta(pcb_solver* h, double* delta) {
  if (!h || !delta) return fail(PCB_E_ARG, "null argument");
  if (int e = set_dev(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  const bool had = h->y_valid;
  if (had) {
    if (!h->yprev.p)
      if (int e = h->yprev.alloc(rn)) return e;
    CUDA_TRY(cudaMemcpyAsync(h->yprev.p, h->y.p, rn * sizeof(double), cudaMemcpyDeviceToDevice,
                             h->stream));
  }
  if (int e = pcb_shadow(h, nullptr, nullptr)) return e;
  *delta = -1.0;
  if (had) {
    const int g = grid_for(rn, RED_BLOCK, NODE_GRID);
    k_diff_norm<<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->yprev.p, rn, h->parts.p);
    LAUNCH_CHECK(h);
    k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, h->norms.p, 1);
    LAUNCH_CHECK(h);
    CUDA_TRY(hostio::d2h(delta, h->norms.p, sizeof(double), h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  return 0;
}

int pcb_apply(pcb_solver* h, double* step_norm) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (h->alg) return fail(PCB_E_STATE, "handle holds a dual-scheme state (init_cold/set_z for AAR)");
  if (!h->have_shadow) return fail(PCB_E_STATE, "apply needs a current shadow (call pcb_shadow)");
  if (int e = set_dev(h)) return e;
  int rc;
  const bool to_log = h->logging && !step_norm;
  if (to_log)
    if (int e = grow_keep(h->normlog, (size_t)(h->nlog + 1), (size_t)h->nlog, h->stream, 4096))
      return e;
  double* nout = to_log ? h->normlog.p + h->nlog : h->norms.p;
  if (h->precision == PCB_F64) {
    if ((rc = update_exact(h, nout))) return rc;
  } else if (h->precision == PCB_F64S) {
    if ((rc = apply_fast<double>(h, nout))) return rc;
  } else {
    if ((rc = apply_fast<float>(h, nout))) return rc;
  }
  if (to_log) h->nlog += 1;
  h->have_shadow = false;
  if (step_norm) {
    CUDA_TRY(hostio::d2h(step_norm, h->norms.p, sizeof(double), h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  return 0;
}

int pcb_check(pcb_solver* h, int nthr, const double* thr, double* energy, double* gap,
              double* dual_obj) {
  if (!h || !thr) return fail(PCB_E_ARG, "null argument");
  if (nthr < 1 || nthr > MAXT) return fail(PCB_E_ARG, "1..%d thresholds supported", MAXT);
  if (!h->have_shadow) return fail(PCB_E_STATE, "check needs a current shadow (call pcb_shadow)");
  if (int e = set_dev(h)) return e;
  // thresholds travel in the tail of vals[]
  CUDA_TRY(hostio::h2d(h->vals.p + 48, thr, nthr * sizeof(double), h->stream));
  const int g = grid_for(h->n, RED_BLOCK, NODE_GRID);
  const int nv = nthr + 3;
  h->x_in_best = false;  // (writes xcur afresh)
  // kernels with the threshold count compiled in for the usual 1..4 (fewer
  // registers, full occupancy), the generic MAXT-slot kernels otherwise
  auto nodes = [&](auto tt) {
    constexpr int TT = decltype(tt)::value;
    const int64_t own = h->n_own < 0 ? h->n : h->n_own;
    if (h->r == 2)
      k_check_nodes<TT, 2><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->w.p, h->n, own, nthr,
                                                           h->vals.p + 48, h->bits.p, h->xcur.p,
                                                           h->parts.p);
    else if (h->r == 3)
      k_check_nodes<TT, 3><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->w.p, h->n, own, nthr,
                                                           h->vals.p + 48, h->bits.p, h->xcur.p,
                                                           h->parts.p);
    else
      k_check_nodes<TT, 4><<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->w.p, h->n, own, nthr,
                                                           h->vals.p + 48, h->bits.p, h->xcur.p,
                                                           h->parts.p);
  };
  switch (nthr) {
    case 1: nodes(std::integral_constant<int, 1>()); break;
    case 2: nodes(std::integral_constant<int, 2>()); break;
    case 3: nodes(std::integral_constant<int, 3>()); break;
    case 4: nodes(std::integral_constant<int, 4>()); break;
    default: nodes(std::integral_constant<int, MAXT>()); break;
  }
  LAUNCH_CHECK(h);
  k_reduce_cols<<<1, 32 * nv, 0, h->stream>>>(h->parts.p, g, nv, h->vals.p);
  LAUNCH_CHECK(h);
  DirPtrs dp{};
  for (int k = 0; k < h->DG.ndir; ++k) dp.p[k] = h->dirw[k].p;
  auto edges = [&](auto tt) {
    constexpr int TT = decltype(tt)::value;
    k_check_edges<TT><<<g, RED_BLOCK, 0, h->stream>>>(h->D, h->DG, dp, h->bits.p, nthr,
                                                      h->parts.p);
  };
  switch (nthr) {
    case 1: edges(std::integral_constant<int, 1>()); break;
    case 2: edges(std::integral_constant<int, 2>()); break;
    case 3: edges(std::integral_constant<int, 3>()); break;
    case 4: edges(std::integral_constant<int, 4>()); break;
    default: edges(std::integral_constant<int, MAXT>()); break;
  }
  LAUNCH_CHECK(h);
  k_reduce_cols<<<1, 32 * nthr, 0, h->stream>>>(h->parts.p, g, nthr, h->vals.p + 16);
  LAUNCH_CHECK(h);
  double hv[32];
  CUDA_TRY(hostio::d2h(hv, h->vals.p, 32 * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  const double dual = hv[nthr];
  for (int t = 0; t < nthr; ++t) {
    const double e = hv[16 + t] - hv[t];
    if (energy) energy[t] = e;
    if (gap) gap[t] = e - dual;
  }
  if (dual_obj) *dual_obj = 0.5 * hv[nthr + 1] - 0.5 * hv[nthr + 2];
  h->have_check = true;
  h->check_T = nthr;
  return 0;
}

int pcb_get_check(pcb_solver* h, int t, uint8_t* labels, int packed, double* x) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!h->have_check) return fail(PCB_E_STATE, "no current check");
  if (t < 0 || t >= h->check_T) return fail(PCB_E_ARG, "threshold index out of range");
  if (int e = set_dev(h)) return e;
  if (labels) {
    if (packed) {
      const int64_t nb = (h->n + 7) / 8;
      if ((int64_t)h->packed.n < nb)
        if (int e = h->packed.alloc(nb)) return e;
      k_pack<<<grid_for(nb, 256, NODE_GRID), 256, 0, h->stream>>>(h->bits.p, h->n, t, h->packed.p);
      LAUNCH_CHECK(h);
      CUDA_TRY(hostio::d2h(labels, h->packed.p, nb, h->stream));
    } else {
      if ((int64_t)h->packed.n < h->n)
        if (int e = h->packed.alloc(h->n)) return e;
      k_labels<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(h->bits.p, h->n, t,
                                                                      h->packed.p);
      LAUNCH_CHECK(h);
      CUDA_TRY(hostio::d2h(labels, h->packed.p, h->n, h->stream));
    }
  }
  if (x)
    CUDA_TRY(hostio::d2h(x, (h->x_in_best ? h->bestx : h->xcur).p, h->n * sizeof(double),
                         h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_log_start(pcb_solver* h) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  h->logging = true;
  h->nlog = 0;
  h->nlab = 0;
  return 0;
}

int pcb_log_stop(pcb_solver* h) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  h->logging = false;
  return 0;
}

int pcb_log_norms(pcb_solver* h, double* out, int64_t cap, int64_t* count) {
  if (!h || !count) return fail(PCB_E_ARG, "null argument");
  if (int e = set_dev(h)) return e;
  *count = h->nlog;
  const int64_t m = h->nlog < cap ? h->nlog : cap;
  if (m > 0) {
    if (!out) return fail(PCB_E_ARG, "null output");
    CUDA_TRY(hostio::d2h(out, h->normlog.p, (size_t)m * sizeof(double), h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_log_labels(pcb_solver* h, int t, int64_t* slot) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!h->have_check) return fail(PCB_E_STATE, "no current check");
  if (t < 0 || t >= h->check_T) return fail(PCB_E_ARG, "threshold index out of range");
  if (int e = set_dev(h)) return e;
  const int64_t nb = (h->n + 7) / 8;
  if (int e = grow_keep(h->lablog, (size_t)((h->nlab + 1) * nb), (size_t)(h->nlab * nb), h->stream,
                        (size_t)(32 * nb)))
    return e;
  k_pack<<<grid_for(nb, 256, NODE_GRID), 256, 0, h->stream>>>(h->bits.p, h->n, t,
                                                              h->lablog.p + h->nlab * nb);
  LAUNCH_CHECK(h);
  if (slot) *slot = h->nlab;
  h->nlab += 1;
  return 0;
}

int pcb_log_label_get(pcb_solver* h, int64_t slot, uint8_t* packed) {
  if (!h || !packed) return fail(PCB_E_ARG, "null argument");
  if (slot < 0 || slot >= h->nlab) return fail(PCB_E_ARG, "label slot out of range");
  if (int e = set_dev(h)) return e;
  const int64_t nb = (h->n + 7) / 8;
  CUDA_TRY(hostio::d2h(packed, h->lablog.p + slot * nb, (size_t)nb, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_log_jaccard(pcb_solver* h, const uint8_t* ref_packed, double* out, int64_t cap) {
  if (!h || !ref_packed) return fail(PCB_E_ARG, "null argument");
  if (cap < h->nlab) return fail(PCB_E_ARG, "output holds %lld of %lld slots", (long long)cap,
                                 (long long)h->nlab);
  if (h->nlab == 0) return 0;
  if (!out) return fail(PCB_E_ARG, "null output");
  if (int e = set_dev(h)) return e;
  const int64_t nb = (h->n + 7) / 8;
  if ((int64_t)h->packed.n < nb)
    if (int e = h->packed.alloc(nb)) return e;
  if ((int64_t)h->parts.n < h->nlab)
    if (int e = h->parts.alloc(h->nlab)) return e;
  CUDA_TRY(hostio::h2d(h->packed.p, ref_packed, (size_t)nb, h->stream));
  if ((int64_t)h->jacc.n < 2 * h->nlab)
    if (int e = h->jacc.alloc(2 * h->nlab)) return e;
  CUDA_TRY(cudaMemsetAsync(h->jacc.p, 0, 2 * h->nlab * sizeof(unsigned long long), h->stream));
  // chunks of about 64 KB per block, at most 65535 labelings per launch row
  const unsigned chunks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(256, nb >> 16));
  for (int64_t l0 = 0; l0 < h->nlab; l0 += 65535) {
    const unsigned rows = (unsigned)std::min<int64_t>(65535, h->nlab - l0);
    k_log_jaccard_part<<<dim3(chunks, rows), 256, 0, h->stream>>>(
        h->lablog.p + l0 * nb, h->packed.p, nb, h->jacc.p + 2 * l0);
    LAUNCH_CHECK(h);
  }
  k_log_jaccard_fin<<<grid_for(h->nlab, 256, 64), 256, 0, h->stream>>>(h->jacc.p, h->nlab,
                                                                         h->parts.p);
  LAUNCH_CHECK(h);
  CUDA_TRY(hostio::d2h(out, h->parts.p, (size_t)h->nlab * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_keep_best(pcb_solver* h, int t) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!h->have_check) return fail(PCB_E_STATE, "no current check");
  if (t < 0 || t >= h->check_T) return fail(PCB_E_ARG, "threshold index out of range");
  if (int e = set_dev(h)) return e;
  if (!h->bestlab.p)
    if (int e = h->bestlab.alloc(h->n)) return e;
  if (!h->bestx.p)
    if (int e = h->bestx.alloc(h->n)) return e;
  k_labels<<<grid_for(h->n, 256, NODE_GRID), 256, 0, h->stream>>>(h->bits.p, h->n, t,
                                                                  h->bestlab.p);
  LAUNCH_CHECK(h);
  // the check's x becomes the best one by a buffer swap (the next check
  // rewrites xcur); until then the current x is read from bestx
  if (!h->x_in_best) {
    swap_buf(h->xcur, h->bestx);
    h->x_in_best = true;
  }
  h->have_best = true;
  return 0;
}

int pcb_get_best(pcb_solver* h, uint8_t* labels, double* x) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!h->have_best) return fail(PCB_E_STATE, "no best iterate kept");
  if (int e = set_dev(h)) return e;
  if (labels)
    CUDA_TRY(hostio::d2h(labels, h->bestlab.p, h->n, h->stream));
  if (x)
    CUDA_TRY(hostio::d2h(x, h->bestx.p, h->n * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_dual_init(pcb_solver* h, int alg, const double* y0) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (alg != PCB_ALG_BCD && alg != PCB_ALG_AP && alg != PCB_ALG_FISTA)
    return fail(PCB_E_ARG, "unknown dual scheme %d", alg);
  if (h->precision != PCB_F64) return fail(PCB_E_ARG, "dual schemes run on fp64 handles");
  if (int e = set_dev(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  if (y0)
    CUDA_TRY(hostio::h2d(h->y.p, y0, rn * sizeof(double), h->stream));
  else
    CUDA_TRY(cudaMemsetAsync(h->y.p, 0, rn * sizeof(double), h->stream));
  if (alg == PCB_ALG_FISTA)  // v = y.copy()
    CUDA_TRY(cudaMemcpyAsync(h->z.p, h->y.p, rn * sizeof(double), cudaMemcpyDeviceToDevice,
                             h->stream));
  const size_t need = (size_t)(alg == PCB_ALG_BCD ? 3 * h->n : 2 * rn);
  if (h->tmp.n < need)
    if (int e = h->tmp.alloc(need)) return e;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->alg = alg;
  h->fista_t = 1.0;
  h->have_state = true;
  h->have_shadow = true;  // y is the iterate pcb_check certifies
  h->y_valid = true;
  h->have_check = false;
  return 0;
}

int pcb_dual_run(pcb_solver* h, int64_t iters, double* monitor, double* stop) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (!h->alg) return fail(PCB_E_STATE, "no dual scheme state (call pcb_dual_init)");
  if (iters < 0) return fail(PCB_E_ARG, "iters must be >= 0");
  if (iters == 0) return 0;
  if (int e = set_dev(h)) return e;
  if ((int64_t)h->norms.n < 2 * iters)
    if (int e = h->norms.alloc(2 * iters)) return e;
  const bool want_stop = stop != nullptr;
  if (h->alg == PCB_ALG_AP && want_stop && !h->yprev.p)
    if (int e = h->yprev.alloc((size_t)h->r * h->n)) return e;
  for (int64_t k = 0; k < iters; ++k) {
    double* mon = h->norms.p + k;
    double* stp = h->norms.p + iters + k;
    int rc = 0;
    if (h->alg == PCB_ALG_BCD)
      rc = bcd_sweep(h, mon, stp);
    else if (h->alg == PCB_ALG_AP)
      rc = ap_step(h, mon, stp, want_stop);
    else
      rc = fista_step(h, mon, stp);
    if (rc) return rc;
  }
  h->have_shadow = true;
  h->y_valid = true;
  h->have_check = false;
  if (monitor)
    CUDA_TRY(hostio::d2h(monitor, h->norms.p, iters * sizeof(double), h->stream));
  if (stop)
    CUDA_TRY(hostio::d2h(stop, h->norms.p + iters, iters * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_level_set(pcb_solver* h, const double* x, double* u, double* energy) {
  if (!h || !u) return fail(PCB_E_ARG, "null argument");
  if (!x && !h->have_check) return fail(PCB_E_STATE, "no current check (pass x or call pcb_check)");
  if (h->n >= ((int64_t)1 << 31) - 2) return fail(PCB_E_ARG, "level sets: n must be < 2^31");
  if (int e = set_dev(h)) return e;
  namespace L = pcb::levels;
  const int64_t n = h->n;
  const int ni = (int)n;
  cudaStream_t st = h->stream;
  DBuf<double> xin, xs, ws, wp, diff, cutp, E, out;
  DBuf<int> idx0, idx, flag, rs, rank_of;
  DBuf<int64_t> last_of;
  DBuf<L::ArgMin> parts;
  DBuf<unsigned char> tmp;
  const double* xd = (h->x_in_best ? h->bestx : h->xcur).p;
  if (x) {
    if (int e = xin.alloc(n)) return e;
    CUDA_TRY(hostio::h2d(xin.p, x, n * sizeof(double), st));
    xd = xin.p;
  }
  if (int e = xs.alloc(n)) return e;
  if (int e = idx0.alloc(n)) return e;
  if (int e = idx.alloc(n)) return e;
  const int g = grid_for(n, 256, NODE_GRID);
  L::k_iota<<<g, 256, 0, st>>>(idx0.p, n);
  LAUNCH_CHECK(h);
  size_t need = 0, b2 = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, xd, xs.p, idx0.p, idx.p, ni, 0, 64, st));
  CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, b2, xs.p, ws.p, ni, st));
  need = need > b2 ? need : b2;
  if (int e = tmp.alloc(need)) return e;
  size_t bytes = need;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, xd, xs.p, idx0.p, idx.p, ni, 0, 64, st));
  idx0.free();
  if (int e = flag.alloc(n)) return e;
  if (int e = rs.alloc(n)) return e;
  L::k_flags<<<g, 256, 0, st>>>(xs.p, n, flag.p);
  LAUNCH_CHECK(h);
  bytes = need;
  CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp.p, bytes, flag.p, rs.p, ni, st));
  flag.free();
  int K = 0;
  CUDA_TRY(hostio::d2h(&K, rs.p + (n - 1), sizeof(int), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (int e = rank_of.alloc(n)) return e;
  if (int e = ws.alloc(n)) return e;
  if (int e = last_of.alloc((size_t)K + 1)) return e;
  L::k_scatter_ranks<<<g, 256, 0, st>>>(rs.p, idx.p, h->w.p, n, rank_of.p, ws.p, last_of.p);
  LAUNCH_CHECK(h);
  if (int e = diff.alloc((size_t)K + 2)) return e;
  CUDA_TRY(cudaMemsetAsync(diff.p, 0, ((size_t)K + 2) * sizeof(double), st));
  DirPtrs dp{};
  for (int k = 0; k < h->DG.ndir; ++k) dp.p[k] = h->dirw[k].p;
  L::k_cut_diff<<<g, 256, 0, st>>>(h->D, h->DG, dp, rank_of.p, diff.p);
  LAUNCH_CHECK(h);
  if (int e = cutp.alloc((size_t)K + 1)) return e;
  if (int e = wp.alloc(n)) return e;
  bytes = need;
  CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp.p, bytes, diff.p, cutp.p, K + 1, st));
  bytes = need;
  CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp.p, bytes, ws.p, wp.p, ni, st));
  if (int e = E.alloc((size_t)K + 1)) return e;
  L::k_energies<<<grid_for(K + 1, 256, NODE_GRID), 256, 0, st>>>(cutp.p, wp.p, last_of.p, K, n,
                                                                 E.p);
  LAUNCH_CHECK(h);
  constexpr int AB = 256;
  const int ga = grid_for(K + 1, AB, 148 * 2);
  if (int e = parts.alloc(ga)) return e;
  if (int e = out.alloc(3)) return e;
  L::k_argmin<<<ga, AB, 0, st>>>(E.p, K + 1, parts.p);
  LAUNCH_CHECK(h);
  L::k_argmin_final<<<1, 1, 0, st>>>(parts.p, ga, xs.p, last_of.p, out.p);
  LAUNCH_CHECK(h);
  double hv[3];
  CUDA_TRY(hostio::d2h(hv, out.p, sizeof(hv), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *u = hv[0];
  if (energy) *energy = hv[1];
  return 0;
}

int pcb_project_K(pcb_solver* h, const double* v, double* out) {
  if (!h || !v || !out) return fail(PCB_E_ARG, "null argument");
  if (int e = set_dev(h)) return e;
  if (int e = ensure_wf64(h)) return e;
  if (int e = ensure_spill(h)) return e;
  const int64_t rn = (int64_t)h->r * h->n;
  if ((int64_t)h->tmp.n < 2 * rn)
    if (int e = h->tmp.alloc(2 * rn)) return e;
  double* src = h->tmp.p;
  double* dst = h->tmp.p + rn;
  CUDA_TRY(hostio::h2d(src, v, rn * sizeof(double), h->stream));
  CUDA_TRY(cudaMemsetAsync(dst, 0, rn * sizeof(double), h->stream));
  if (int e = sweep_exact(h, src, dst)) return e;
  CUDA_TRY(hostio::d2h(out, dst, rn * sizeof(double), h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int pcb_set_family_mask(pcb_solver* h, unsigned mask) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if ((mask & ((1u << h->r) - 1u)) == 0) return fail(PCB_E_ARG, "empty family mask");
  h->fmask = mask & ((1u << h->r) - 1u);
  return 0;
}

int pcb_apply_g(pcb_solver* h, uintptr_t g_dev) {
  if (!h || !g_dev) return fail(PCB_E_ARG, "null argument");
  if (h->precision != PCB_F32) return fail(PCB_E_ARG, "apply_g needs the f32 path");
  if (int e = set_dev(h)) return e;
  const int g = grid_for(h->n, 256, NODE_GRID);
  k_apply_g<<<g, 256, 0, h->stream>>>(reinterpret_cast<const float*>(g_dev), h->X32.p,
                                      h->cdrift.p, h->n, h->n_own < 0 ? h->n : h->n_own,
                                      1.0 / (double)h->r, (double)h->r, h->parts.p);
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, h->norms.p + 1, 0);
  LAUNCH_CHECK(h);
  return 0;
}

// Slab side of a sharded iteration, fused (distributed.py overlapped
// schedule): g = G + d_z (the cross family's d received in the pencil ->
// slab exchange, layout [P][dz][cp]), the drift / primal update x -= g,
// c += (x - g) / r, and the new drift straight into the slab -> pencil send
// buffer (same layout, which is the pencils' node order) -- one pass instead
// of a transposed add, a transposed copy and apply_g, and no update pass on
// the pencils (they receive their drift).
__global__ void k_apply_g_xchg(const float* __restrict__ G, const float* __restrict__ recv,
                               double* __restrict__ send, float* __restrict__ X,
                               double* __restrict__ cdr, int ns, int plane, int dz, int cp,
                               double inv_r, double rd, double* parts) {
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
    const int zr = i / plane, col = i - zr * plane;
    const int q = col / cp, cc = col - q * cp;
    const int t = (q * dz + zr) * cp + cc;
    const float g32 = G[i] + recv[t];
    const double gv = (double)g32;
    const double xn = (double)X[i] - gv;
    X[i] = (float)xn;
    const double dcv = (xn - gv) * inv_r;
    const double cn = cdr[i] + dcv;
    cdr[i] = cn;
    send[t] = cn;  // the pencils take the new drift as it is: no update pass there
    acc += 2.0 * dcv * gv + rd * dcv * dcv;  // the LAST role's norm term
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

int pcb_apply_g_exchange(pcb_solver* h, uintptr_t recv_dev, uintptr_t send_dev, int P, int dz,
                         int cp) {
  if (!h || !recv_dev || !send_dev) return fail(PCB_E_ARG, "null argument");
  if (h->precision != PCB_F32) return fail(PCB_E_ARG, "apply_g needs the f32 path");
  if (h->n_own >= 0 && h->n_own != h->n) return fail(PCB_E_ARG, "halo slabs use pcb_apply_g");
  if (P < 1 || dz < 1 || cp < 1 || (int64_t)P * cp * dz != h->n)
    return fail(PCB_E_ARG, "exchange layout does not match the handle");
  if (int e = set_dev(h)) return e;
  const int g = grid_for(h->n, 256, NODE_GRID);
  k_apply_g_xchg<<<g, 256, 0, h->stream>>>(h->G32.p, reinterpret_cast<const float*>(recv_dev),
                                           reinterpret_cast<double*>(send_dev), h->X32.p,
                                           h->cdrift.p, (int)h->n, P * cp, dz, cp,
                                           1.0 / (double)h->r, (double)h->r, h->parts.p);
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, h->norms.p + 1, 0);
  LAUNCH_CHECK(h);
  return 0;
}

int pcb_set_owned(pcb_solver* h, int64_t n_own) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (n_own < 0 || n_own > h->n) return fail(PCB_E_ARG, "owned node count %lld out of [0, %lld]",
                                             (long long)n_own, (long long)h->n);
  h->n_own = n_own == h->n ? -1 : n_own;
  h->have_check = false;
  return 0;
}

int pcb_device_buffer(pcb_solver* h, int which, uintptr_t* ptr, int64_t* count) {
  if (!h || !ptr || !count) return fail(PCB_E_ARG, "null argument");
  switch (which) {
    case PCB_BUF_G: *ptr = (uintptr_t)h->G32.p; *count = h->G32.p ? h->n : 0; break;
    case PCB_BUF_X: *ptr = (uintptr_t)h->X32.p; *count = h->X32.p ? h->n : 0; break;
    case PCB_BUF_C: *ptr = (uintptr_t)h->cdrift.p; *count = h->cdrift.p ? h->n : 0; break;
    case PCB_BUF_Y: *ptr = (uintptr_t)h->y.p; *count = (int64_t)h->r * h->n; break;
    case PCB_BUF_NORMS: *ptr = (uintptr_t)h->norms.p; *count = (int64_t)h->norms.n; break;
    case PCB_BUF_P: *ptr = (uintptr_t)h->p32.p; *count = h->p32.p ? (int64_t)h->r * h->n : 0; break;
    case PCB_BUF_BITS: *ptr = (uintptr_t)h->bits.p; *count = h->bits.p ? h->n : 0; break;
    default: return fail(PCB_E_ARG, "unknown buffer id %d", which);
  }
  if (!*ptr) return fail(PCB_E_STATE, "buffer %d not allocated for this precision", which);
  return 0;
}

int pcb_verify_stats(pcb_solver* h, int* modes, int64_t* sweeps, int64_t* repaired,
                     int64_t* scans, int64_t* changed) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (int e = set_dev(h)) return e;
  int v[VSTATE_INTS] = {};
  if (h->vstate.p) {
    CUDA_TRY(cudaMemcpyAsync(v, h->vstate.p, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  long long st[4 * MAXR];
  memcpy(st, v + VS_FAM * MAXR, sizeof(st));
  for (int j = 0; j < h->r; ++j) {
    if (modes) modes[j] = h->sg[j].p ? v[VS_FAM * j] : -1;
    if (sweeps) sweeps[j] = st[4 * j];
    if (repaired) repaired[j] = st[4 * j + 1];
    if (scans) scans[j] = st[4 * j + 2];
    if (changed) changed[j] = st[4 * j + 3];
  }
  return 0;
}

int pcb_set_graph_after(pcb_solver* h, int64_t iters) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  if (iters < 0) return fail(PCB_E_ARG, "iters must be >= 0");
  h->graph_after = iters;
  return 0;
}

int pcb_set_profiling(pcb_solver* h, int on) {
  if (!h) return fail(PCB_E_ARG, "null handle");
  h->profiling = on != 0;
  h->ev_used = 0;
  h->ev_fam.clear();
  return 0;
}

int pcb_profile_read(pcb_solver* h, double* ms, int64_t* launches) {
  if (!h || !ms || !launches) return fail(PCB_E_ARG, "null argument");
  if (int e = set_dev(h)) return e;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int j = 0; j < h->r; ++j) {
    ms[j] = 0.0;
    launches[j] = 0;
  }
  for (size_t q = 0; q < h->ev_fam.size(); ++q) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, h->ev_pool[2 * q], h->ev_pool[2 * q + 1]));
    ms[h->ev_fam[q]] += (double)t;
    launches[h->ev_fam[q]] += 1;
  }
  h->ev_used = 0;
  h->ev_fam.clear();
  return 0;
}

int64_t pcb_launch_count(const pcb_solver* h) { return h ? h->launches : 0; }

void pcb_reset_launch_count(pcb_solver* h) {
  if (h) h->launches = 0;
}

// ----------------------------------------------------------------- operator level

int pcb_project_L(const double* w, const int64_t* degree, const uint8_t* support, int r, int64_t n,
                  const double* v, double* out, int device) {
  if (!w || !degree || !support || !v || !out) return fail(PCB_E_ARG, "null argument");
  if (r < 1 || n < 1) return fail(PCB_E_ARG, "empty decomposition");
  CUDA_TRY(cudaSetDevice(device));
  const int64_t rn = (int64_t)r * n;
  DBuf<double> d_w, d_v, d_out;
  DBuf<int64_t> d_deg;
  DBuf<uint8_t> d_sup;
  DBuf<int> d_bad;
  if (int e = d_w.alloc(n)) return e;
  if (int e = d_v.alloc(rn)) return e;
  if (int e = d_out.alloc(rn)) return e;
  if (int e = d_deg.alloc(n)) return e;
  if (int e = d_sup.alloc(rn)) return e;
  if (int e = d_bad.alloc(1)) return e;
  CUDA_TRY(hostio::h2d(d_w.p, w, n * sizeof(double), 0));
  CUDA_TRY(hostio::h2d(d_v.p, v, rn * sizeof(double), 0));
  CUDA_TRY(hostio::h2d(d_deg.p, degree, n * sizeof(int64_t), 0));
  CUDA_TRY(hostio::h2d(d_sup.p, support, rn, 0));
  CUDA_TRY(cudaMemset(d_bad.p, 0, sizeof(int)));
  k_project_L<<<grid_for(n, 256, NODE_GRID), 256>>>(d_w.p, d_deg.p, d_sup.p, r, n, d_v.p, d_out.p,
                                                    d_bad.p);
  LAUNCH_CHECK((pcb_solver*)nullptr);
  int bad = 0;
  CUDA_TRY(hostio::d2h(&bad, d_bad.p, sizeof(int), 0));
  if (bad) return fail(PCB_E_ARG, "w has mass on coordinates covered by no class");
  CUDA_TRY(hostio::d2h(out, d_out.p, rn * sizeof(double), 0));
  return 0;
}

static int csr_spill(int64_t nch, const int64_t* lens_host, DBuf<int64_t>& soff, DBuf<int>& cx,
                     DBuf<double>& cy, DBuf<int>& fx, DBuf<double>& fy) {
  std::vector<int64_t> off(nch > 0 ? nch : 1);
  int64_t tot = 0;
  for (int64_t c = 0; c < nch; ++c) {
    off[c] = tot;
    const int64_t need = lens_host[c] + 1 - HC;
    tot += need > 0 ? need : 0;
  }
  if (tot == 0) tot = 1;
  if (int e = soff.alloc(off.size())) return e;
  CUDA_TRY(hostio::h2d(soff.p, off.data(), off.size() * sizeof(int64_t), 0));
  if (int e = cx.alloc(tot)) return e;
  if (int e = fx.alloc(tot)) return e;
  if (int e = cy.alloc(tot)) return e;
  if (int e = fy.alloc(tot)) return e;
  return 0;
}

int pcb_prox_chains(const int64_t* node_idx, const int64_t* chain_ptr, const double* edge_w,
                    int64_t c_lo, int64_t c_hi, int64_t n_nodes, int64_t n_idx, int64_t n_edges,
                    const double* v, double* out, int as_projection, int device) {
  if (!node_idx || !chain_ptr || !v || !out) return fail(PCB_E_ARG, "null argument");
  if (c_lo < 0 || c_hi < c_lo) return fail(PCB_E_ARG, "bad chain range");
  if (c_hi == c_lo) return 0;
  CUDA_TRY(cudaSetDevice(device));
  const int64_t nch = c_hi - c_lo;
  std::vector<int64_t> lens(nch);
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t m = chain_ptr[c_lo + c + 1] - chain_ptr[c_lo + c];
    if (m < 0 || chain_ptr[c_lo + c + 1] > n_idx)
      return fail(PCB_E_ARG, "chain_ptr out of range");
    lens[c] = m;
  }
  DBuf<int64_t> d_idx, d_ptr, soff;
  DBuf<double> d_ew, d_v, d_out, cy, fy;
  DBuf<int> cx, fx;
  if (int e = d_idx.alloc(n_idx)) return e;
  if (int e = d_ptr.alloc(c_hi + 1)) return e;
  if (int e = d_ew.alloc(n_edges)) return e;
  if (int e = d_v.alloc(n_nodes)) return e;
  if (int e = d_out.alloc(n_nodes)) return e;
  CUDA_TRY(hostio::h2d(d_idx.p, node_idx, n_idx * sizeof(int64_t), 0));
  CUDA_TRY(hostio::h2d(d_ptr.p, chain_ptr, (c_hi + 1) * sizeof(int64_t), 0));
  if (n_edges > 0 && edge_w)
    CUDA_TRY(hostio::h2d(d_ew.p, edge_w, n_edges * sizeof(double), 0));
  CUDA_TRY(hostio::h2d(d_v.p, v, n_nodes * sizeof(double), 0));
  // out is updated only on chain nodes: start from the caller's contents
  CUDA_TRY(hostio::h2d(d_out.p, out, n_nodes * sizeof(double), 0));
  if (int e = csr_spill(nch, lens.data(), soff, cx, cy, fx, fy)) return e;
  Spill sp{cx.p, cy.p, fx.p, fy.p};
  const int g = (int)((nch + FAM_BLOCK - 1) / FAM_BLOCK);
  k_prox_csr<<<g, FAM_BLOCK>>>(d_idx.p, d_ptr.p, d_ew.p, c_lo, c_hi, d_v.p, d_out.p,
                               as_projection ? 1 : 0, sp, soff.p);
  LAUNCH_CHECK((pcb_solver*)nullptr);
  CUDA_TRY(hostio::d2h(out, d_out.p, n_nodes * sizeof(double), 0));
  return 0;
}

int pcb_tv1d_prox_batch(const double* s, const double* a, const int64_t* ptr, int64_t nchains,
                        double* x, int device) {
  if (!s || !ptr || !x) return fail(PCB_E_ARG, "null argument");
  if (nchains <= 0) return 0;
  CUDA_TRY(cudaSetDevice(device));
  std::vector<int64_t> lens(nchains);
  const int64_t total = ptr[nchains];
  for (int64_t c = 0; c < nchains; ++c) {
    lens[c] = ptr[c + 1] - ptr[c];
    if (lens[c] < 1) return fail(PCB_E_ARG, "empty signal in batch");
  }
  const int64_t nedge = total - nchains;
  DBuf<int64_t> d_ptr, soff;
  DBuf<double> d_s, d_a, d_x, cy, fy;
  DBuf<int> cx, fx;
  if (int e = d_ptr.alloc(nchains + 1)) return e;
  if (int e = d_s.alloc(total)) return e;
  if (int e = d_a.alloc(nedge)) return e;
  if (int e = d_x.alloc(total)) return e;
  CUDA_TRY(hostio::h2d(d_ptr.p, ptr, (nchains + 1) * sizeof(int64_t), 0));
  CUDA_TRY(hostio::h2d(d_s.p, s, total * sizeof(double), 0));
  if (nedge > 0 && a) CUDA_TRY(hostio::h2d(d_a.p, a, nedge * sizeof(double), 0));
  if (int e = csr_spill(nchains, lens.data(), soff, cx, cy, fx, fy)) return e;
  Spill sp{cx.p, cy.p, fx.p, fy.p};
  const int g = (int)((nchains + FAM_BLOCK - 1) / FAM_BLOCK);
  k_tv1d<<<g, FAM_BLOCK>>>(d_s.p, d_a.p, d_ptr.p, nchains, d_x.p, sp, soff.p);
  LAUNCH_CHECK((pcb_solver*)nullptr);
  CUDA_TRY(hostio::d2h(x, d_x.p, total * sizeof(double), 0));
  return 0;
}

}  // extern "C"
