// fast_sweep.cuh -- staged warp kernel for the fp32-state AAR sweep (PCB_F32).
//
// One warp owns 32 chains of one family (lane l <-> chain c0 + l).  Chain data
// streams through a per-warp shared-memory ring of RL positions (NT tiles of TP
// positions) filled with cp.async (LDGSTS) a few tiles ahead of the scan:
//
//   mode A (lane = chain, one instruction per position): family-owned arrays
//          (p_j, weights, both chain-interleaved [pos][C]) and, for families
//          whose chains are strided in memory (cols, y, z), the shared node
//          arrays c, G, X -- 128-byte coalesced;
//   mode B (lanes along positions, TP lanes per chain): shared node arrays of
//          row-like families (rows, 3D x, 2D-8 zig-zags), so those reads are
//          coalesced along the rows instead of 32-way strided.
//
// Ring layout [lane][RL] with the slot XOR-swizzled by the lane id: both load
// modes and the lockstep retire loops are bank-conflict free, and per-lane
// reads at divergent positions spread over banks.
//
// Each lane runs a stackless taut string: only the minimum-slope ceiling
// point and maximum-slope floor point from the anchor are kept (the bottom
// entries of the reference's hull stacks, _kernels.py:47-95 -- the only hull
// entries its cone tests read).  A bend emits the segment with value
// (y_bend - y_anchor)/len, i.e. the string's slope, which equals the
// reference's (sum + tube offsets)/len.  The scan pauses when it needs a
// position the ring does not hold yet; emitted positions are updated in the
// ring and written back coalesced when their tile retires.  A lane whose
// anchor lags behind the ring reads/writes those positions directly in global
// memory (tile retirement is masked by each lane's emitted frontier), so a
// long segment never blocks the warp.
#pragma once

namespace pcb {
namespace fast {

constexpr int TP = 8;          // positions per tile
constexpr int NT = 4;          // tiles in the ring
constexpr int RL = TP * NT;    // ring length (positions); must be 32 for the swizzle
constexpr int WARPS = 4;       // warps per block
static_assert(RL == 32, "swizzle assumes a 32-position ring");
static_assert(TP == 8, "mode-B lane mapping assumes 8-position tiles");

enum Role { FIRST = 0, MID = 1, LAST = 2, SHADOW = 3 };

struct Args {
  Fam F;
  float* p;         // family state, interleaved [pos][C]
  const float* wf;  // family weights, interleaved [pos][C]
  double* c;        // drift (natural node layout)
  float* G;         // accumulator of p_new - p_old over families (natural)
  float* X;         // primal x = w - sum_j p_j (natural)
  double* y;        // SHADOW output (natural)
  double inv_r, rd;
  double* parts;    // per-block monitor partials
};

__device__ __forceinline__ void cp4(void* dst, const void* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp8(void* dst, const void* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait(int pending) {
  // pending = groups allowed to stay in flight (0..NT-1)
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    default: asm volatile("cp.async.wait_group 3;\n" ::); break;
  }
}

// ring index of (lane row l, position pos)
__device__ __forceinline__ int rix(int l, int pos) { return (l << 5) | ((pos & (RL - 1)) ^ l); }

template <int ROLE>
struct RingPtrs {
  double* rc;
  float* rp;
  float* ra;
  float* rG;
  float* rX;
};

template <int ROLE>
__device__ __forceinline__ constexpr int ring_bytes_per_warp() {
  return 32 * RL * (8 + 4 + 4 + ((ROLE == MID || ROLE == LAST) ? 4 : 0) + (ROLE == LAST ? 4 : 0));
}
template <int ROLE>
constexpr int ring_bytes_host() {
  return 32 * RL * (8 + 4 + 4 + ((ROLE == MID || ROLE == LAST) ? 4 : 0) + (ROLE == LAST ? 4 : 0));
}

template <int ROLE, bool ROWLIKE>
__global__ void __launch_bounds__(WARPS * 32) k_sweep(Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Fam F = A.F;
  const int64_t c0 = ((int64_t)blockIdx.x * WARPS + wib) * 32;
  double nrm = 0.0;

  unsigned char* base = smem_raw + (size_t)wib * ring_bytes_per_warp<ROLE>();
  RingPtrs<ROLE> R;
  R.rc = reinterpret_cast<double*>(base);
  R.rp = reinterpret_cast<float*>(base + 32 * RL * 8);
  R.ra = R.rp + 32 * RL;
  R.rG = R.ra + 32 * RL;
  R.rX = R.rG + 32 * RL;

  const bool warp_live = c0 < F.C;
  const int nvalid = warp_live ? (int)min((int64_t)32, F.C - c0) : 0;
  const bool valid = lane < nvalid;
  const int64_t c = c0 + lane;
  const int m = F.m;
  const int ntiles = (m + TP - 1) / TP;
  const int64_t my_base = valid ? fam_base(F, c) : 0;
  const int64_t C = F.C;

  // lane state (stackless taut string)
  int i0 = 0, pe = m, k = 0, c0x = 0, f0x = 0;
  double a_val = 0.0, a_S = 0.0, sk = 0.0, c0y = 0.0, f0y = 0.0;
  bool hc = false, hf = false;
  bool done = !valid;

  int t_lo = 0, t_ld = 0, t_rdy = 0;

  auto issue = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {  // mode A: family-owned arrays
      const int pos = k0 + q;
      const bool pr = valid && pos < m;
      const int64_t fi = pr ? (int64_t)pos * C + c : 0;
      cp4(&R.rp[rix(lane, pos)], A.p + fi, pr);
      cp4(&R.ra[rix(lane, pos)], A.wf + (pos < m - 1 ? fi : 0), pr && pos < m - 1);
      if (!ROWLIKE) {
        const int64_t nd = pr ? fam_node(F, my_base, pos) : 0;
        cp8(&R.rc[rix(lane, pos)], A.c + nd, pr);
        if (ROLE == MID || ROLE == LAST) cp4(&R.rG[rix(lane, pos)], A.G + nd, pr);
        if (ROLE == LAST) cp4(&R.rX[rix(lane, pos)], A.X + nd, pr);
      }
    }
    if (ROWLIKE) {  // mode B: 8 lanes along each chain's row, chains {b, b+8, b+16, b+24}
      const int q = lane & 7;
      const int pos = k0 + q;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        const bool pr = i < nvalid && pos < m;
        const int64_t nd = pr ? fam_node(F, bi, pos) : 0;
        cp8(&R.rc[rix(i, pos)], A.c + nd, pr);
        if (ROLE == MID) cp4(&R.rG[rix(i, pos)], A.G + nd, pr);
      }
    }
    cp_commit();
  };

  // global fall-back accessors for positions below the ring (lagging lanes)
  auto s_at = [&](int pos, int lo_pos) -> double {
    if (pos >= lo_pos) {
      const int ix = rix(lane, pos);
      return (double)R.rp[ix] + R.rc[ix];
    }
    return (double)A.p[(int64_t)pos * C + c] + A.c[fam_node(F, my_base, pos)];
  };
  auto a_at = [&](int pos, int lo_pos) -> double {
    if (pos >= lo_pos) return (double)R.ra[rix(lane, pos)];
    return (double)A.wf[(int64_t)pos * C + c];
  };

  // per-node completion in global memory (shared by retire and the lag path)
  auto finish_node = [&](int64_t fi, int64_t nd, float p32, float d, double pn, double cz,
                         float gin, float xin, bool from_ring) {
    if (ROLE == SHADOW) {
      A.y[nd] = pn;
      return;
    }
    A.p[fi] = p32;
    if (ROLE == FIRST) {
      A.G[nd] = d;
    } else if (ROLE == MID) {
      A.G[nd] = (float)((double)(from_ring ? gin : A.G[nd]) + (double)d);
    } else {
      const double g = (double)(from_ring ? gin : A.G[nd]) + (double)d;
      const double xn = (double)(from_ring ? xin : A.X[nd]) - g;
      A.X[nd] = (float)xn;
      const double dc = (xn - g) * A.inv_r;
      A.c[nd] = cz + dc;
      nrm += 2.0 * dc * g + A.rd * dc * dc;
    }
  };

  auto emit = [&](int j, double fill, int lo_pos) {
    if (j >= lo_pos) {
      const int ix = rix(lane, j);
      const float pold = R.rp[ix];
      const double cz = R.rc[ix];
      const double pn = ((double)pold + cz) - fill;
      if (ROLE == SHADOW) {
        R.rc[ix] = pn;
      } else {
        const float p32 = (float)pn;
        const double d = (double)p32 - (double)pold;
        R.rp[ix] = p32;
        R.ra[ix] = (float)d;
        nrm += d * d;
      }
    } else {
      const int64_t fi = (int64_t)j * C + c;
      const int64_t nd = fam_node(F, my_base, j);
      const float pold = A.p[fi];
      const double cz = A.c[nd];
      const double pn = ((double)pold + cz) - fill;
      const float p32 = (float)pn;
      const double d = (double)p32 - (double)pold;
      if (ROLE != SHADOW) nrm += d * d;
      finish_node(fi, nd, p32, (float)d, pn, cz, 0.f, 0.f, false);
    }
  };

  auto retire = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      if (valid && pos < m && pos < i0) {
        const int ix = rix(lane, pos);
        const int64_t fi = (int64_t)pos * C + c;
        if (ROLE != SHADOW) A.p[fi] = R.rp[ix];
        if (!ROWLIKE) {
          const int64_t nd = fam_node(F, my_base, pos);
          if (ROLE == SHADOW) {
            A.y[nd] = R.rc[ix];
          } else if (ROLE == FIRST) {
            A.G[nd] = R.ra[ix];
          } else if (ROLE == MID) {
            A.G[nd] = (float)((double)R.rG[ix] + (double)R.ra[ix]);
          } else {
            const double g = (double)R.rG[ix] + (double)R.ra[ix];
            const double xn = (double)R.rX[ix] - g;
            A.X[nd] = (float)xn;
            const double dc = (xn - g) * A.inv_r;
            A.c[nd] = R.rc[ix] + dc;
            nrm += 2.0 * dc * g + A.rd * dc * dc;
          }
        }
      }
    }
    if (ROWLIKE) {
      const int q = lane & 7;
      const int pos = k0 + q;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int i0_i = __shfl_sync(0xffffffffu, i0, i);
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        if (i < nvalid && pos < m && pos < i0_i) {
          const int ix = rix(i, pos);
          const int64_t nd = fam_node(F, bi, pos);
          if (ROLE == SHADOW) A.y[nd] = R.rc[ix];
          else if (ROLE == FIRST) A.G[nd] = R.ra[ix];
          else if (ROLE == MID) A.G[nd] = (float)((double)R.rG[ix] + (double)R.ra[ix]);
        }
      }
    }
  };

  if (warp_live) {
    // prologue: fill the ring
    while (t_ld < ntiles && t_ld < NT) issue(t_ld++);
    cp_wait(t_ld - 1);
    __syncwarp();
    t_rdy = 1;
    for (;;) {
      const int lo_pos = t_lo * TP;
      const int avail_hi = min(t_rdy * TP, m);
      // ---------------- lanes advance until they need data beyond avail_hi
      while (!done) {
        if (k >= avail_hi) break;
        const int kp = k;
        const double sv = s_at(kp, lo_pos);
        k = kp + 1;
        sk += sv;
        double rk = 0.0;
        if (k < m) {
          rk = a_at(kp, lo_pos);
          if (rk == 0.0) pe = k;
        }
        const double dk = (double)(k - i0);
        int bk = -1, bt = 0;
        double by = 0.0;
        const double uy = sk + rk;
        if (!hc || (uy - a_val) * (double)(c0x - i0) <= (c0y - a_val) * dk) {
          c0x = k;
          c0y = uy;
          hc = true;
        }
        if (hf && (c0y - a_val) * (double)(f0x - i0) < (f0y - a_val) * (double)(c0x - i0)) {
          bk = f0x;
          by = f0y;
          bt = -1;
        } else {
          const double ly = sk - rk;
          if (!hf || (ly - a_val) * (double)(f0x - i0) >= (f0y - a_val) * dk) {
            f0x = k;
            f0y = ly;
            hf = true;
          }
          if ((f0y - a_val) * (double)(c0x - i0) > (c0y - a_val) * (double)(f0x - i0)) {
            bk = c0x;
            by = c0y;
            bt = 1;
          } else if (k == pe) {
            const double dpe = (double)(pe - i0);
            if (c0x != pe && (c0y - a_val) * dpe < (sk - a_val) * (double)(c0x - i0)) {
              bk = c0x;
              by = c0y;
              bt = 1;
            } else if (f0x != pe && (f0y - a_val) * dpe > (sk - a_val) * (double)(f0x - i0)) {
              bk = f0x;
              by = f0y;
              bt = -1;
            } else {
              bk = pe;
              by = sk;
              bt = 0;
            }
          }
        }
        if (bk >= 0) {
          const double fill = (by - a_val) / (double)(bk - i0);
          const double nS = (bt == 0) ? by : by - (double)bt * a_at(bk - 1, lo_pos);
          for (int j = i0; j < bk; ++j) emit(j, fill, lo_pos);
          i0 = bk;
          if (i0 == pe) {
            a_val = 0.0;
            a_S = 0.0;
            pe = m;
            if (i0 >= m) done = true;
          } else {
            a_val = by;
            a_S = nS;
          }
          k = i0;
          sk = a_S;
          hc = hf = false;
        }
      }
      __syncwarp();
      const bool all_done = __all_sync(0xffffffffu, done);
      if (all_done) {
        cp_wait(0);
        __syncwarp();
        for (int T = t_lo; T < t_ld; ++T) retire(T);
        break;
      }
      // ---------------- retire tiles every lane has emitted
      const int front = __reduce_min_sync(0xffffffffu, done ? 0x7fffffff : i0);
      while (t_lo < t_rdy && (t_lo + 1) * TP <= front) retire(t_lo++);
      if (t_rdy == t_ld && t_ld - t_lo == NT) {
        // ring full, every lane waits for the next tile: retire the oldest
        // tile now; lanes still anchored in it continue in global memory
        retire(t_lo++);
      }
      __syncwarp();
      while (t_ld < ntiles && t_ld - t_lo < NT) issue(t_ld++);
      if (t_rdy < t_ld) {
        cp_wait(t_ld - t_rdy - 1);
        __syncwarp();
        ++t_rdy;
      }
    }
  }
  if (ROLE != SHADOW) {
    __shared__ double sh[WARPS];
    const double v = warp_sum(nrm);
    if (lane == 0) sh[wib] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < WARPS; ++w) t += sh[w];
      A.parts[blockIdx.x] = t;
    }
  }
}

}  // namespace fast
}  // namespace pcb
