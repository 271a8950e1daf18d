// fast_sweep.cuh -- staged warp kernel for the fp32-state AAR sweep (PCB_F32).
//
// One warp owns 32 chains of one family (lane l <-> chain c0 + l).  Chain data
// streams through a per-warp shared-memory ring of RL = 32 positions (NT
// tiles of TP positions) filled with cp.async (LDGSTS) a few tiles ahead:
//
//   mode A (lane = chain, one instruction per position): family-owned arrays
//          (p_j, weights -- chain-interleaved [pos][C]) and, for families
//          whose chains are strided in memory (cols, y, z), the shared drift
//          c: 128-byte coalesced;
//   mode B (8 lanes along a row, 4 chains per instruction): c for row-like
//          families (rows, 3D x, 2D-8 zig-zags), coalesced along the rows.
//
// Ring layout [lane][32], slot XOR-swizzled by the lane id: both load modes,
// the lockstep passes and per-lane reads at equal positions are conflict
// free.  When a tile lands one lockstep pass turns the c slot into z = p + c.
// Retire-only inputs (accumulator G, primal X) are prefetched into registers
// one round before their tile retires.
//
// Each lane runs a stackless taut string in the anchor's frame.  It keeps
// the minimum-slope ceiling point and the maximum-slope floor point only --
// the bottom entries of the reference's hull stacks (_kernels.py:47-95), the
// only entries its cone tests read -- as (gate, slope) pairs, so the cone
// tests are plain compares and a bend's prox value is the stored slope:
// (y_bend - y_anchor)/(bk - i0) equals the reference's (sum + tube
// offsets)/len.  Slopes use exact reciprocals of the small integer offsets
// from a shared table.  Closing a segment is O(1): the lane writes
// q = z_i0 - fill at the segment start and sets a start bit; per-node
// outputs are produced by a lockstep retire pass over whole tiles
// (p_new = (z_j - z_start) + q) and written back coalesced.  A lane whose
// anchor falls behind the ring reads and writes those positions in global
// memory; retirement is masked by each lane's emitted frontier.
#pragma once

namespace pcb {
namespace fast {

constexpr int TP = 8;          // positions per tile
constexpr int NT = 4;          // tiles in the ring
constexpr int RL = TP * NT;    // ring length (positions)
constexpr int WARPS = 4;       // warps per block
constexpr int INV_N = 64;      // reciprocal table size
static_assert(RL == 32, "swizzle and start masks assume a 32-position ring");
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
__host__ __device__ constexpr int ring_bytes_host() {
  // rz f64, rp f32, ra f32 (+ rf f64 for SHADOW)
  return 32 * RL * (8 + 4 + 4 + (ROLE == SHADOW ? 8 : 0));
}

// lagging-lane accessors (positions below the ring), kept out of line
__device__ __noinline__ double z_global(const Args& A, int64_t fi, int64_t nd) {
  return (double)A.p[fi] + A.c[nd];
}
__device__ __noinline__ double a_global(const Args& A, int64_t fi) { return (double)A.wf[fi]; }

template <int ROLE>
__device__ __noinline__ double finish_global(const Args& A, int64_t fi, int64_t nd, double fill) {
  const float pold = A.p[fi];
  const double cz = A.c[nd];
  const double pn = ((double)pold + cz) - fill;
  if (ROLE == SHADOW) {
    A.y[nd] = pn;
    return 0.0;
  }
  const float p32 = (float)pn;
  const double d = (double)p32 - (double)pold;
  double nrm = d * d;
  A.p[fi] = p32;
  if (ROLE == FIRST) {
    A.G[nd] = (float)d;
  } else if (ROLE == MID) {
    A.G[nd] = (float)((double)A.G[nd] + d);
  } else {
    const double g = (double)A.G[nd] + d;
    const double xn = (double)A.X[nd] - g;
    A.X[nd] = (float)xn;
    const double dcv = (xn - g) * A.inv_r;
    A.c[nd] = cz + dcv;
    nrm += 2.0 * dcv * g + A.rd * dcv * dcv;
  }
  return nrm;
}

template <int ROLE, bool ROWLIKE>
__global__ void __launch_bounds__(WARPS * 32) k_sweep(Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double inv_tab[INV_N];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Fam F = A.F;
  const int64_t c0 = ((int64_t)blockIdx.x * WARPS + wib) * 32;
  double nrm = 0.0;
  for (int t = threadIdx.x; t < INV_N; t += blockDim.x) inv_tab[t] = t ? 1.0 / (double)t : 0.0;
  __syncthreads();

  unsigned char* base = smem_raw + (size_t)wib * ring_bytes_host<ROLE>();
  double* rz = reinterpret_cast<double*>(base);
  double* rf = rz + 32 * RL;  // SHADOW only
  float* rp = reinterpret_cast<float*>(base + 32 * RL * (ROLE == SHADOW ? 16 : 8));
  float* ra = rp + 32 * RL;

  const bool warp_live = c0 < F.C;
  const int nvalid = warp_live ? (int)min((int64_t)32, F.C - c0) : 0;
  const bool valid = lane < nvalid;
  const int64_t c = c0 + lane;
  const int m = F.m;
  const int ntiles = (m + TP - 1) / TP;
  const int64_t my_base = valid ? fam_base(F, c) : 0;
  const int64_t C = F.C;

  // ---- lane state: stackless taut string in the anchor frame
  int i0 = 0, pe = m, k = 0, c0x = -1, f0x = -1;
  double skr = 0.0;   // running sum minus the anchor value
  double cs = 0.0;    // min slope anchor -> ceiling points
  double fs = 0.0;    // max slope anchor -> floor points
  bool done = !valid;
  unsigned smask = 0u;        // segment starts inside the ring (bit = slot)
  double zs = 0.0, qs = 0.0;  // retire carry: z at the current segment start, q there

  // retire-only inputs prefetched into registers (G for MID/LAST, X for LAST)
  float gpre[TP], xpre[TP];
  int pre_tile = -1;

  int t_lo = 0, t_ld = 0, t_rdy = 0;

  auto issue = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {  // mode A
      const int pos = k0 + q;
      const bool pr = valid && pos < m;
      const int64_t fi = pr ? (int64_t)pos * C + c : 0;
      cp4(&rp[rix(lane, pos)], A.p + fi, pr);
      cp4(&ra[rix(lane, pos)], A.wf + (pos < m - 1 ? fi : 0), pr && pos < m - 1);
      if (!ROWLIKE) {
        const int64_t nd = pr ? fam_node(F, my_base, pos) : 0;
        cp8(&rz[rix(lane, pos)], A.c + nd, pr);
      }
    }
    if (ROWLIKE) {  // mode B: lanes 8g..8g+7 along chain rows {8g + ib}
      const int q = lane & 7;
      const int pos = k0 + q;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        const bool pr = i < nvalid && pos < m;
        const int64_t nd = pr ? fam_node(F, bi, pos) : 0;
        cp8(&rz[rix(i, pos)], A.c + nd, pr);
      }
    }
    cp_commit();
  };

  // G/X of tile T into registers (mode A natural; mode B rows for row-like MID)
  auto prefetch = [&](int T) {
    pre_tile = T;
    if (ROLE != MID && ROLE != LAST) return;
    const int k0 = T * TP;
    if (!ROWLIKE) {
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        const int pos = k0 + q;
        const bool pr = valid && pos < m;
        const int64_t nd = pr ? fam_node(F, my_base, pos) : 0;
        gpre[q] = pr ? A.G[nd] : 0.f;
        if (ROLE == LAST) xpre[q] = pr ? A.X[nd] : 0.f;
      }
    } else {
      const int pos = k0 + (lane & 7);
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        const bool pr = i < nvalid && pos < m;
        gpre[ib] = pr ? A.G[fam_node(F, bi, pos)] : 0.f;
      }
    }
  };

  // tile T landed: c slot -> z = p + c (lockstep)
  auto to_z = [&](int T) {
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int ix = rix(lane, T * TP + q);
      rz[ix] = (double)rp[ix] + rz[ix];
    }
  };

  // lockstep retire of tile T: per-node outputs from (z, segment markers), write back
  auto retire = [&](int T) {
    if (pre_tile != T) prefetch(T);
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      if (valid && pos < m && pos < i0) {
        const int slot = pos & (RL - 1);
        const int ix = rix(lane, pos);
        const double zj = rz[ix];
        if ((smask >> slot) & 1u) {
          zs = zj;
          qs = (ROLE == SHADOW) ? rf[ix] : (double)ra[ix];
        }
        const double pn = (zj - zs) + qs;
        if (ROLE == SHADOW) {
          if (!ROWLIKE) A.y[fam_node(F, my_base, pos)] = pn;
          else rz[ix] = pn;
        } else {
          const float pold = rp[ix];
          const float p32 = (float)pn;
          const double d = (double)p32 - (double)pold;
          nrm += d * d;
          A.p[(int64_t)pos * C + c] = p32;
          if (!ROWLIKE) {
            const int64_t nd = fam_node(F, my_base, pos);
            if (ROLE == FIRST) {
              A.G[nd] = (float)d;
            } else if (ROLE == MID) {
              A.G[nd] = (float)((double)gpre[q] + d);
            } else {
              const double g = (double)gpre[q] + d;
              const double xn = (double)xpre[q] - g;
              A.X[nd] = (float)xn;
              const double dcv = (xn - g) * A.inv_r;
              A.c[nd] = (zj - (double)pold) + dcv;  // c_old = z - p_old
              nrm += 2.0 * dcv * g + A.rd * dcv * dcv;
            }
          } else {
            ra[ix] = (float)d;
          }
        }
      }
    }
    smask &= ~(0xffu << ((k0 & (RL - 1))));
    if (ROWLIKE) {
      __syncwarp();
      const int pos = k0 + (lane & 7);
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int i0_i = __shfl_sync(0xffffffffu, i0, i);
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        if (i < nvalid && pos < m && pos < i0_i) {
          const int ix = rix(i, pos);
          const int64_t nd = fam_node(F, bi, pos);
          if (ROLE == SHADOW) A.y[nd] = rz[ix];
          else if (ROLE == FIRST) A.G[nd] = ra[ix];
          else if (ROLE == MID) A.G[nd] = (float)((double)gpre[ib] + (double)ra[ix]);
        }
      }
      __syncwarp();
    }
  };

  if (warp_live) {
    while (t_ld < ntiles && t_ld < NT) issue(t_ld++);
    cp_wait(t_ld - 1);
    __syncwarp();
    to_z(0);
    t_rdy = 1;
    for (;;) {
      const int lo_pos = t_lo * TP;
      const int avail_hi = min(t_rdy * TP, m);
      if (pre_tile != t_lo) prefetch(t_lo);
      // ---------------- scan until every lane needs data beyond avail_hi
      while (!done && k < avail_hi) {
        const int kp = k;
        double zv, av = 0.0;
        if (kp >= lo_pos) {
          const int ix = rix(lane, kp);
          zv = rz[ix];
          av = ra[ix];
        } else {
          const int64_t fi = (int64_t)kp * C + c;
          zv = z_global(A, fi, fam_node(F, my_base, kp));
          if (kp < m - 1) av = a_global(A, fi);
        }
        k = kp + 1;
        skr += zv;
        const int dki = k - i0;
        const double inv = dki < INV_N ? inv_tab[dki] : 1.0 / (double)dki;
        double rk = 0.0;
        if (k < m) {
          rk = av;
          if (rk == 0.0) pe = k;
        }
        const double su = (skr + rk) * inv;
        if (c0x < 0 || su <= cs) {
          c0x = k;
          cs = su;
        }
        int bk = -1, bt = 0;
        double fill = 0.0;
        if (f0x >= 0 && cs < fs) {
          bk = f0x; fill = fs; bt = -1;
        } else {
          const double sl = (skr - rk) * inv;
          if (f0x < 0 || sl >= fs) {
            f0x = k;
            fs = sl;
          }
          if (fs > cs) {
            bk = c0x; fill = cs; bt = 1;
          } else if (k == pe) {
            const double sa = skr * inv;
            if (c0x != pe && cs < sa) {
              bk = c0x; fill = cs; bt = 1;
            } else if (f0x != pe && fs > sa) {
              bk = f0x; fill = fs; bt = -1;
            } else {
              bk = pe; fill = sa; bt = 0;
            }
          }
        }
        if (bk >= 0) {
          // close segment [i0, bk): its prox value is the string slope `fill`
          double nskr = 0.0;
          if (bt != 0) {
            const int pa = bk - 1;
            const double ab = pa >= lo_pos ? (double)ra[rix(lane, pa)]
                                           : a_global(A, (int64_t)pa * C + c);
            nskr = -(double)bt * ab;
          }
          int s0 = i0;
          if (s0 < lo_pos) {  // lagging lane: the part below the ring goes straight to memory
            const int e = min(bk, lo_pos);
            for (int j = s0; j < e; ++j)
              nrm += finish_global<ROLE>(A, (int64_t)j * C + c, fam_node(F, my_base, j), fill);
            s0 = e;
          }
          if (s0 < bk) {
            const int ix = rix(lane, s0);
            const double qv = rz[ix] - fill;
            if (ROLE == SHADOW) rf[ix] = qv;
            else ra[ix] = (float)qv;
            smask |= 1u << (s0 & (RL - 1));
          }
          i0 = bk;
          if (i0 == pe) {
            pe = m;
            skr = 0.0;
            done = i0 >= m;
          } else {
            skr = nskr;
          }
          k = i0;
          c0x = f0x = -1;
        }
      }
      __syncwarp();
      if (__all_sync(0xffffffffu, done)) {
        cp_wait(0);
        __syncwarp();
        for (int T = t_lo; T < t_ld; ++T) retire(T);
        break;
      }
      // ---------------- retire tiles every lane has emitted
      const int front = __reduce_min_sync(0xffffffffu, done ? 0x7fffffff : i0);
      while (t_lo < t_rdy && (t_lo + 1) * TP <= front) retire(t_lo++);
      if (t_rdy == t_ld && t_ld - t_lo == NT) retire(t_lo++);  // ring full: lagging lanes go global
      __syncwarp();
      while (t_ld < ntiles && t_ld - t_lo < NT) issue(t_ld++);
      if (t_rdy < t_ld) {
        cp_wait(t_ld - t_rdy - 1);
        __syncwarp();
        to_z(t_rdy);
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
