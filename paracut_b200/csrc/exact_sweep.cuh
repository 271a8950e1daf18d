// exact_sweep.cuh -- staged warp kernel for the fp64 reference-exact sweep (PCB_F64).
//
// Same streaming structure as fast_sweep.cuh (one warp = 32 chains, a
// shared-memory ring per lane filled tiles ahead with cp.async, lockstep
// retire pass), but each lane runs the reference taut
// string itself (_kernels.py:11-142, as restated in taut_string.cuh): hull
// stacks with the reference's pop tests, absolute running sums, the segment
// value (sum + tube offsets)/len from a fresh sequential sum with the
// constant-run shortcut, and y = z - fill.  Every floating-point operation is
// the reference's, in the reference's order (compiled with -fmad=false), so
// the shadow is bitwise equal to prox_chains; chains are never split (that
// would change the running sums).
//
// Ring per lane: z (fp64, the AAR point of this family) and the edge weight
// (fp64); when a segment closes its value overwrites the weight slot of its
// first position (dead by then) and a start bit is set; the retire pass
// writes y_j = z_j - fill for whole tiles.  The segment sum is kept
// incrementally (same additions, same order as the reference's fresh sum),
// so closing a segment is O(1) and the warp does not diverge on it.  Hull
// stacks: the first HCX entries per lane in shared memory, deeper ones in
// the handle's global spill region.
#pragma once

namespace pcb {
namespace exact {

using fast::cp8;
using fast::cp_commit;
using fast::cp_wait;

// The fp64 scan is latency bound (~1.3 IPC).  Large grids (many warps per
// SM) want occupancy: a 16-position ring (two tiles in flight; a tile keeps
// a warp busy far longer than an HBM round trip) and 6 shared hull entries
// give 12.5 KB per warp, 16 warps per SM.  Small grids (fewer chain warps
// than SMs; 2D grids have only ~side chains per family) are bound by one
// warp's own latency and want the deeper 32-position ring.  All families of
// a sweep are independent (y_j depends on z_j only) and run in one launch.
#ifndef PCB_EXACT_UNROLL
#define PCB_EXACT_UNROLL 1
#endif
#ifndef PCB_EXACT_KEEP
#define PCB_EXACT_KEEP 16  // a round ends when at most this many lanes still have data
#endif
constexpr int WARPS = 4;
constexpr int TP = 8;   // positions per tile
constexpr int HCX = 6;  // hull entries per lane in shared memory

// ring slot of (lane, position): rows of RL slots, XOR-swizzled so that 32
// lanes at one position, or 8 positions of 4 lanes, hit distinct banks
template <int RL>
__device__ __forceinline__ int rix(int l, int pos) {
  static_assert(RL == 16 || RL == 32, "ring length");
  return RL == 32 ? ((l << 5) | ((pos & 31) ^ l)) : ((l << 4) | ((pos & 15) ^ (l & 15)));
}

constexpr int hull_bytes = 2 * HCX * 32 * (8 + 4);  // (y, x) x 2 hulls
template <int RL>
__host__ __device__ constexpr int warp_bytes() {
  return 32 * RL * (8 + 8) + hull_bytes;  // ring (z, a/fill) + hulls
}

struct Args {
  Fam F;
  const double* z;   // family AAR point, natural node layout
  double* y;         // shadow out, natural layout
  const double* wf;  // family weights, interleaved [pos][C]
  int* spx;          // hull spill (x), [(e - HCX) * gs + chain]
  double* spy;
  int* sfx;
  double* sfy;
  int64_t gs;
};

struct ArgSet {
  Args f[4];  // families, blockIdx.y selects
};

template <bool ROWLIKE, int RL>
__device__ __forceinline__ void sweep_warp(const Args& A, unsigned char* base, int64_t c0) {
  constexpr int NT = RL / TP;  // tiles in flight
  const int lane = threadIdx.x & 31;
  const Fam F = A.F;
  double* rz = reinterpret_cast<double*>(base);
  double* ra = rz + 32 * RL;
  double* hcy = reinterpret_cast<double*>(base + 32 * RL * 16);
  double* hfy = hcy + HCX * 32;
  int* hcx = reinterpret_cast<int*>(hfy + HCX * 32);
  int* hfx = hcx + HCX * 32;
  auto rix = [](int l, int pos) { return exact::rix<RL>(l, pos); };

  const int nvalid = (int)min((int64_t)32, F.C - c0);
  const bool valid = lane < nvalid;
  const int64_t c = c0 + lane;
  const int m = F.m;
  const int ntiles = (m + TP - 1) / TP;
  const int64_t my_base = valid ? fam_base(F, c) : 0;
  const int64_t C = F.C;

  // hull entry e of this lane: shared for e < HCX, global spill beyond
  auto cx_get = [&](int e) -> int {
    return e < HCX ? hcx[e * 32 + lane] : A.spx[(int64_t)(e - HCX) * A.gs + c];
  };
  auto cy_get = [&](int e) -> double {
    return e < HCX ? hcy[e * 32 + lane] : A.spy[(int64_t)(e - HCX) * A.gs + c];
  };
  auto fx_get = [&](int e) -> int {
    return e < HCX ? hfx[e * 32 + lane] : A.sfx[(int64_t)(e - HCX) * A.gs + c];
  };
  auto fy_get = [&](int e) -> double {
    return e < HCX ? hfy[e * 32 + lane] : A.sfy[(int64_t)(e - HCX) * A.gs + c];
  };
  auto c_put = [&](int e, int xv, double yv) {
    if (e < HCX) {
      hcx[e * 32 + lane] = xv;
      hcy[e * 32 + lane] = yv;
    } else {
      A.spx[(int64_t)(e - HCX) * A.gs + c] = xv;
      A.spy[(int64_t)(e - HCX) * A.gs + c] = yv;
    }
  };
  auto f_put = [&](int e, int xv, double yv) {
    if (e < HCX) {
      hfx[e * 32 + lane] = xv;
      hfy[e * 32 + lane] = yv;
    } else {
      A.sfx[(int64_t)(e - HCX) * A.gs + c] = xv;
      A.sfy[(int64_t)(e - HCX) * A.gs + c] = yv;
    }
  };

  // ---- lane state: the reference taut string (taut_string.cuh / _kernels.py)
  int i0 = 0, pe = m, k = 0, nc = 0, nf = 0, a_t = 0;
  double a_val = 0.0, a_S = 0.0, sk = 0.0, a_im1 = 0.0;
  double ref = 0.0, tot = 0.0, tc0 = 0.0, tf0 = 0.0;
  bool alleq = true, ec0 = true, ef0 = true;
  int c0x = 0, f0x = 0;
  double c0y = 0.0, f0y = 0.0;
  bool done = !valid;
  unsigned smask = 0u;  // ring positions that start a segment (value in the weight slot)
  double fcarry = 0.0;
  int t_lo = 0, t_ld = 0, t_rdy = 0;

  auto issue = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      const bool pr = valid && pos < m;
      const bool pa = pr && pos < m - 1;
      cp8(&ra[rix(lane, pos)], A.wf + (pa ? (int64_t)pos * C + c : 0), pa);
      if (!ROWLIKE) cp8(&rz[rix(lane, pos)], A.z + (pr ? fam_node(F, my_base, pos) : 0), pr);
    }
    if (ROWLIKE) {
      const int q = lane & 7;
      const int pos = k0 + q;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        const bool pr = i < nvalid && pos < m;
        cp8(&rz[rix(i, pos)], A.z + (pr ? fam_node(F, bi, pos) : 0), pr);
      }
    }
    cp_commit();
  };

  auto s_at = [&](int pos, int lo_pos) -> double {
    if (pos >= lo_pos) return rz[rix(lane, pos)];
    return A.z[fam_node(F, my_base, pos)];
  };
  auto a_at = [&](int pos, int lo_pos) -> double {
    if (pos >= lo_pos) return ra[rix(lane, pos)];
    return A.wf[(int64_t)pos * C + c];
  };

  // lockstep retire of tile T: y = z - fill for every emitted position
  auto retire = [&](int T) {
    const int k0 = T * TP;
    // every lane emitted the whole tile (the usual case): straight-line, ring
    // slots rix(k0) ^ q, strided outputs at a per-tile base + q * ns
    if (__all_sync(0xffffffffu, valid && k0 + TP <= m && k0 + TP <= i0)) {
      const int ixb = rix(lane, k0);
      const unsigned stile = smask >> (k0 & (RL - 1));
      double* const yb = ROWLIKE ? nullptr : A.y + fam_node(F, my_base, k0);
      // (row-like: the ring stores after the loop, so the loop's ring loads
      // are not ordered behind them)
      double yq[TP];
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        const int ix = ixb ^ q;
        if ((stile >> q) & 1u) fcarry = ra[ix];
        yq[q] = rz[ix] - fcarry;
        if (!ROWLIKE) yb[(int64_t)q * F.ns] = yq[q];
      }
      if (ROWLIKE) {
#pragma unroll
        for (int q = 0; q < TP; ++q) rz[ixb ^ q] = yq[q];
      }
    } else {
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      if (valid && pos < m && pos < i0) {
        const int ix = rix(lane, pos);
        if ((smask >> (pos & (RL - 1))) & 1u) fcarry = ra[ix];
        const double yv = rz[ix] - fcarry;
        if (!ROWLIKE) A.y[fam_node(F, my_base, pos)] = yv;
        else rz[ix] = yv;
      }
    }
    }
    smask &= ~(((1u << TP) - 1u) << (k0 & (RL - 1)));
    if (ROWLIKE) {
      __syncwarp();
      const int pos = k0 + (lane & 7);
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int i0_i = __shfl_sync(0xffffffffu, i0, i);
        const int64_t bi = __shfl_sync(0xffffffffu, my_base, i);
        if (i < nvalid && pos < m && pos < i0_i) A.y[fam_node(F, bi, pos)] = rz[rix(i, pos)];
      }
      __syncwarp();
    }
  };

  // Hull tops in registers: t1 = entry n-1, t2 = entry n-2 (the anchor when
  // n == 1), so a push that pops nothing (the common case) touches shared
  // memory only to store the new entry.  Entry 0 is (c0x, c0y) / (f0x, f0y).
  int ct1x = 0, ct2x = 0, ft1x = 0, ft2x = 0;
  double ct1y = 0.0, ct2y = 0.0, ft1y = 0.0, ft2y = 0.0;

  auto scan = [&](int lo_pos, int avail_hi, int keep_min) {
    // software-pipelined ring reads: the next gate's z and weight are loaded
    // at the end of the previous trip (slots >= k are never written by the scan)
    double zn = 0.0, an = 0.0;
    if (!done && k < avail_hi) {
      zn = s_at(k, lo_pos);
      an = k < m - 1 ? a_at(k, lo_pos) : 0.0;
    }
    auto trip = [&]() {
      const bool act = !done && k < avail_hi;
      if (!act) return;
      // ---- one gate of the reference loop (_kernels.py:41-95)
      ++k;
      const double v = zn;
      sk += v;
      // the segment sum from the anchor, in the reference's order (a fresh
      // sequential sum from 0.0), kept incrementally: the closing position
      // is always the current gate or one of the two bottom hull points,
      // whose prefixes are kept with them
      ref = (k == i0 + 1) ? v : ref;
      tot += v;
      alleq = alleq && (v == ref);
      double rk = 0.0;
      if (k < m) {
        rk = an;
        if (rk == 0.0) pe = k;
      }
      int bk = -1, bt = 0;
      double by = 0.0;
      const double uy = sk + rk;
      while (nc >= 1) {
        if ((ct1y - ct2y) * (double)(k - ct1x) >= (uy - ct1y) * (double)(ct1x - ct2x)) {
          --nc;
          ct1x = ct2x;
          ct1y = ct2y;
          if (nc >= 3) {
            ct2x = cx_get(nc - 2);
            ct2y = cy_get(nc - 2);
          } else if (nc == 2) {
            ct2x = c0x;
            ct2y = c0y;
          } else {
            ct2x = i0;
            ct2y = a_val;
          }
        } else {
          break;
        }
      }
      c_put(nc, k, uy);
      if (nc == 0) {
        c0x = k;
        c0y = uy;
        tc0 = tot;
        ec0 = alleq;
        ct2x = i0;
        ct2y = a_val;
      } else {
        ct2x = ct1x;
        ct2y = ct1y;
      }
      ct1x = k;
      ct1y = uy;
      ++nc;
      if (nf >= 1 && (c0y - a_val) * (double)(f0x - i0) < (f0y - a_val) * (double)(c0x - i0)) {
        bk = f0x;
        by = f0y;
        bt = -1;
      } else {
        const double ly = sk - rk;
        while (nf >= 1) {
          if ((ft1y - ft2y) * (double)(k - ft1x) <= (ly - ft1y) * (double)(ft1x - ft2x)) {
            --nf;
            ft1x = ft2x;
            ft1y = ft2y;
            if (nf >= 3) {
              ft2x = fx_get(nf - 2);
              ft2y = fy_get(nf - 2);
            } else if (nf == 2) {
              ft2x = f0x;
              ft2y = f0y;
            } else {
              ft2x = i0;
              ft2y = a_val;
            }
          } else {
            break;
          }
        }
        f_put(nf, k, ly);
        if (nf == 0) {
          f0x = k;
          f0y = ly;
          tf0 = tot;
          ef0 = alleq;
          ft2x = i0;
          ft2y = a_val;
        } else {
          ft2x = ft1x;
          ft2y = ft1y;
        }
        ft1x = k;
        ft1y = ly;
        ++nf;
        if ((f0y - a_val) * (double)(c0x - i0) > (c0y - a_val) * (double)(f0x - i0)) {
          bk = c0x;
          by = c0y;
          bt = 1;
        } else if (k == pe) {
          // piece end (_kernels.py:97-114)
          if (c0x != pe && (c0y - a_val) * (double)(pe - i0) < (sk - a_val) * (double)(c0x - i0)) {
            bk = c0x;
            by = c0y;
            bt = 1;
          } else if (f0x != pe &&
                     (f0y - a_val) * (double)(pe - i0) > (sk - a_val) * (double)(f0x - i0)) {
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
        // ---- close [i0, bk) (_kernels.py:116-137)
        const double stot = (bk == k) ? tot : (bk == c0x) ? tc0 : tf0;
        const bool seq = (bk == k) ? alleq : (bk == c0x) ? ec0 : ef0;
        double corr = 0.0;
        const double abk = (bt != 0) ? a_at(bk - 1, lo_pos) : 0.0;
        if (bt != 0) corr += (double)bt * abk;
        if (a_t != 0) corr -= (double)a_t * a_im1;
        const double fill = (seq && corr == 0.0) ? ref : (stot + corr) / (double)(bk - i0);
        int e2 = i0;
        if (i0 < lo_pos) {
          // lagging lane (anchor below the ring): positions below go straight out
          e2 = min(bk, lo_pos);
          for (int j = i0; j < e2; ++j) {
            const int64_t nd = fam_node(F, my_base, j);
            A.y[nd] = A.z[nd] - fill;
          }
        }
        if (e2 < bk) {
          ra[rix(lane, e2)] = fill;  // weight slot of e2 is dead from here: holds the value
          smask |= 1u << (e2 & (RL - 1));
        }
        i0 = bk;
        if (i0 == pe) {
          a_val = 0.0;
          a_t = 0;
          a_S = 0.0;
          pe = m;
          done = i0 >= m;
        } else {
          a_val = by;
          a_t = bt;
          a_S = (bt == 0) ? by : by - (double)bt * abk;
        }
        a_im1 = abk;
        k = i0;
        sk = a_S;
        tot = 0.0;
        alleq = true;
        nc = nf = 0;
      }
      if (!done && k < avail_hi) {
        zn = s_at(k, lo_pos);
        an = k < m - 1 ? a_at(k, lo_pos) : 0.0;
        // The first gate after a restart pushes one point on both hulls and
        // cannot bend unless it ends the piece (zero weight, chain end), so it
        // is taken here with the same operations instead of in a trip of its
        // own.  Entry 0 of a hull lives in registers only.
        if (bk >= 0 && k + 1 < pe && an != 0.0) {
          ++k;
          const double v1 = zn;
          sk += v1;
          ref = v1;
          tot += v1;
          alleq = alleq && (v1 == ref);
          const double u1 = sk + an, l1 = sk - an;
          c0x = k;
          c0y = u1;
          tc0 = tot;
          ec0 = alleq;
          ct2x = i0;
          ct2y = a_val;
          ct1x = k;
          ct1y = u1;
          nc = 1;
          f0x = k;
          f0y = l1;
          tf0 = tot;
          ef0 = alleq;
          ft2x = i0;
          ft2y = a_val;
          ft1x = k;
          ft1y = l1;
          nf = 1;
          if (k < avail_hi) {
            zn = s_at(k, lo_pos);
            an = k < m - 1 ? a_at(k, lo_pos) : 0.0;
          }
        }
      }
    };
    for (;;) {
      if (__popc(__ballot_sync(0xffffffffu, !done && k < avail_hi)) <= keep_min) break;
      // PCB_EXACT_UNROLL trips per exit vote (same gates, fewer votes)
#pragma unroll
      for (int u = 0; u < PCB_EXACT_UNROLL; ++u) trip();
    }
  };

  {
    while (t_ld < ntiles && t_ld < NT) issue(t_ld++);
    cp_wait(t_ld - 1);
    __syncwarp();
    t_rdy = 1;
    for (;;) {
      const int lo_pos = t_lo * TP;
      const int avail_hi = min(t_rdy * TP, m);
      scan(lo_pos, avail_hi, (t_rdy < t_ld) ? PCB_EXACT_KEEP : 0);
      __syncwarp();
      if (__all_sync(0xffffffffu, done)) {
        cp_wait(0);
        __syncwarp();
        for (int T = t_lo; T < t_ld; ++T) retire(T);
        break;
      }
      const int front = __reduce_min_sync(0xffffffffu, done ? 0x7fffffff : i0);
      while (t_lo < t_rdy && (t_lo + 1) * TP <= front) retire(t_lo++);
      const bool any_act = __any_sync(0xffffffffu, !done && k < avail_hi);
      if (!any_act && t_rdy == t_ld && t_ld - t_lo == NT) retire(t_lo++);
      __syncwarp();
      while (t_ld < ntiles && t_ld - t_lo < NT) issue(t_ld++);
      if (t_rdy < t_ld) {
        cp_wait(t_ld - t_rdy - 1);
        __syncwarp();
        ++t_rdy;
      }
    }
  }
}

template <int RL>
__global__ void __launch_bounds__(WARPS * 32) k_sweep_exact(ArgSet S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Args& A = S.f[blockIdx.y];
  const int wib = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * WARPS + wib) * 32;
  if (c0 >= A.F.C) return;  // warp-uniform; no block-wide barrier below
  unsigned char* base = smem_raw + (size_t)wib * warp_bytes<RL>();
  if (fam_rowlike(A.F.kind))
    sweep_warp<true, RL>(A, base, c0);
  else
    sweep_warp<false, RL>(A, base, c0);
}

}  // namespace exact
}  // namespace pcb
