// lean_verify.cuh -- the verified sweep of one chain family.
//
// Each AAR iteration changes the input z of a family's prox only slightly, and
// after the first few dozen iterations almost every chain keeps its
// segmentation (measured: < 3 % of chains change after ~100
// iterations on cfg4).  This kernel takes last iteration's segmentation (the
// per-edge hints the scan writes) as a candidate solution, computes it in
// closed form and checks the complete KKT conditions of the prox
// (_kernels.py:11-142 computes the same minimiser with the taut string):
//
//   x_i = z_i - u_i + u_{i-1},   |u_i| <= a_i,
//   u_i = -a_i sign(x_{i+1} - x_i)  where x jumps,
//
// with u the dual on the edges (u = -a at a ceiling touch of the string, +a at
// a floor touch, 0 at a piece end).  A segment [s, e] between two touches has
// x = (sum z + u_{s-1} - u_e) / len, its interior duals are prefix sums and
// must stay in the tube (a cone of slopes from the segment start), and the
// jump over each touch must have the touch's sign.  Chains whose candidate
// fails anywhere are repaired after the sweep (repair_lane in fast_sweep.cuh:
// the exact taut string between two true points around the failures).
//
// Layout: one warp = 32 consecutive chains of the family (lane = chain), one
// position per step for all lanes in lockstep, tiles of TP = 8 positions.  No
// shared-memory ring: the next tile is loaded straight into registers while
// the current one is verified -- p_j and the weights (interleaved [pos][C])
// and, for strided families, c / G / X are coalesced across the lanes; for
// row-like families (rows, 3D x) a chain's c / G / X are contiguous, so each
// lane moves its own 8 positions as 16-byte vectors.  A tile is retired
// (p', d, G, X, c, step-norm terms) one tile later, when the segments covering
// it have closed; the segment-start values q = z_s - x live in a 16-slot
// per-lane shared array.  A segment still open after that window (longer than
// about a tile) leaves a hole -- NaN in p' and no fused update -- and marks the
// chain for repair, which rewrites the range.
#pragma once

namespace pcb {
namespace fast {

constexpr int LV_WARPS = 4;  // warps per block (no ring: occupancy is register bound)
constexpr int NREG = 4;      // failure regions repaired separately per chain
constexpr int RGAP = 16;     // failures further apart than this start a new region
#ifndef PCB_VTOL
#define PCB_VTOL 4e-6f  // slack of the KKT checks (fp32 rounding; values are O(weights))
#endif


// ---------------------------------------------------------------------------
// Fast local repair (the common case at late iterations: one failure region
// a few positions long).  The same algorithm as repair_lane, with the window
// [g0, g0 + RW) of z and a staged into shared memory first (all loads in
// flight together instead of one dependent global load per step), the new
// segment values kept there until the string has reached a consistent bend,
// and the outputs written in a final pass.  Returns false -- having written
// nothing -- when the repair would leave the window; repair_lane then runs.
// repair diagnostics (pcb_debug_counters without PCB_COUNT): fast repairs,
// fast-path exits (no true point / left the window in the search / in the
// string), slow repairs
__device__ unsigned long long g_rep[8];
#define PCB_REP(i) atomicAdd(&g_rep[i], 1ull)
constexpr int RW = 48;    // window positions
constexpr int RROWS = 8;  // lanes repaired at a time per warp
struct RepairWin {
  double z[RW][RROWS];
  double x[RW][RROWS];
  float p[RW][RROWS];
  float a[RW][RROWS];
};

template <int ROLE, bool ROWLIKE>
__device__ __noinline__ bool repair_fast(const Args& A, int c32, int base32, int ff, int fl,
                                         RepairWin& W, int row, double* nrm_out) {
  const Fam& F = A.F;
  const int m = F.m, C32 = (int)F.C, ns32 = (int)F.ns;
  auto node = [&](int pos) { return base32 + pos * ns32; };
  const int g0 = max(0, ff - 12);
  const int wn = min(RW, m - g0);
#pragma unroll 8
  for (int j = 0; j < RW; ++j) {
    if (j < wn) {
      const int pos = g0 + j;
      const float pv = __ldg(A.p + pos * C32 + c32);
      const double cv = __ldg(A.c + node(pos));
      W.p[j][row] = pv;
      W.z[j][row] = (double)pv + cv;
      W.a[j][row] = pos < m - 1 ? __ldg(A.wf + pos * C32 + c32) : 0.f;
    }
  }
  bool oob = false;
  auto za = [&](int pos, double* z, double* a) {
    const int j = pos - g0;
    if (j >= 0 && j < wn) {
      *z = W.z[j][row];
      *a = (double)W.a[j][row];
    } else {
      oob = true;
      *z = 0.0;
      *a = 1.0;
    }
  };
  auto cand = [&](int e) {
    const unsigned w = A.sg[(e / TP) * C32 + c32];
    const int q = e % TP;
    return (int)((w >> q) & 1u) - (int)((w >> (8 + q)) & 1u);
  };
  // 1. q_L inside the window
  int qL = -1, qt = 0;
  for (int delta = 4; delta <= 8; delta *= 2) {
    const int g = ff - delta;
    if (g <= 0) {
      qL = 0;
      break;
    }
    if (g < g0) break;
    const double ag = (double)W.a[g - 1 - g0 >= 0 ? g - 1 - g0 : 0][row];
    if (g - 1 < g0) break;
    if (ag == 0.0) {
      qL = g;
      break;
    }
    Spec Fs{g, m, g, -1, -1, 0.0, ag, 0.0, 0.0, 0.0, 0.0, true};
    Spec Us{g, m, g, -1, -1, 0.0, -ag, 0.0, 0.0, 0.0, 0.0, true};
    int pf, tf, pu, tu;
    spec_next_bend(Fs, m, za, &pf, &tf);
    spec_next_bend(Us, m, za, &pu, &tu);
    int q = -1, t = 0;
    for (;;) {
      if (oob) break;
      if (pf == pu && tf == tu) {
        q = pf;
        t = tf;
        break;
      }
      if (min(pf, pu) > ff) break;
      if (pf <= pu) spec_next_bend(Fs, m, za, &pf, &tf);
      else spec_next_bend(Us, m, za, &pu, &tu);
    }
    if (oob) {
      PCB_REP(2);
      return false;
    }
    if (q >= 0 && q <= ff && (t == 0 || cand(q - 1) == t)) {
      qL = q;
      qt = t;
      break;
    }
  }
  if (qL < 0) {
    PCB_REP(1);
    return false;
  }
  // 2. the exact string from q_L, segment values into the window
  const double a0 = (qL > 0 && qt != 0) ? (double)W.a[qL - 1 - g0][row] : 0.0;
  Spec S{qL, m, qL, -1, -1, 0.0, -(double)qt * a0, 0.0, 0.0, 0.0, 0.0, true};
  int s0 = qL, b = qL;
  for (;;) {
    int bk, bt;
    double xv;
    spec_next_bend(S, m, za, &bk, &bt, &xv);
    if (oob || bk - g0 > wn) {
      PCB_REP(3);
      return false;
    }
    for (int j = s0; j < bk; ++j) W.x[j - g0][row] = xv;
    s0 = bk;
    if (bk >= m || (bk - 1 > fl && (bt == 0 || cand(bk - 1) == bt))) {
      b = bk;
      break;
    }
  }
  // 3. outputs of [q_L, b) and hints of its inner edges
  double nrm = 0.0;
  for (int j = qL; j < b; ++j) {
    const int fi = j * C32 + c32, nd = node(j), w = j - g0;
    const float pin = W.p[w][row];
    const double z = W.z[w][row];
    const double cz = z - (double)pin;
    const float p32 = (float)(z - W.x[w][row]);
    const double d = (double)p32 - (double)pin;
    const float pw = A.po[fi];
    const bool was = !isnan(pw);
    const double dw = was ? (double)pw - (double)pin : 0.0;
    double r = d * d - dw * dw;
    A.po[fi] = p32;
    if (ROLE == FIRST) {
      A.G[nd] = (float)d;
    } else if (ROLE == MID) {
      A.G[nd] = (float)((double)A.Gi[nd] + d);
    } else {
      const double gi = (double)A.Gi[nd], xi = (double)A.X[nd];
      const double g = (double)(float)(gi + d);
      const double xn = xi - g;
      A.Xo[nd] = (float)xn;
      const double dcv = (xn - g) * A.inv_r;
      A.co[nd] = cz + dcv;
      r += dcv * (A.rd * dcv + g + g);
      if (was) {
        const double gw = (double)(float)(gi + dw);
        const double dcw = ((xi - gw) - gw) * A.inv_r;
        r -= dcw * (A.rd * dcw + gw + gw);
      }
    }
    nrm += r;
    if (j < b - 1 && j < m - 1) {  // edge j: the jump between the new values
      const double xa = W.x[w][row], xb = W.x[w + 1][row];
      uint16_t* wp = A.sg + (j / TP) * C32 + c32;
      const int q = j % TP;
      unsigned hw = *wp & ~((1u << q) | (1u << (8 + q)));
      hw |= xb > xa ? (1u << q) : (xb < xa ? (1u << (8 + q)) : 0u);
      *wp = (uint16_t)hw;
    }
  }
  *nrm_out = nrm;
  PCB_REP(0);
  return true;
}

template <int ROLE, bool ROWLIKE>
__global__ void __launch_bounds__(LV_WARPS * 32, 3)
    k_verify(const __grid_constant__ Args A) {
  if (A.vmode != nullptr && *A.vmode != 1) return;  // the scan runs this iteration
  __shared__ float qsm[LV_WARPS][17][32];            // q at segment starts (slot = pos & 15)
  __shared__ RepairWin rwin[LV_WARPS];
  __shared__ int2 regs_sm[LV_WARPS][NREG - 1][32];  // closed failure regions (first, last)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const Fam F = A.F;
  const int m = F.m;
  const int C32 = (int)F.C;
  const int gw = blockIdx.x * LV_WARPS + wib;  // global warp index
  const int c0 = gw * 32;
  const int c32 = c0 + lane;
  const bool valid = c32 < C32;  // (warps past the last chain run through with no lanes)
  const int ns32 = (int)F.ns;
  const int base32 = valid ? (int)fam_base(F, c32) : 0;
  // node of position pos: strided families step ns, row-like rows are contiguous (ns = 1)
  auto node = [&](int pos) { return base32 + pos * ns32; };
  const int ntiles = (m + TP - 1) / TP;
  // row-like chains are contiguous rows of m nodes: 16-byte vectors need m % 4 == 0
  const bool vec = ROWLIKE && (m & 3) == 0;

  // ---- tile registers: next (loading), cur (verifying), prev (retiring)
  float pn_[TP], an_[TP];
  double cn_[TP];
  unsigned hn = 0u;
  auto load = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      const bool pr = valid && pos < m;
      pn_[q] = pr ? __ldg(A.p + pos * C32 + c32) : 0.f;
      an_[q] = (pr && pos < m - 1) ? __ldg(A.wf + pos * C32 + c32) : 0.f;
      if (!ROWLIKE) cn_[q] = pr ? __ldg(A.c + node(pos)) : 0.0;
    }
    if (ROWLIKE) {
      if (vec && valid && k0 + TP <= m) {
        const double2* v = reinterpret_cast<const double2*>(A.c + node(k0));
#pragma unroll
        for (int h = 0; h < TP / 2; ++h) {
          const double2 t = __ldg(v + h);
          cn_[2 * h] = t.x;
          cn_[2 * h + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < TP; ++q) cn_[q] = (valid && k0 + q < m) ? __ldg(A.c + node(k0 + q)) : 0.0;
      }
    }
    hn = valid ? (unsigned)A.sg[T * C32 + c32] : 0u;
  };
  // retire-only inputs (G in for MID / LAST, X for LAST) of a tile
  float gr_[TP], xr_[TP];
  auto load_gx = [&](int T) {
    if (ROLE != MID && ROLE != LAST) return;
    const int k0 = T * TP;
    if (vec && valid && k0 + TP <= m) {
      const float4* g = reinterpret_cast<const float4*>(A.Gi + node(k0));
      const float4 g0 = __ldg(g), g1 = __ldg(g + 1);
      gr_[0] = g0.x; gr_[1] = g0.y; gr_[2] = g0.z; gr_[3] = g0.w;
      gr_[4] = g1.x; gr_[5] = g1.y; gr_[6] = g1.z; gr_[7] = g1.w;
      if (ROLE == LAST) {
        const float4* x = reinterpret_cast<const float4*>(A.X + node(k0));
        const float4 x0 = __ldg(x), x1 = __ldg(x + 1);
        xr_[0] = x0.x; xr_[1] = x0.y; xr_[2] = x0.z; xr_[3] = x0.w;
        xr_[4] = x1.x; xr_[5] = x1.y; xr_[6] = x1.z; xr_[7] = x1.w;
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const bool pr = valid && k0 + q < m;
      gr_[q] = pr ? __ldg(A.Gi + node(k0 + q)) : 0.f;
      if (ROLE == LAST) xr_[q] = pr ? __ldg(A.X + node(k0 + q)) : 0.f;
    }
  };

  double zc_[TP], zp_[TP];
  float pc_[TP], ac_[TP], pp_[TP];
  unsigned hc = 0u;

  // ---- lane state: the open candidate segment [i0, .)
  constexpr float FINF = __builtin_huge_valf();
  int i0 = 0;
  double vt = 0.0, tp = 0.0;  // anchors (z at the start) of the open / previous segment
  float Q = 0.f, LO = -FINF, HI = FINF, xrp = 0.f;
  float sL = 0.f;  // side of the open segment's left edge (0: piece start)
  unsigned smask = 0u;        // segment starts marked, bit = pos & 15
  int ff = 0x7fffffff, fl = -1;  // the current failure region [ff, fl]
  int nreg = 0;                   // closed regions in regs_sm
  bool hole = false;          // the open segment has positions no longer retirable
  double zs = 0.0, qs = 0.0;  // retire carry
  double nrm = 0.0;

  // q slots: qsm[wib][slot][lane] as a shared-memory byte offset; slot 16 is a
  // dummy row taking the (unconditional) store of a position that closes nothing
  const unsigned qbase = (unsigned)__cvta_generic_to_shared(&qsm[wib][0][lane]);
  auto qst = [&](int slot, float v) {
    asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(qbase + ((unsigned)slot << 7)), "f"(v) : "memory");
  };
  auto qld = [&](int slot) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(qbase + ((unsigned)slot << 7)) : "memory");
    return v;
  };
  auto verify_tile = [&](int T) {
    const int k0 = T * TP;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int k = k0 + q;
      if (k < m) {  // warp-uniform
        // branch-free: a close and an interior step are both computed and
        // selected, so the warp never diverges here
        const bool last = k == m - 1;
        const double z = zc_[q];
        const float ak = last ? 0.f : ac_[q];
        const float sf = (float)((int)((hc >> q) & 1u) - (int)((hc >> (8 + q)) & 1u));
        vt = (k == i0) ? z : vt;
        Q += (float)(z - vt);
        const float inv = rcp_r<float>(k - i0 + 1);
        const bool piece = last | (ak == 0.f);
        const bool cl = piece | (sf != 0.f);
        const float uR = piece ? 0.f : -sf * ak;  // ceiling (+1): u = -a
        const float xr = (Q - uR) * inv;          // segment value - vt, if it closes here
        const float dx = (xr - xrp) + (float)(vt - tp);
        const bool bad = cl & ((LO > xr + PCB_VTOL) | (xr > HI + PCB_VTOL) | (sL * dx < -PCB_VTOL));
        if (bad | (cl & hole)) {  // rare: failure bookkeeping
          // failure regions: a failure far past the current region closes it
          // (kept in shared memory, up to NREG - 1) and opens a new one
          if (bad) {
            if (ff != 0x7fffffff && i0 > fl + RGAP && nreg < NREG - 1) {
              regs_sm[wib][nreg][lane] = make_int2(ff, fl);
              ++nreg;
              ff = i0;
            } else {
              ff = min(ff, i0);
            }
          }
          fl = max(fl, k);
        }
        const bool mark = cl & !hole;             // (a hole's head is the repair's)
        qst(mark ? (i0 & 15) : 16, -xr);          // q = z(i0) - x
        smask |= (unsigned)mark << (i0 & 15);
        hole = hole & !cl;
        xrp = cl ? xr : xrp;
        tp = cl ? vt : tp;
        sL = cl ? (piece ? 0.f : sf) : sL;
        LO = cl ? -FINF : fmaxf(LO, (Q - ak) * inv);
        HI = cl ? FINF : fminf(HI, (Q + ak) * inv);
        Q = cl ? uR : Q;
        i0 = cl ? k + 1 : i0;
      }
    }
  };

  auto retire_tile = [&](int T) {
    const int k0 = T * TP;
    float gout[TP], xout[TP];
    double cout[TP];
    double na = 0.0, nb = 0.0;
    const bool open_here = i0 < min(k0 + TP, m);  // the open segment reaches into this tile
    if (open_here && valid && !hole) {  // a hole opens: a failure region from i0
      if (ff != 0x7fffffff && i0 > fl + RGAP && nreg < NREG - 1) {
        regs_sm[wib][nreg][lane] = make_int2(ff, fl);
        ++nreg;
        ff = i0;
      } else {
        ff = min(ff, i0);
      }
      fl = max(fl, i0);
      hole = true;
    }
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      double& nq = (q & 1) ? nb : na;
      const bool em = valid && pos < m && pos < i0;
      float p32 = __int_as_float(0x7fc00000);  // NaN: not emitted (repair writes it)
      double d = 0.0;
      if (em) {
        if ((smask >> (pos & 15)) & 1u) {
          zs = zp_[q];
          qs = (double)qld(pos & 15);
        }
        p32 = (float)((zp_[q] - zs) + qs);
        d = (double)p32 - (double)pp_[q];
        nq = __fma_rn(d, d, nq);
      }
      if (valid && pos < m) A.po[pos * C32 + c32] = p32;
      if (ROLE == FIRST) {
        gout[q] = (float)d;
      } else if (ROLE == MID) {
        gout[q] = (float)((double)gr_[q] + d);
      } else {
        const float g32 = (float)((double)gr_[q] + d);
        const double g = (double)g32;
        const double xn = (double)xr_[q] - g;
        xout[q] = (float)xn;
        const double dcv = (xn - g) * A.inv_r;
        cout[q] = (zp_[q] - (double)pp_[q]) + dcv;  // c_old = z - p_old
        if (em) nq = __fma_rn(dcv, __fma_rn(A.rd, dcv, g + g), nq);
      }
      // (non-emitted positions get no fused update; the repair writes them)
      if (!ROWLIKE && em) {
        const int nd = node(pos);
        if (ROLE == FIRST || ROLE == MID) A.G[nd] = gout[q];
        else {
          A.Xo[nd] = xout[q];
          A.co[nd] = cout[q];
        }
      }
    }
    smask &= ~(0xffu << (k0 & 15));
    if (ROWLIKE && valid) {
      const bool full = vec && k0 + TP <= m && i0 >= k0 + TP;
      if (full) {
        if (ROLE == FIRST || ROLE == MID) {
          float4* g = reinterpret_cast<float4*>(A.G + node(k0));
          g[0] = make_float4(gout[0], gout[1], gout[2], gout[3]);
          g[1] = make_float4(gout[4], gout[5], gout[6], gout[7]);
        } else {
          float4* x = reinterpret_cast<float4*>(A.Xo + node(k0));
          x[0] = make_float4(xout[0], xout[1], xout[2], xout[3]);
          x[1] = make_float4(xout[4], xout[5], xout[6], xout[7]);
          double2* cc = reinterpret_cast<double2*>(A.co + node(k0));
#pragma unroll
          for (int h = 0; h < TP / 2; ++h) cc[h] = make_double2(cout[2 * h], cout[2 * h + 1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < TP; ++q) {
          const int pos = k0 + q;
          if (pos < m && pos < i0) {
            if (ROLE == FIRST || ROLE == MID) A.G[node(pos)] = gout[q];
            else {
              A.Xo[node(pos)] = xout[q];
              A.co[node(pos)] = cout[q];
            }
          }
        }
      }
    }
    nrm += na + nb;
  };

  // ---- pipeline: load T+1 | verify T | retire T-1
  load(0);
  for (int T = 0; T < ntiles; ++T) {
    // the loaded tile becomes current: z = p + c
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      pc_[q] = pn_[q];
      ac_[q] = an_[q];
      zc_[q] = (double)pn_[q] + cn_[q];
    }
    hc = hn;
    if (T + 1 < ntiles) load(T + 1);
    if (T > 0) load_gx(T - 1);
    verify_tile(T);
    if (T > 0) retire_tile(T - 1);
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      zp_[q] = zc_[q];
      pp_[q] = pc_[q];
    }
  }
  load_gx(ntiles - 1);
  retire_tile(ntiles - 1);

  // ---- repair of the chains whose candidate failed (or left a hole): up to
  // RROWS lanes at a time through the staged window, the rest (and any repair
  // that leaves its window) from global memory
  __syncwarp();
  const bool dirty = valid && ff != 0x7fffffff;
  const unsigned dall = __ballot_sync(0xffffffffu, dirty);
#ifndef PCB_NO_REPAIR  // timing experiments only: results are wrong without the repair
  if (dall) {
    unsigned left = dall;
    while (left) {
      unsigned sel = 0u, t = left;
      for (int r = 0; r < RROWS && t; ++r) {
        const unsigned lb = t & (0u - t);
        sel |= lb;
        t ^= lb;
      }
      if ((sel >> lane) & 1u) {
        const int row = __popc(sel & ((1u << lane) - 1u));
        for (int r = 0; r <= nreg; ++r) {
          const int2 rg = r < nreg ? regs_sm[wib][r][lane] : make_int2(ff, fl);
          double dn = 0.0;
          if (repair_fast<ROLE, ROWLIKE>(A, c32, base32, rg.x, rg.y, rwin[wib], row, &dn)) {
            nrm += dn;
          } else {
            PCB_REP(4);
            nrm += repair_lane<ROLE, ROWLIKE>(A, c32, base32, rg.x, rg.y, -1);
          }
        }
      }
      left &= ~sel;
      __syncwarp();
    }

  }
#endif
  const int nch = __popc(dall);
  if (lane == 0 && nch && A.vcount) atomicAdd(A.vcount, nch);

  // ---- step-norm partial: the scan's slot of these 32 chains (one per warp)
  const double v = warp_sum(nrm);
  const int nslots = ((C32 + WARPS * 32 - 1) / (WARPS * 32)) * WARPS;
  if (lane == 0 && gw < nslots) A.parts[gw] = v;
}

}  // namespace fast
}  // namespace pcb
