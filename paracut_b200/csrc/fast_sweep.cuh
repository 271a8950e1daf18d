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
// offsets)/len.  Slopes use a MUFU reciprocal of the small integer offset
// refined by one fp64 Newton step.  Closing a segment is O(1): the lane writes
// q = z_i0 - fill at the segment start and sets a start bit; per-node
// outputs are produced by a lockstep retire pass over whole tiles
// (p_new = (z_j - z_start) + q) and written back coalesced.  A lane whose
// anchor falls behind the ring reads and writes those positions in global
// memory; retirement is masked by each lane's emitted frontier.
#pragma once
#include <cuda.h>  // CUtensorMap
#include <type_traits>

namespace pcb {
namespace fast {

#ifdef PCB_COUNT
// diagnostics build only: warp trips, lane gates, bends, tiles issued, tiles retired
__device__ unsigned long long g_count[8];
#define PCB_CNT(i, v) ((void)(lane == 0 ? atomicAdd(&g_count[i], (unsigned long long)(v)) : 0ull))
#else
#define PCB_CNT(i, v) ((void)0)
#endif

constexpr int TP = 8;          // positions per tile
constexpr int NT = 4;          // tiles in the ring
constexpr int RL = TP * NT;    // ring length (positions)
#ifndef PCB_SWEEP_WARPS
#define PCB_SWEEP_WARPS 2
#endif
constexpr int WARPS = PCB_SWEEP_WARPS;  // warps per block (2 x 16.5 KB rings, 6 blocks/SM; 1: 13 warps/SM, slower; 4: -1-2 %)
constexpr int MWARPS = 4;               // warps per block of the merge kernel
#ifndef PCB_SCAN_UNROLL
#define PCB_SCAN_UNROLL 2  // trips per exit vote (lag-free rounds)
#endif
#ifndef PCB_SCAN_KEEP
#define PCB_SCAN_KEEP 20  // a round ends when at most this many lanes still have data (16-20 flat)
#endif
static_assert(RL == 32, "swizzle and start masks assume a 32-position ring");
static_assert(TP == 8, "mode-B lane mapping assumes 8-position tiles");

enum Role { FIRST = 0, MID = 1, LAST = 2, SHADOW = 3 };

// ST: storage type of the family state, weights, accumulator and primal --
// float for the fp32-state mode, double for the fp64 split mode (f64s).
template <class ST>
struct ArgsT {
  Fam F;
  ST* p;            // family state, interleaved [pos][C]
  const ST* wf;     // family weights, interleaved [pos][C]
  double* c;        // drift (natural node layout)
  ST* G;            // accumulator of p_new - p_old over families (natural)
  ST* X;            // primal x = w - sum_j p_j (natural)
  double* y;        // SHADOW output (natural)
  double inv_r, rd;
  double* parts;    // per-block monitor partials
  // intra-chain split (nullptr: whole chains).  Unit (chain c, block b) runs
  // the string from the merge point of block b (merge[b*C + c]; block 0 starts
  // at the chain start) up to the next block's merge point.  Code:
  // pos * 4 + (touch + 1), touch -1 floor / +1 ceiling / 0 piece start; -1 none.
  const int* merge;
  int nb;
  int export_g;     // LAST: also store the per-node g = sum_j d_j (fp32) in G
  // Double-buffered step (nullptr: in place).  The sweep reads p, c, X and
  // Gi and writes po, co, Xo and G, so its inputs stay intact for the local
  // repair of a verified sweep (VER) and for any other reader of the step.
  ST* po;           // new family state
  double* co;       // LAST: new drift
  ST* Xo;           // LAST: new primal
  const ST* Gi;     // MID / LAST: accumulator in (G is the accumulator out)
  // Segment hints (SCAN writes, VER reads): per tile of TP positions one
  // uint16 per chain, [tile][C]; bit q: the left boundary of position
  // tile*TP+q is a ceiling touch (x rises), bit 8+q: a floor touch (x falls).
  uint16_t* sg;
  const int* vmode; // device mode word of this family: 1 = VER sweeps, else SCAN
  int* vcount;      // SCAN: chains whose hints changed; VER: chains repaired
};

using Args = ArgsT<float>;
using Args64 = ArgsT<double>;

// in-place defaults for the double-buffer fields
template <class ST>
inline void args_inplace(ArgsT<ST>& a) {
  if (!a.po) a.po = a.p;
  if (!a.co) a.co = a.c;
  if (!a.Xo) a.Xo = a.X;
  if (!a.Gi) a.Gi = a.G;
}

// TMA descriptors of one family launch.  Strided families (cols, 3D y / z)
// whose warps' 32 chains are 32 consecutive nodes at every position load
// their ring tiles -- p_j and the weights (interleaved [pos][C]) and the
// drift c (natural layout) -- as (32 chains x 8 positions) boxes, one
// instruction per array per tile, completing on a per-tile mbarrier.
//
// Row families (2D rows, 3D x lines: a chain is one contiguous row of the
// node arrays) with row = 1: p_j and the weights as above, and the drift as
// a (8 positions x 32 rows) box of the natural layout, 64-B swizzled, landing
// in the tile's z slots as [row][pos]; to_z transposes it to the ring's
// [pos][lane] layout (k_sweep<..., RT = true>).
struct Maps {
  CUtensorMap p, a, c;
  int tma;      // 1: use the maps (else cp.async per lane)
  int c3;       // the c map is 3D: (x = c % cdiv, pos, c / cdiv)
  int row;      // row family: the c map is (pos, row), SWIZZLE_64B
};

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(unsigned dst, const CUtensorMap* map, int x, int y,
                                      unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma3d(unsigned dst, const CUtensorMap* map, int x, int y, int z,
                                      unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// p' of a whole tile as one bulk tensor store from the ring's p slots (the
// row-TMA FIRST sweep)
__device__ __forceinline__ void tma2d_store(const CUtensorMap* map, int x, int y, unsigned src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
               "cp.async.bulk.commit_group;\n" ::"l"(map), "r"(x), "r"(y), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// Predicated copies (no zero fill): slots of positions past the chain end or
// of lanes without a chain are never read, so skipping them is enough and
// avoids the src-size arithmetic of the zero-filling form.
__device__ __forceinline__ void cp4(void* dst, const void* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(s),
      "l"(src), "r"((int)pred));
}
__device__ __forceinline__ void cp8(void* dst, const void* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(s),
      "l"(src), "r"((int)pred));
}
// one state / weight element (4 or 8 bytes)
template <class T>
__device__ __forceinline__ void cp_elem(void* dst, const T* src, bool pred) {
  if (sizeof(T) == 8) cp8(dst, src, pred);
  else cp4(dst, src, pred);
}
// unpredicated forms with a 32-bit shared address (the whole-tile issue path)
__device__ __forceinline__ void cp4s(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp8s(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void l2_prefetch(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
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

// 1/d for a small positive integer d: MUFU approximation + one fp64 Newton step
// (relative error ~2^-46, plenty for slope comparisons and segment values).
__device__ __forceinline__ double rcp_small(int di, double dd) {
  float r32;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r32) : "f"((float)di));
  const double r = (double)r32;
  return __fma_rn(r, __fma_rn(-dd, r, 1.0), r);
}

template <class Rt>
__device__ __forceinline__ Rt rcp_r(int di);
template <>
__device__ __forceinline__ float rcp_r<float>(int di) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)di));
  return r;
}
template <>
__device__ __forceinline__ double rcp_r<double>(int di) {
  return rcp_small(di, (double)di);
}

// ring index of (lane row l, position pos): (l << 5) | ((pos & 31) ^ l), written
// as one masked XOR with (l << 5 | l) so it is a single LOP3 (the scan is
// ALU-pipe bound)
__device__ __forceinline__ int rix(int l, int pos) { return (pos & (RL - 1)) ^ ((l << 5) | l); }

// [pos][lane] ring index ((pos & 31) << 5) | l as one LOP3 on pos << 5 (the
// shift is an IMAD on the FMA pipe; the scan is ALU-pipe bound)
__device__ __forceinline__ int pix(int l, int pos) {
  int r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(pos << 5), "r"((RL - 1) << 5), "r"(l));
  return r;
}

template <int ROLE, class ST = float>
__host__ __device__ constexpr int ring_bytes_host() {
  // rz f64, rp / ra one state element each (an fp32 SHADOW keeps its fp64
  // segment values split over the dead rp / ra slots), + NT tile mbarriers,
  // padded to 512 B so every warp's tile slots stay aligned to the 64-B
  // swizzle atom of the row families' drift boxes
  return (32 * RL * (8 + 2 * (int)sizeof(ST)) + 128 + 511) & ~511;
}

// lagging-lane accessors (positions below the ring), kept out of line
template <class ST>
__device__ __noinline__ double z_global(const ArgsT<ST>& A, int64_t fi, int64_t nd) {
  return (double)A.p[fi] + A.c[nd];
}
template <class ST>
__device__ __noinline__ double a_global(const ArgsT<ST>& A, int64_t fi) { return (double)A.wf[fi]; }

// monitor terms with explicit FMAs (the TU is built with -fmad=false for the
// exact path; the fp32-state monitor has no bitwise contract)
__device__ __forceinline__ double nrm_d(double d, double acc) { return __fma_rn(d, d, acc); }
// LAST role: 2 dcv g + r dcv^2 = dcv (2 g + r dcv)
__device__ __forceinline__ double nrm_last(double dcv, double g, double rd, double acc) {
  return __fma_rn(dcv, __fma_rn(rd, dcv, g + g), acc);
}

template <int ROLE, class ST>
__device__ __noinline__ double finish_global(const ArgsT<ST>& A, int64_t fi, int64_t nd, double fill) {
  const ST pold = A.p[fi];
  const double cz = A.c[nd];
  const double pn = ((double)pold + cz) - fill;
  if (ROLE == SHADOW) {
    A.y[nd] = pn;
    return 0.0;
  }
  const ST p32 = (ST)pn;
  const double d = (double)p32 - (double)pold;
  double nrm = nrm_d(d, 0.0);
  A.po[fi] = p32;
  if (ROLE == FIRST) {
    A.G[nd] = (ST)d;
  } else if (ROLE == MID) {
    A.G[nd] = (ST)((double)A.Gi[nd] + d);
  } else {
    const ST g32 = (ST)((double)A.Gi[nd] + d);
    const double g = (double)g32;
    const double xn = (double)A.X[nd] - g;
    A.Xo[nd] = (ST)xn;
    const double dcv = (xn - g) * A.inv_r;
    A.co[nd] = cz + dcv;
    if (A.export_g) A.G[nd] = g32;
    nrm = nrm_last(dcv, g, A.rd, nrm);
  }
  return nrm;
}

struct Spec {
  int i0, pe, k, c0x, f0x;
  double t, skr, cs, fs, Lc, Lf;
  bool fresh;
};

template <class ZA>
__device__ __forceinline__ void spec_next_bend(Spec& S, int m, const ZA& za, int* bk_out,
                                               int* bt_out, double* xv_out = nullptr) {
  for (;;) {
    const int kp = S.k;
    double zabs, av;
    za(kp, &zabs, &av);
    S.k = kp + 1;
    if (S.fresh) {
      S.t = zabs;
      S.fresh = false;
    }
    S.skr += zabs - S.t;
    const bool inner = S.k < m;
    const double rk = inner ? av : 0.0;
    if (inner && av == 0.0) S.pe = S.k;
    const double inv = rcp_r<double>(S.k - S.i0);
    S.Lc += S.cs;
    S.Lf += S.fs;
    const double u = S.skr + rk;
    if (S.c0x < 0 || u <= S.Lc) {
      S.c0x = S.k;
      S.cs = u * inv;
      S.Lc = u;
    }
    int bk = -1, bt = 0;
    double fill = 0.0;
    if (S.f0x >= 0 && S.cs < S.fs) {
      bk = S.f0x; bt = -1; fill = S.fs;
    } else {
      const double l = S.skr - rk;
      if (S.f0x < 0 || l >= S.Lf) {
        S.f0x = S.k;
        S.fs = l * inv;
        S.Lf = l;
      }
      if (S.fs > S.cs) {
        bk = S.c0x; bt = 1; fill = S.cs;
      } else if (S.k == S.pe) {
        if (S.c0x != S.pe && S.Lc < S.skr) {
          bk = S.c0x; bt = 1; fill = S.cs;
        } else if (S.f0x != S.pe && S.Lf > S.skr) {
          bk = S.f0x; bt = -1; fill = S.fs;
        } else {
          bk = S.pe; bt = 0; fill = S.skr * inv;
        }
      }
    }
    if (bk >= 0) {
      if (xv_out) *xv_out = S.t + fill;  // the closed segment's prox value
      double ab = 0.0;
      if (bt != 0) {
        double dz;
        za(bk - 1, &dz, &ab);
      }
      const bool piece_end = bk == S.pe;
      S.i0 = S.k = bk;
      S.fresh = true;
      S.skr = piece_end ? 0.0 : -(double)bt * ab;
      if (piece_end) S.pe = m;
      S.c0x = S.f0x = -1;
      S.cs = S.fs = S.Lc = S.Lf = 0.0;
      *bk_out = bk;
      *bt_out = piece_end ? 0 : bt;
      return;
    }
  }
}


// ---------------------------------------------------------------------------
// Local repair of a verified chain whose candidate failed somewhere in
// [ff, fl] (VER sweep; everything from global memory, inputs intact in the
// double-buffered step).  The true string is localised between two points:
//  * q_L <= ff: the first common bend of the two strings anchored at the
//    floor and at the ceiling of a gate g < ff (taut strings to a common end
//    never cross, so the true one passes there too -- the merge-point argument
//    of k_merge), accepted if the candidate has the same touch there (then the
//    candidate before q_L, which passed every check, is the true solution);
//    g moves back until that holds (g = 0, the chain start, always does);
//  * the taut string from q_L is exact; it is emitted bend by bend until a
//    bend past fl where the candidate has the same touch -- from there on the
//    candidate (checked, with a true left dual) is the true solution.
// The emitted range replaces what the sweep wrote; the step-norm partial is
// corrected by the difference.  Hints of the range are rewritten.
template <int ROLE, bool ROWLIKE>
__device__ __noinline__ double repair_lane(const Args& A, int c32, int base32, int ff, int fl,
                                           int emit_hi) {
  const Fam& F = A.F;
  const int m = F.m, C32 = (int)F.C;
  const int ns32 = (int)F.ns, zz32 = (int)F.zz, ph32 = F.phase;
  auto node = [&](int pos) {
    return ROWLIKE ? base32 + pos * ns32 + zz32 * ((pos + ph32) & 1) : base32 + pos * ns32;
  };
  auto za = [&](int pos, double* z, double* a) {
    const int fi = pos * C32 + c32;
    *z = (double)A.p[fi] + A.c[node(pos)];
    *a = pos < m - 1 ? (double)A.wf[fi] : 0.0;
  };
  auto cand = [&](int e) {  // hinted side of edge e (+1 ceiling, -1 floor, 0 none)
    const unsigned w = A.sg[(e / TP) * C32 + c32];
    const int q = e % TP;
    return (int)((w >> q) & 1u) - (int)((w >> (8 + q)) & 1u);
  };
  // 1. q_L
  int qL = 0, qt = 0;
  for (int delta = 4;; delta *= 2) {
    const int g = ff - delta;
    if (g <= 0) break;
    const double ag = (double)A.wf[(g - 1) * C32 + c32];
    if (ag == 0.0) {  // a piece start: a true point for every string
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
      if (pf == pu && tf == tu) {
        q = pf;
        t = tf;
        break;
      }
      if (min(pf, pu) > ff) break;
      if (pf <= pu) spec_next_bend(Fs, m, za, &pf, &tf);
      else spec_next_bend(Us, m, za, &pu, &tu);
    }
    if (q >= 0 && q <= ff && (t == 0 || cand(q - 1) == t)) {
      qL = q;
      qt = t;
      break;
    }
  }
  // 2. the exact string from q_L
  double nrm = 0.0;
  const double a0 = (qL > 0 && qt != 0) ? (double)A.wf[(qL - 1) * C32 + c32] : 0.0;
  Spec S{qL, m, qL, -1, -1, 0.0, -(double)qt * a0, 0.0, 0.0, 0.0, 0.0, true};
  int s0 = qL;
  for (;;) {
    int bk, bt;
    double xv;
    spec_next_bend(S, m, za, &bk, &bt, &xv);
    const bool stop = bk >= m || (bk - 1 > fl && (bt == 0 || cand(bk - 1) == bt));
    for (int j = s0; j < bk; ++j) {
      const int fi = j * C32 + c32, nd = node(j);
      const float pin = A.p[fi];
      const double cz = A.c[nd];
      const float p32 = (float)(((double)pin + cz) - xv);
      const double d = (double)p32 - (double)pin;
      double r = d * d;
      // the sweep emitted (and counted) this position: below emit_hi, or (the
      // lean sweep, emit_hi < 0) wherever it did not leave a NaN hole
      const bool was = emit_hi >= 0 ? j < emit_hi : !isnan(A.po[fi]);
      const double dw = was ? (double)A.po[fi] - (double)pin : 0.0;
      if (was) r -= dw * dw;
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
    }
    // hints of the emitted edges: interior, then the bend's touch
    for (int e = s0; e < bk && e < m - 1; ++e) {
      const int side = e == bk - 1 ? bt : 0;
      uint16_t* wp = A.sg + (e / TP) * C32 + c32;
      const int q = e % TP;
      unsigned w = *wp & ~((1u << q) | (1u << (8 + q)));
      w |= side > 0 ? (1u << q) : (side < 0 ? (1u << (8 + q)) : 0u);
      *wp = (uint16_t)w;
    }
    s0 = bk;
    if (stop) break;
  }
  return nrm;
}

// RT: a row family fed by TMA (Maps::row); it runs the strided families'
// [pos][lane] ring (ROWLIKE = false), with the drift box transposed in to_z
// and its node-order outputs stored as per-lane vectors along the row.
// XG: the LAST role also stores its per-node g = sum_j d_j in G (sharded
// runs, PCB_STEP_EXPORT_G); compiled in, so the plain step carries no test
template <int ROLE, bool ROWLIKE, bool VER = false, class ST = float, bool RT = false,
          bool XG = false>
__global__ void __launch_bounds__(WARPS * 32)
    k_sweep(const __grid_constant__ ArgsT<ST> A, const __grid_constant__ Maps M) {
  static_assert(!VER || sizeof(ST) == 4, "verified sweeps run in the fp32-state mode");
  static_assert(!RT || (!ROWLIKE && !VER && (ROLE == FIRST || ROLE == SHADOW)),
                "row-TMA sweeps: first family or shadow only");
  static_assert(!XG || ROLE == LAST, "only the LAST role exports g");
  constexpr bool S64 = sizeof(ST) == 8;  // fp64 state (f64s): fp64 scan, fp64 ring slots
  // TMA store of p' (UTMASTG): pays in the row-TMA FIRST sweep, whose retire has
  // few other stores (cfg4 x 0.158 -> 0.154 ms, cfg5 0.921 -> 0.889); the MID /
  // LAST sweeps lose 4-6 % with it, with or without the wait before the
  // slot's reload (profiles/r2/ab_tma_store.txt; PCB_TMA_STORE_ALL: every
  // TMA-fed role)
#ifdef PCB_TMA_STORE_ALL
  constexpr bool TST = !ROWLIKE && !VER && ROLE != SHADOW;
#else
  constexpr bool TST = RT && ROLE == FIRST;
#endif
  extern __shared__ __align__(1024) unsigned char smem_raw[];  // TMA boxes land 512-B aligned
  // device-side choice between the two sweeps of a family (both are launched;
  // the one the mode word does not select returns at once)
  if (A.vmode != nullptr && ((*A.vmode == 1) != VER)) return;
  // the next (programmatically launched) sweep may start once every block of
  // this one has started: it fills this grid's tail
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Fam F = A.F;
  const int64_t c0 = ((int64_t)blockIdx.x * WARPS + wib) * 32;
  double nrm = 0.0;

  unsigned char* base = smem_raw + (size_t)wib * ring_bytes_host<ROLE, ST>();
  double* rz = reinterpret_cast<double*>(base);
  ST* rp = reinterpret_cast<ST*>(base + 32 * RL * 8);
  ST* ra = rp + 32 * RL;
  // ring layout: [pos][lane] rows of 32 for strided families (every access is
  // lane-contiguous, and a (positions x 32 chains) box is one contiguous
  // block); row-like families keep [lane][pos] with the XOR swizzle that
  // their 8-lanes-along-a-row loads need
  auto rx = [](int l, int pos) { return ROWLIKE ? rix(l, pos) : pix(l, pos); };
  const unsigned rz_s = (unsigned)__cvta_generic_to_shared(rz);
  const unsigned rp_s = (unsigned)__cvta_generic_to_shared(rp);
  const unsigned ra_s = (unsigned)__cvta_generic_to_shared(ra);
  // ring index of position k0 + q of a tile (k0 a multiple of TP, q < TP): in
  // the [pos][lane] layout the tile's rows are 32 apart with no wrap inside a
  // tile, so the per-q offset folds into the shared-memory address immediate
  // (row-like: k0 is a multiple of TP = 8, so slot (k0 + q) ^ swizzle = slot(k0) ^ q)
  auto tix = [&](int k0, int q) { return ROWLIKE ? (rix(lane, k0) ^ q) : pix(lane, k0) + (q << 5); };
  const bool use_tma = RT || (!ROWLIKE && M.tma);  // (RT: the host builds its maps)
  unsigned long long* mbar =
      reinterpret_cast<unsigned long long*>(base + 32 * RL * (8 + 2 * sizeof(ST)));

  const bool warp_live = c0 < F.C;
  const int nvalid = warp_live ? (int)min((int64_t)32, F.C - c0) : 0;
  const bool valid = lane < nvalid;
  const int64_t c = c0 + lane;
  const int m = F.m;
  const int64_t C = F.C;
  // 32-bit index arithmetic: pcb_create keeps n below 2^31, so every node
  // index and interleaved index pos * C + c fits (half the address IMADs)
  const int C32 = (int)F.C, c32 = (int)c;
  const int ns32 = (int)F.ns, zz32 = (int)F.zz, ph32 = F.phase;
#ifdef PCB_DIV64
  const int base32 = valid ? (int)fam_base(F, c) : 0;
#else
  // (n < 2^31: chain index, cdiv and the base fit in 32 bits; the 64-bit
  // division of fam_base is ~100 instructions)
  const unsigned cdv = (unsigned)F.cdiv;
  const unsigned cq = (unsigned)c32 / cdv, cr = (unsigned)c32 - cq * cdv;
  const int base32 = valid ? (int)(cq * (unsigned)F.chi + cr * (unsigned)F.clo) : 0;
#endif
  // zig-zag families are row-like, so strided families have no zig-zag term
  auto node = [&](int b, int pos) {
    return ROWLIKE ? b + pos * ns32 + zz32 * ((pos + ph32) & 1) : b + pos * ns32;
  };
  // mode B (row-like families): lane works on chains 8*(lane/8) + ib, ib < 8;
  // their node bases are fixed for the whole launch
  int bB[8];
  if (ROWLIKE) {
#pragma unroll
    for (int ib = 0; ib < 8; ++ib) bB[ib] = __shfl_sync(0xffffffffu, base32, ((lane >> 3) << 3) + ib);
  }

  // this unit's range [start, stop) of the chain and the tube touches there;
  // the string is forced through the next unit's merge point at gate `stop`
  // (a true point of the string), so a unit never reads past its range and
  // units of one chain never race on the in-place state
  int start = 0, stop = m, stouch = 0, etouch = 0;
  bool has = valid;
  if (A.merge != nullptr && valid) {
    const int b = blockIdx.y;
    if (b > 0) {
      const int e = A.merge[(int64_t)b * C + c];
      has = e >= 0;
      start = e >> 2;
      stouch = (e & 3) - 1;
    }
    for (int b2 = b + 1; b2 < A.nb; ++b2) {
      const int e = A.merge[(int64_t)b2 * C + c];
      if (e >= 0) {
        stop = e >> 2;
        etouch = (e & 3) - 1;
        break;
      }
    }
    if (!has || start >= stop) {
      has = false;
      start = stop = 0;
    }
  }
  if (!has) start = stop = 0;  // lanes without a unit (past the last chain) are finished
  const int rlo = __reduce_min_sync(0xffffffffu, has ? start : 0x7fffffff);
  const int rhi = __reduce_max_sync(0xffffffffu, has ? stop : 0);
  const int t_first = rlo == 0x7fffffff ? 0 : rlo / TP;
  const int ntiles = (rhi + TP - 1) / TP;
  const int ntile_sg = (m + TP - 1) / TP;  // hint words per chain

  // ---- lane state: stackless taut string in the anchor frame.  The scan runs
  // in R = fp32 for the in-place roles (values are taken relative to the
  // anchor's z, so they stay O(|p| + local drift) and fp32 keeps ~1e-7 of
  // them) and in fp64 for the shadow, whose output feeds the certificates.
  using R = typename std::conditional<ROLE == SHADOW || S64, double, float>::type;
  // fp32-state SHADOW: its fp64 segment values are split over the rp / ra slots
  constexpr bool QSPLIT = ROLE == SHADOW && !S64;
  // a lane is finished when its anchor reaches `stop` (lanes without a unit
  // have start = stop = 0); it is never active again, and its whole range
  // counts as emitted
  int i0 = start, k = start, c0x = -1, f0x = -1;
  // weights of the edges left of the ceiling / floor points (a(c0x - 1),
  // a(f0x - 1)): a bend's restart value without a ring read
  R acx = R(0), afx = R(0);
  int ixi0 = rx(lane, start);  // ring index of the anchor i0
  double t = 0.0;          // z at the anchor: scan values are z - t
  R skr = R(0);            // running sum of (z - t) minus the anchor value
  // Cone state.  "No ceiling / floor point yet" (a fresh anchor) is Lc = +inf,
  // Lf = fs = -inf: the next gate's cone tests then accept its tube points
  // and no bend test can fire, without index sentinels in the trip.
  constexpr R RINF = R(__builtin_huge_valf());
  R cs = R(0), Lc = RINF;  // min slope to the ceiling points; cs * (k - i0)
  R fs = -RINF, Lf = -RINF;  // max slope to the floor points; fs * (k - i0)
  unsigned smask = 0u;        // segment starts inside the ring (bit = slot)
  double zs = 0.0, qs = 0.0;  // retire carry: z at the current segment start, q there
  // Segment hints (SCAN writes them for the next iteration's VER sweep): the
  // side of edge e is the sign of the jump between the segment values around
  // it, found at retire time from consecutive segment starts.  Bit 7 + q of
  // hup / hdn is edge k0 + q - 1 of the tile being retired (its first bit is
  // the previous tile's last edge, so a tile's word is stored one retire later).
#ifdef PCB_NO_HINT_WRITE  // experiment: scans without hint writes
  const bool SGW = false;
#else
  // (hints are written only by the scan right before a verified probe: mode 2)
  const bool SGW = !VER && ROLE != SHADOW && A.sg != nullptr && A.vmode && *A.vmode == 2;
#endif
  double xprev = __longlong_as_double(0x7ff8000000000000ll);  // NaN: no previous segment
  unsigned hup = 0u, hdn = 0u;
  unsigned hold_prev = 0u, hold_cur = 0u;  // hint words before this iteration (change count)
  bool hchanged = false;

  // retire-only inputs prefetched into registers (G for MID/LAST, X for LAST)
  ST gpre[TP], xpre[TP];
  int pre_tile = -1;

  int t_lo = t_first, t_ld = t_first, t_rdy = t_first;
#ifdef PCB_DIV64
  const int cx0 = (int)(c0 % F.cdiv), co0 = (int)(c0 / F.cdiv);  // TMA box origin of c
#else
  const int co0 = (int)((unsigned)c0 / (unsigned)F.cdiv);  // TMA box origin of c
  const int cx0 = (int)((unsigned)c0 - (unsigned)co0 * (unsigned)F.cdiv);
#endif
  if (use_tma && warp_live) {
    if (lane == 0) {
      for (int u = 0; u < NT; ++u) mbar_init((unsigned)__cvta_generic_to_shared(&mbar[u]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
  }
  // tile T has landed (TMA: its mbarrier; cp.async: all but the newer groups)
  auto land = [&](int T) {
    if (use_tma) {
      const int u = T - t_first;
      mbar_wait((unsigned)__cvta_generic_to_shared(&mbar[u & (NT - 1)]), (unsigned)((u / NT) & 1));
    } else {
      cp_wait(t_ld - T - 1);
    }
    __syncwarp();
  };
  if (has && start > 0 && stouch != 0)  // anchored on a tube touch: skr = -touch * a(start-1)
    skr = (R)(-(double)stouch * (double)A.wf[((start - 1) * C32 + c32)]);
  // end value offset at `stop`: the string ends at S_stop + touch * a(stop-1)
  const R eoff = (has && stop < m && etouch != 0)
                     ? (R)((double)etouch * (double)A.wf[((stop - 1) * C32 + c32)]) : R(0);

  unsigned long long sw = 0ull;  // VER: hint words of the issued tiles (16 bits per slot T & 3)
  auto issue = [&](int T) {
    const int k0 = T * TP;
    PCB_CNT(3, 1);
    if (VER && valid && T < ntile_sg) {
      const unsigned sh = (unsigned)(T & (NT - 1)) * 16u;
      sw = (sw & ~(0xffffull << sh)) | ((unsigned long long)A.sg[T * C32 + c32] << sh);
    }
    // (row-like families only: the strided families' retire inputs are one
    // 128-byte line per position and array, and their register prefetch a
    // round ahead hides DRAM by itself -- cfg4 z 0.1729 -> 0.1696 ms without)
    if (ROWLIKE && (ROLE == MID || ROLE == LAST)) {
      // pull the tile's retire-only inputs (G, X: natural layout) towards L2
      // now, so the register prefetch a round before retirement hits L2
      if (valid && k0 < m) {  // each lane: its chain's 8 positions
        l2_prefetch(A.Gi + node(base32, k0));
        if (ROLE == LAST) l2_prefetch(A.X + node(base32, k0));
      }
    }
    if (use_tma) {  // one elected lane moves the three (8 x 32) boxes of the tile
      if (lane == 0) {
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&mbar[(T - t_first) & (NT - 1)]);
        const int slot = (T & (NT - 1)) * TP * 32;
#ifndef PCB_NO_PROXY_FENCE  // (experiment knob: the fence's cost)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // ring was read generically
#endif
        if (TST) bulk_wait_read();  // this slot's p' store (issued by this lane) has read the ring
        mbar_expect(bar, TP * 32 * (2 * sizeof(ST) + 8));
        tma2d((unsigned)__cvta_generic_to_shared(rp + slot), &M.p, (int)c0, k0, bar);
        tma2d((unsigned)__cvta_generic_to_shared(ra + slot), &M.a, (int)c0, k0, bar);
        if (RT)  // (8 positions x 32 rows) of the natural drift, rows = the warp's chains
          tma2d((unsigned)__cvta_generic_to_shared(rz + slot), &M.c, k0, (int)c0, bar);
        else if (M.c3)
          tma3d((unsigned)__cvta_generic_to_shared(rz + slot), &M.c, cx0, k0, co0, bar);
        else
          tma2d((unsigned)__cvta_generic_to_shared(rz + slot), &M.c, (int)c0, k0, bar);
      }
      return;
    }
    if (k0 + TP < m && nvalid == 32) {
      // whole tile of a full warp (the usual case): every position has a weight
      // and every lane a chain, so no per-copy predicates; shared addresses are
      // a per-tile base XOR / + an immediate (the ring rows of a tile: row-like
      // slot (k0 + q) ^ swizzle = slot(k0) ^ q, strided rows 32 slots apart)
      const unsigned bx = ROWLIKE ? (unsigned)rix(lane, k0) : (unsigned)pix(lane, k0);
      const unsigned P0 = rp_s + bx * (unsigned)sizeof(ST), A0 = ra_s + bx * (unsigned)sizeof(ST);
      const unsigned Z0 = rz_s + bx * 8u;
      const int fi0 = k0 * C32 + c32;
      const ST* const gp = A.p;
      const ST* const ga = A.wf;
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        const unsigned o = ROWLIKE ? ((unsigned)q * (unsigned)sizeof(ST)) : 0u;
        const unsigned so = ROWLIKE ? 0u : (unsigned)(q << 5) * (unsigned)sizeof(ST);
        const int fi = fi0 + q * C32;
        if (sizeof(ST) == 8) {
          cp8s(ROWLIKE ? (P0 ^ o) : P0 + so, gp + fi);
          cp8s(ROWLIKE ? (A0 ^ o) : A0 + so, ga + fi);
        } else {
          cp4s(ROWLIKE ? (P0 ^ o) : P0 + so, gp + fi);
          cp4s(ROWLIKE ? (A0 ^ o) : A0 + so, ga + fi);
        }
        if (!ROWLIKE) cp8s(Z0 + (unsigned)(q << 5) * 8u, A.c + (base32 + (k0 + q) * ns32));
      }
      if (ROWLIKE) {  // mode B: lanes 8g..8g+7 along chain rows {8g + ib}
        const int pos = k0 + (lane & 7);
        const int poff = pos * ns32 + zz32 * ((pos + ph32) & 1);
        const int gb = (lane >> 3) << 3;
        const double* const cg = A.c;
#pragma unroll
        for (int ib = 0; ib < 8; ++ib)
          cp8s(rz_s + (unsigned)(rix(gb, pos) ^ (ib * 33)) * 8u, cg + (unsigned)(bB[ib] + poff));
      }
      cp_commit();
      return;
    }
#pragma unroll
    for (int q = 0; q < TP; ++q) {  // mode A
      const int pos = k0 + q;
      const bool pr = valid && pos < m;
      const int fi = pr ? (pos * C32 + c32) : 0;
      cp_elem(&rp[rx(lane, pos)], A.p + fi, pr);
      cp_elem(&ra[rx(lane, pos)], A.wf + (pos < m - 1 ? fi : 0), pr && pos < m - 1);
      if (!ROWLIKE) {
        const int nd = pr ? node(base32, pos) : 0;
        cp8(&rz[rx(lane, pos)], A.c + nd, pr);
      }
    }
    if (ROWLIKE) {  // mode B: lanes 8g..8g+7 along chain rows {8g + ib}
      const int q = lane & 7;
      const int pos = k0 + q;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int bi = bB[ib];
        const bool pr = i < nvalid && pos < m;
        const int nd = pr ? node(bi, pos) : 0;
        cp8(&rz[rx(i, pos)], A.c + nd, pr);
      }
    }
    cp_commit();
  };

  // G/X of tile T into registers (mode A natural; mode B rows for row-like MID)
  bool dep_ok = false;  // the previous sweep's output (G, X) may be read
  auto prefetch = [&](int T) {
    pre_tile = T;
    if (ROLE != MID && ROLE != LAST) return;
    if (!dep_ok) {
      // programmatic dependent launch: everything before this point reads
      // only this family's state, its weights and the drift; G / X (and the
      // LAST role's writes of X and c) come after the previous grid is done.
      // A no-op when the kernel was launched the ordinary way.
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      dep_ok = true;
    }
    const int k0 = T * TP;
    if (!ROWLIKE) {
      if (nvalid == 32 && k0 + TP <= m) {
        // whole tile of a full warp (the usual case): no predicates, one
        // per-tile base per array and one IMAD.WIDE + load per position
        const ST* gi_t = A.Gi + (base32 + k0 * ns32);
        const ST* x_t = A.X + (base32 + k0 * ns32);
#pragma unroll
        for (int q = 0; q < TP; ++q) {
          gpre[q] = gi_t[q * ns32];
          if (ROLE == LAST) xpre[q] = x_t[q * ns32];
        }
        return;
      }
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        const int pos = k0 + q;
        const bool pr = valid && pos < m;
        const int nd = pr ? node(base32, pos) : 0;
        gpre[q] = pr ? A.Gi[nd] : ST(0);
        if (ROLE == LAST) xpre[q] = pr ? A.X[nd] : ST(0);
      }
    } else {
      const int pos = k0 + (lane & 7);
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const int bi = bB[ib];
        const bool pr = i < nvalid && pos < m;
        const int nd = pr ? node(bi, pos) : 0;
        gpre[ib] = pr ? A.Gi[nd] : ST(0);
        if (ROLE == LAST) xpre[ib] = pr ? A.X[nd] : ST(0);
      }
    }
  };

  // tile T landed: c slot -> z = p + c (lockstep)
  auto to_z = [&](int T) {
    // every load of the tile first, then the stores: the compiler cannot tell
    // the ring arrays apart, so an interleaved form serialises load -> store
    ST pv[TP];
    double cv[TP];
    if (RT) {
      // the drift box sits in the tile's z slots as [row = lane][8 positions],
      // 64-B swizzled (16-B chunk j of a 64-B row at j ^ address bits 7-8):
      // each lane reads its own row as four 16-B vectors (conflict free: the
      // 8 lanes of a phase cover distinct bank quads), then, after every lane
      // has read, the z values go to the [pos][lane] slots
      const unsigned rb = rz_s + (unsigned)pix(0, T * TP) * 8u + (unsigned)lane * 64u;
#pragma unroll
      for (int j = 0; j < TP / 2; ++j) {
        const unsigned a = rb + (unsigned)j * 16u;
        const unsigned ph = a ^ (((a >> 7) & 3u) << 4);
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n"
                     : "=d"(cv[2 * j]), "=d"(cv[2 * j + 1]) : "r"(ph) : "memory");
      }
#pragma unroll
      for (int q = 0; q < TP; ++q) pv[q] = rp[tix(T * TP, q)];
      __syncwarp();
    } else {
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        const int ix = tix(T * TP, q);
        pv[q] = rp[ix];
        cv[q] = rz[ix];
      }
    }
#pragma unroll
    for (int q = 0; q < TP; ++q) rz[tix(T * TP, q)] = (double)pv[q] + cv[q];
  };

  // lockstep retire of tile T: per-node outputs from (z, segment markers), write back
  // (HINTS: this sweep writes segment hints -- a separate instantiation of the
  // per-position body, so the common case carries no hint arithmetic)
  // FULL: every lane emitted the whole tile (the usual case), so the
  // per-position emit tests go
  auto retire_impl = [&](int T, auto hints_tag, auto full_tag) {
    constexpr bool HINTS = decltype(hints_tag)::value;
    constexpr bool FULL = decltype(full_tag)::value;
    const int k0 = T * TP;
    // the tile's output rows: p' in the family layout (32-bit element index),
    // G / X / c in node order
    const int pi0 = k0 * C32 + c32;
    const int nd0 = node(base32, k0);
    // per-tile output bases kept in registers (opaque to the compiler, which
    // otherwise re-reads the argument pointers from the constant bank and
    // rebuilds a 64-bit address from the element index at every position):
    // a position's store address is then one IMAD.WIDE off the base
    ST* po_t = A.po + pi0;
    ST* G_t = A.G + nd0;
    ST* Xo_t = A.Xo + nd0;
    double* co_t = A.co + nd0;
#ifndef PCB_NO_RETIRE_BASES
    if (ROLE != SHADOW) {
      asm volatile("" : "+l"(po_t));
      if (!ROWLIKE && !RT) {
        if (ROLE != LAST || XG) asm volatile("" : "+l"(G_t));
        if (ROLE == LAST) {
          asm volatile("" : "+l"(Xo_t));
          asm volatile("" : "+l"(co_t));
        }
      }
      // (still global memory: keeps the stores STG rather than generic ST)
      __builtin_assume(__isGlobal(po_t));
      __builtin_assume(__isGlobal(G_t));
      __builtin_assume(__isGlobal(Xo_t));
      __builtin_assume(__isGlobal(co_t));
    }
#endif
    // strided families: the tile's ring rows are 32 slots apart from a per-tile
    // base, so every per-position ring access is base + immediate
    const int ixb = ROWLIKE ? rix(lane, k0) : pix(lane, k0);
    // positions of this tile my chain emitted: [max(start, k0), min(stop, i0))
    const int elo = max(start, k0) - k0, ehi = min(min(stop, i0), k0 + TP) - k0;
    const unsigned emask = (has && ehi > elo) ? (((1u << ehi) - 1u) & ~((1u << elo) - 1u)) : 0u;
    double na = 0.0, nb = 0.0;  // two monitor accumulators: shorter dependency chains
    const unsigned stile = smask >> (k0 & (RL - 1));  // segment starts of this tile (bit q)
    // row-like values for the ring (d, or the shadow's y) are stored after the
    // loop: the compiler cannot tell the ring arrays apart, so a store inside
    // it would order every later ring load behind it
    ST dsv[TP];
    double ysv[TP];
    // TST: the tile's p' goes through the ring's p slots and one bulk tensor
    // store (in-place steps only: the output array is the map's)
    ST psv[TP];
    const bool tma_st = TST && use_tma && A.po == A.p;
#pragma unroll
    for (int q = 0; q < TP; ++q) {
      const int pos = k0 + q;
      double& nq = (q & 1) ? nb : na;
      if (FULL || ((emask >> q) & 1u)) {
        const int ix = ROWLIKE ? (ixb ^ q) : ixb + (q << 5);
        const double zj = rz[ix];
        if ((stile >> q) & 1u) {
          zs = zj;
          // (SHADOW: the fp64 q split over the dead p / weight slots)
          if (QSPLIT)
            qs = __hiloint2double(__float_as_int((float)ra[ix]), __float_as_int((float)rp[ix]));
          else
            qs = (double)ra[ix];
          if (HINTS) {
            // the segment's prox value; jumps below 1e-6 (fp32 rounding of q)
            // count as none, so the change count sees segmentation changes
            // rather than rounding noise
            const double xs = zj - qs, dj = xs - xprev;
            hup |= (unsigned)(dj > 1e-6) << (7 + q);
            hdn |= (unsigned)(dj < -1e-6) << (7 + q);
            xprev = xs;
          }
        }
        const double pn = (zj - zs) + qs;
        if (ROLE == SHADOW) {
          if (!ROWLIKE && !RT) A.y[node(base32, pos)] = pn;
          else ysv[q] = pn;
        } else {
          const ST pold = rp[ix];
          const ST p32 = (ST)pn;
          // d in the state type (fp32: one FADD, d rounded once; the G sums
          // below are single fp32 adds, which equal the fp64-then-round form)
          const ST dS = p32 - pold;
          const double d = (double)dS;
          nq = nrm_d(d, nq);
          if (TST && FULL && tma_st) psv[q] = p32;
          else po_t[q * C32] = p32;
          if (RT) {
            dsv[q] = dS;
          } else if (!ROWLIKE) {
            const int nd = q * ns32;  // strided: node(base32, k0 + q) - nd0
            if (ROLE == FIRST) {
              G_t[nd] = dS;
            } else if (ROLE == MID) {
              G_t[nd] = gpre[q] + dS;
            } else {
              const ST g32 = gpre[q] + dS;
              const double g = (double)g32;
              const double xn = (double)xpre[q] - g;
              Xo_t[nd] = (ST)xn;
              const double dcv = (xn - g) * A.inv_r;
              co_t[nd] = (zj - (double)pold) + dcv;  // c_old = z - p_old
              if (XG) G_t[nd] = g32;
              nq = nrm_last(dcv, g, A.rd, nq);
            }
          } else {
            dsv[q] = dS;
          }
        }
      }
    }
    if (ROWLIKE) {
#pragma unroll
      for (int q = 0; q < TP; ++q) {
        if (FULL || ((emask >> q) & 1u)) {
          if (ROLE == SHADOW) rz[ixb ^ q] = ysv[q];
          else ra[ixb ^ q] = dsv[q];
        }
      }
    }
    if (TST && FULL && tma_st) {
#pragma unroll
      for (int q = 0; q < TP; ++q) rp[ixb + (q << 5)] = psv[q];
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> async reads
      __syncwarp();
      if (lane == 0)
        tma2d_store(&M.p, (int)c0, k0, rp_s + (unsigned)pix(0, k0) * (unsigned)sizeof(ST));
    }
    if (RT) {  // the tile's node-order outputs: this lane's row, positions k0..k0+7
      if (FULL) {  // 16-B vectors (pcb_create keeps row starts 4-element aligned for RT)
        if (ROLE == SHADOW) {
          double* yp = A.y + nd0;
#pragma unroll
          for (int j = 0; j < TP / 2; ++j)
            asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(yp + 2 * j),
                         "d"(ysv[2 * j]), "d"(ysv[2 * j + 1]) : "memory");
        } else {
          ST* gp = A.G + nd0;
          if (sizeof(ST) == 4) {
#pragma unroll
            for (int j = 0; j < TP / 4; ++j)
              asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(gp + 4 * j),
                           "f"((float)dsv[4 * j]), "f"((float)dsv[4 * j + 1]),
                           "f"((float)dsv[4 * j + 2]), "f"((float)dsv[4 * j + 3]) : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < TP / 2; ++j)
              asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(gp + 2 * j),
                           "d"((double)dsv[2 * j]), "d"((double)dsv[2 * j + 1]) : "memory");
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < TP; ++q) {
          if ((emask >> q) & 1u) {
            if (ROLE == SHADOW) A.y[nd0 + q] = ysv[q];
            else A.G[nd0 + q] = dsv[q];
          }
        }
      }
    }
    smask &= ~(0xffu << ((k0 & (RL - 1))));
    if (HINTS && valid) {
      // the word of tile T - 1 is complete now (its last edge's side came from
      // a segment start at k0); the old word of tile T is read for the next one
      hold_prev = hold_cur;
      if (T < ntile_sg) hold_cur = A.sg[T * C32 + c32];
      if (T > t_first) {
        const unsigned wd = (hup & 0xffu) | ((hdn & 0xffu) << 8);
        hchanged |= wd != hold_prev;
        A.sg[(T - 1) * C32 + c32] = (uint16_t)wd;
      }
      hup >>= 8;
      hdn >>= 8;
    }
    if (ROWLIKE) {
      __syncwarp();
      const int q = lane & 7;
      const int pos = k0 + q;
      // ring slot of row gb + ib at pos: rix(gb, pos) ^ (ib * 33) (gb a multiple of 8)
      const int rgb = rix((lane >> 3) << 3, pos);
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int i = ((lane >> 3) << 3) + ib;
        const unsigned em_i = FULL ? 0xffu : __shfl_sync(0xffffffffu, emask, i);
        const int bi = bB[ib];
        if (FULL || ((em_i >> q) & 1u)) {
          const int ix = rgb ^ (ib * 33);
          const int nd = node(bi, pos);
          if (ROLE == SHADOW) {
            A.y[nd] = rz[ix];
          } else if (ROLE == FIRST) {
            A.G[nd] = ra[ix];
          } else if (ROLE == MID) {
            A.G[nd] = gpre[ib] + ra[ix];
          } else {
            const ST g32 = gpre[ib] + ra[ix];
            const double g = (double)g32;
            const double xn = (double)xpre[ib] - g;
            A.Xo[nd] = (ST)xn;
            const double dcv = (xn - g) * A.inv_r;
            A.co[nd] = (rz[ix] - (double)rp[ix]) + dcv;  // c_old = z - p_old
            if (XG) A.G[nd] = g32;
            double& nq = (ib & 1) ? nb : na;
            nq = nrm_last(dcv, g, A.rd, nq);
          }
        }
      }
      __syncwarp();
    }
    nrm += na + nb;
  };
  auto retire = [&](int T) {
    PCB_CNT(4, 1);
    if (pre_tile != T) prefetch(T);
    const int k0 = T * TP;
    const bool full = has && max(start, k0) == k0 && min(min(stop, i0), k0 + TP) == k0 + TP;
    if (SGW) retire_impl(T, std::true_type(), std::false_type());
    else if (__all_sync(0xffffffffu, full)) retire_impl(T, std::false_type(), std::true_type());
    else retire_impl(T, std::false_type(), std::false_type());
  };

  // one round of scanning; LAG: some lane's anchor is below the ring
  // keep_min: leave the round once at most this many lanes still have data
  // (they continue next round), so a few slow lanes do not idle the warp
  auto scan = [&](int lo_pos, int avail_hi, int keep_min, auto lag_tag) {
    constexpr bool LAG = decltype(lag_tag)::value;
    asm volatile("" : "+r"(keep_min));  // keep it in a register, not re-derived per trip
    // software-pipelined ring reads: the next gate's z and a are loaded at the
    // end of the previous trip (slots >= k are never written by the scan)
    double zn = rz[rx(lane, k)];
    ST an = ra[rx(lane, k)];
    const int lim = min(avail_hi, stop);  // gates are consumed while k < lim
    // an anchor gate not consumed yet (unit start, or a restart whose gate
    // was not loaded when the string bent): t is its z
    if (!LAG && k == i0 && k < lim) t = zn;
    auto trip = [&]() {
      const bool act = k < lim;
      if (act) {
        const int kp = k;
        double zabs = zn;
        ST af = an;
        if (LAG && kp < lo_pos) {  // lagging lane below the ring
          const int fi = (kp * C32 + c32);
          zabs = z_global(A, fi, node(base32, kp));
          af = kp < m - 1 ? (ST)a_global(A, fi) : ST(0);
        }
        k = kp + 1;
        if (LAG) t = kp == i0 ? zabs : t;  // the anchor gate itself
        skr += (R)(zabs - t);
        const bool at_stop = k == stop;  // forced end point (merge point or chain end)
        const bool inner = !at_stop;     // (k <= stop)
        const R rk = inner ? (R)af : R(0);
        // a zero weight (or the unit end) makes this gate a mandatory piece end;
        // after an earlier bend the rescan reaches the same gate again, so no
        // piece-end state needs to be kept
        const bool zw = !inner || af == ST(0);
        const R inv = rcp_r<R>(k - i0);
        Lc += cs;
        Lf += fs;
        const R sE = at_stop ? skr + eoff : skr;  // string value required at an end gate
        // ceiling: keep the minimum slope from the anchor
        const R u = sE + rk;
        const bool cu = u <= Lc;
        c0x = cu ? k : c0x;
        acx = cu ? rk : acx;
        cs = cu ? u * inv : cs;
        Lc = cu ? u : Lc;
        const bool b1 = cs < fs;  // ceiling dips under the floor cone
        // floor: keep the maximum slope (not pushed when b1 already bends)
        const R l = sE - rk;
        const bool fu = !b1 && l >= Lf;
        f0x = fu ? k : f0x;
        afx = fu ? rk : afx;
        fs = fu ? l * inv : fs;
        Lf = fu ? l : Lf;
        const bool b2 = !b1 && fs > cs;       // floor rises over the ceiling cone
        const bool e = !b1 && !b2 && zw;  // piece end: S_k is mandatory
        // (a ceiling / floor point taken at this gate has Lc = sE + rk >= sE /
        // Lf = sE - rk <= sE, so these tests need no "is it this gate" check)
        const bool ec = e && Lc < sE;
        const bool ef = e && !ec && Lf > sE;
        const bool bend = b1 || b2 || e;
#ifdef PCB_COUNT
        if (bend) atomicAdd(&g_count[2], 1ull);
#endif
        const bool tf = b1 || ef;  // touches the floor
        const bool tc = b2 || ec;  // touches the ceiling
        const int bk = tf ? f0x : (tc ? c0x : k);
        const R fill = tf ? fs : (tc ? cs : sE * inv);
        // ---- close segment [i0, bk): its prox value is the string slope `fill` (+ t)
        int s0 = i0;
        R qv = -fill;  // q = z_i0 - fill, and z_i0 - t = 0
        if (LAG && bend && i0 < lo_pos) {
          const double fabs_ = (double)fill + t;
          const int e2 = min(min(bk, lo_pos), stop);
          for (int j = i0; j < e2; ++j)
            nrm += finish_global<ROLE, ST>(A, (j * C32 + c32), node(base32, j), fabs_);
          s0 = e2;
          if (s0 < bk) qv = (R)((rz[rx(lane, s0)] - t) - (double)fill);
        }
        // (lag-free: s0 = i0 < k <= stop)
        const bool mark = LAG ? (bend && s0 < stop && s0 < bk) : bend;
        const int ixs = LAG ? rx(lane, s0) : ixi0;
        if (mark) {
          if (QSPLIT) {  // fp64 q: low word in the p slot, high word in the weight slot
            const double qd = (double)qv;
            rp[ixs] = (ST)__int_as_float(__double2loint(qd));
            ra[ixs] = (ST)__int_as_float(__double2hiint(qd));
          }
          else ra[ixs] = (ST)qv;
        }
        smask |= (unsigned)mark << (s0 & (RL - 1));
        // after a touch the string leaves the tube point: skr = -touch * a(bk-1)
        // (a free piece end restarts at 0; a touch at the unit's stop gate, where
        // rk = 0 was recorded, ends the unit)
        const R nskr = tf ? afx : (tc ? -acx : R(0));
        i0 = bend ? bk : i0;
        k = bend ? bk : k;
        skr = bend ? nskr : skr;
        // a fresh anchor: the next gate overwrites cs, Lc, fs, Lf
        Lc = bend ? RINF : Lc;
        Lf = bend ? -RINF : Lf;
        fs = bend ? -RINF : fs;
        const int ixn = rx(lane, k);
        ixi0 = bend ? ixn : ixi0;  // i0 = k = bk after a bend
        zn = rz[ixn];
        an = ra[ixn];
        // non-lagging: the anchor value of a restarted string is the next gate's
        // z, unless that gate is not loaded yet (then the next round takes it)
        if (!LAG) {
          t = bend ? zn : t;
          // The first gate after a restart cannot bend (one point: both cones
          // coincide, slopes skr +- a over a distance of 1), so it is taken
          // here instead of in a trip of its own -- about one trip per segment,
          // i.e. nearly every rescan.  Not at a zero weight or the unit end
          // (a mandatory piece end) or when position k is not loaded yet.
          const int k1 = k + 1;
          const bool triv = bend && k < lim && k1 < stop && an != ST(0);
          if (triv) {
            const R rk1 = (R)an;
            c0x = k1;
            f0x = k1;
            acx = rk1;
            afx = rk1;
            cs = skr + rk1;
            Lc = cs;
            fs = skr - rk1;
            Lf = fs;
            k = k1;
            const int ix1 = rx(lane, k1);
            zn = rz[ix1];
            an = ra[ix1];
          }
        }
      }
    };
    for (;;) {
      const int nact = __popc(__ballot_sync(0xffffffffu, k < lim));
      if (nact <= keep_min) break;
      PCB_CNT(0, 1);
      PCB_CNT(1, nact);
      trip();
      // more trips per exit vote (the vote, popcount and loop branch are ~5
      // of the ~110 instructions of a trip); a round may run a few trips past
      // the keep threshold
#pragma unroll
      for (int u = 1; u < (LAG ? 1 : PCB_SCAN_UNROLL); ++u) trip();
    }
  };

  // ---------------- VER: verify last iteration's segmentation as a candidate.
  // Lanes advance in lockstep, one position per step.  Each candidate segment
  // [i0, k] (ended by a hinted tube touch, a zero weight or the chain end) gets
  // its value from the sum of z and the duals at its ends (u = -a at a ceiling
  // touch, +a at a floor touch, 0 at a piece end), and the complete KKT
  // conditions are checked: |u_j| <= a_j on the interior edges (a cone of
  // slopes, as in the taut string) and the sign of the jump at a touch.  A
  // segment that fails is still emitted; its lane is repaired after the sweep
  // (repair_lane: a taut string between true points around the failures).
  int ff = 0x7fffffff, fl = -1;  // VER: first failing segment start, last failing position
  if constexpr (VER) if (warp_live && rhi > 0) {
    constexpr float FINF = __builtin_huge_valf();
    bool vdone = !has;            // closed the chain's last segment, or abandoned
    double vt = 0.0, tp = 0.0;    // anchor (z at i0) of the open / previous segment
    float Q = 0.f, LO = -FINF, HI = FINF, xrp = 0.f;
    int sideL = 0;                // side of the open segment's left edge (0: piece start)
    auto vtrip = [&](int k0, int q, unsigned w) {
      const int kk = k0 + q;
      if (vdone || kk >= stop) return;
      const int ix = tix(k0, q);
      const double z = rz[ix];
      const float a = ra[ix];
      const bool last = kk == m - 1;
      const float ak = last ? 0.f : a;
      const int side = (int)((w >> q) & 1u) - (int)((w >> (8 + q)) & 1u);
      const bool fresh = kk == i0;
      vt = fresh ? z : vt;
      const float zr = (float)(z - vt);
      Q += zr;
      const float inv = rcp_r<float>(kk - i0 + 1);
      const bool piece = last || ak == 0.f;
      const bool cl = piece || side != 0;
      const float uR = piece ? 0.f : (side > 0 ? -ak : ak);
      if (cl) {
        const float xr = (Q - uR) * inv;                  // segment value - vt
        const float dx = (xr - xrp) + (float)(vt - tp);   // jump over the left edge
        const float tol = 4e-6f * (1.f + fabsf(xr));
        const bool bad = (LO > xr + tol) || (xr > HI + tol) || ((float)sideL * dx < -tol);
        ff = bad ? min(ff, i0) : ff;
        fl = bad ? kk : fl;
        ra[rx(lane, i0)] = -xr;  // q = p'(i0) = z(i0) - x; the retire rebuilds the rest
        smask |= 1u << (i0 & (RL - 1));
        xrp = xr;
        tp = vt;
        sideL = piece ? 0 : side;
        Q = uR;
        LO = -FINF;
        HI = FINF;
        i0 = kk + 1;
        vdone = i0 >= stop;
      } else {  // interior edge kk: (Q - a) / len <= x - vt <= (Q + a) / len
        LO = fmaxf(LO, (Q - ak) * inv);
        HI = fminf(HI, (Q + ak) * inv);
      }
    };
    int T = t_first;  // next tile to verify
    while (t_ld < ntiles && t_ld - t_first < NT) issue(t_ld++);
    for (;;) {
      if (T < t_ld) {
        land(T);
        to_z(T);
        t_rdy = T + 1;
        const unsigned w = (unsigned)(sw >> ((unsigned)(T & (NT - 1)) * 16u)) & 0xffffu;
#pragma unroll
        for (int q = 0; q < TP; ++q) vtrip(T * TP, q, w);
        ++T;
      }
      if (__all_sync(0xffffffffu, vdone)) {
        for (int X = T; X < t_ld; ++X) land(X);  // nothing may be in flight at exit
        if (!use_tma) {
          cp_wait(0);
          __syncwarp();
        }
        for (int X = t_lo; X < t_ld; ++X) retire(X);
        break;
      }
      const int front = __reduce_min_sync(0xffffffffu, vdone ? 0x7fffffff : i0);
      while (t_lo < T && (t_lo + 1) * TP <= front) retire(t_lo++);
      if (t_lo < T && pre_tile != t_lo) prefetch(t_lo);  // G / X of the next tile to retire
      if (t_ld - t_lo == NT && T == t_ld) {
        // ring full and a lane's open segment spans it: that lane gives up
        // here (its positions from i0 on stay unemitted) and is repaired
        if (!vdone && i0 < (t_lo + 1) * TP) {
          ff = min(ff, i0);
          fl = m;
          vdone = true;
        }
        __syncwarp();
        retire(t_lo++);
      }
      __syncwarp();
      while (t_ld < ntiles && t_ld - t_lo < NT) issue(t_ld++);
    }
  }
  if (!VER && warp_live && rhi > 0) {
    while (t_ld < ntiles && t_ld - t_first < NT) issue(t_ld++);
    land(t_first);
    to_z(t_first);
    t_rdy = t_first + 1;
    for (;;) {
      const int lo_pos = t_lo * TP;
      const int avail_hi = min(t_rdy * TP, m);
      // (MID / LAST: not before the first retire, so that a programmatic
      // launch scans its first tiles while the previous sweep drains)
      if (pre_tile != t_lo && (dep_ok || (ROLE != MID && ROLE != LAST))) prefetch(t_lo);
      // ---------------- scan until every lane needs data beyond avail_hi.
      // One gate per trip.  Warps with no lagging lane (the normal case) run
      // a variant without any below-the-ring checks, with the segment close
      // fully predicated so the warp stays converged through bends.
      const int keep = (t_rdy < t_ld) ? PCB_SCAN_KEEP : 0;
      if (__any_sync(0xffffffffu, i0 < lo_pos && i0 < stop))
        scan(lo_pos, avail_hi, keep, std::true_type());
      else
        scan(lo_pos, avail_hi, keep, std::false_type());
      __syncwarp();
      if (__all_sync(0xffffffffu, i0 >= stop)) {
        if (use_tma) {
          for (int T = t_rdy; T < t_ld; ++T) land(T);  // no TMA may be in flight at exit
        } else {
          cp_wait(0);
          __syncwarp();
        }
        for (int T = t_lo; T < t_ld; ++T) retire(T);
        if (SGW && valid && ntiles > t_first) {  // the last tile's word
          const unsigned wd = (hup & 0xffu) | ((hdn & 0xffu) << 8);
          hchanged |= wd != hold_cur;
          A.sg[(ntiles - 1) * C32 + c32] = (uint16_t)wd;
        }
        break;
      }
      // ---------------- retire tiles every lane has emitted
      const int front = __reduce_min_sync(0xffffffffu, i0 < stop ? i0 : 0x7fffffff);
      while (t_lo < t_rdy && (t_lo + 1) * TP <= front) retire(t_lo++);
      const bool any_act = __any_sync(0xffffffffu, k < min(avail_hi, stop));
      if (!any_act && t_rdy == t_ld && t_ld - t_lo == NT)
        retire(t_lo++);  // ring full: lagging lanes go global
      __syncwarp();
      while (t_ld < ntiles && t_ld - t_lo < NT) issue(t_ld++);
      if (t_rdy < t_ld) {
        land(t_rdy);
        to_z(t_rdy);
        ++t_rdy;
      }
    }
  }
  if constexpr (VER) {
    __syncwarp();  // the sweep's writes (mode-B lanes write other chains) are visible
    const bool dirty = valid && ff != 0x7fffffff;
#ifndef PCB_NO_REPAIR  // timing experiments only: results are wrong without the repair
    if (dirty) nrm += repair_lane<ROLE, ROWLIKE>(A, c32, base32, ff, fl, i0);
#endif
    const int nch = __popc(__ballot_sync(0xffffffffu, dirty));
    if (lane == 0 && nch && A.vcount) atomicAdd(A.vcount, nch);
  }
  if (SGW && warp_live) {  // chains whose hints changed: the mode policy's signal
    const int nch = __popc(__ballot_sync(0xffffffffu, hchanged && valid));
    if (lane == 0 && nch && A.vcount) atomicAdd(A.vcount, nch);
  }
  // (the stores have read the ring before the block's shared memory goes away)
  if (TST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  if (ROLE != SHADOW) {  // step-norm partial: one slot per warp (no block barrier)
    const double v = warp_sum(nrm);
    if (lane == 0) A.parts[(blockIdx.x + (int64_t)blockIdx.y * gridDim.x) * WARPS + wib] = v;
  }
}


// ---------------------------------------------------------------------------
// Intra-chain split: merge points.  For block b >= 1 of chain c the true
// string crosses gate g = b * lb somewhere inside the tube [S_g - a, S_g + a].
// The taut strings anchored at the floor point and at the ceiling point of
// that gate bracket it (taut strings to a common end point never cross), so
// at their first common tube touch all three coincide and stay equal.  Each
// thread scans both speculative strings (fp64 stackless scan, data from
// global memory) bend by bend until they share a bend point, or gives up
// after `window` positions (merge = -1: the previous unit continues).
// One warp = 32 chains at block b.  The first MW positions from the block
// gate are staged in shared memory with coalesced cp.async (mode A / mode B
// like the sweep); merges almost always happen inside that window, positions
// beyond it are read from global memory.
constexpr int MW = 16;
__device__ __forceinline__ int mix(int l, int q) { return l * MW + (q ^ (l & (MW - 1))); }

template <bool ROWLIKE, class ST = float>
__global__ void __launch_bounds__(MWARPS * 32) k_merge(Fam F, const ST* p, const ST* wf,
                                                      const double* cdr, int lb, int nb, int window,
                                                      int* merge) {
  __shared__ double sz[MWARPS][32 * MW];
  __shared__ ST sa[MWARPS][32 * MW];
  __shared__ ST sp[MWARPS][32 * MW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * MWARPS + wib) * 32;
  const int b = blockIdx.y + 1;
  const int64_t C = F.C;
  const int m = F.m;
  const int g = b * lb;
  if (c0 >= C || b >= nb || g >= m) return;  // warp-uniform
  const int nvalid = (int)min((int64_t)32, C - c0);
  const bool valid = lane < nvalid;
  const int64_t c = c0 + lane;
  const int C32 = (int)C, c32 = (int)c;  // n < 2^31: 32-bit index math
  const int ns32 = (int)F.ns, zz32 = (int)F.zz, ph32 = F.phase;
  const int base = valid ? (int)fam_base(F, c) : 0;
  auto node = [&](int bb, int pos) { return bb + pos * ns32 + zz32 * ((pos + ph32) & 1); };
  double* z_s = sz[wib];
  ST* a_s = sa[wib];
  ST* p_s = sp[wib];
  // ---- stage positions [g, g + MW)
#pragma unroll 4
  for (int q = 0; q < MW; ++q) {
    const int pos = g + q;
    const bool pr = valid && pos < m;
    const int fi = pr ? pos * C32 + c32 : 0;
    cp_elem(&p_s[mix(lane, q)], p + fi, pr);
    cp_elem(&a_s[mix(lane, q)], wf + (pos < m - 1 ? fi : 0), pr && pos < m - 1);
    if (!ROWLIKE) cp8(&z_s[mix(lane, q)], cdr + (pr ? node(base, pos) : 0), pr);
  }
  if (ROWLIKE) {
#pragma unroll 4
    for (int ib = 0; ib < 32; ib += 32 / MW) {
      const int i = ib + lane / MW;
      const int q = lane % MW;
      const int bi = __shfl_sync(0xffffffffu, base, i);
      const int pos = g + q;
      const bool pr = i < nvalid && pos < m;
      cp8(&z_s[mix(i, q)], cdr + (pr ? node(bi, pos) : 0), pr);
    }
  }
  cp_commit();
  cp_wait(0);
  __syncwarp();
  // z = p + c in chunks of 8 positions, loads before stores (the compiler
  // cannot tell the staging arrays apart and would serialise load -> store)
#pragma unroll
  for (int q0 = 0; q0 < MW; q0 += 8) {
    ST pv[8];
    double cv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ix = mix(lane, q0 + q);
      pv[q] = p_s[ix];
      cv[q] = z_s[ix];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) z_s[mix(lane, q0 + q)] = (double)pv[q] + cv[q];
  }
  __syncwarp();
  if (!valid) return;
  auto za = [&](int pos, double* z, double* a) {
    const int q = pos - g;
    if (q >= 0 && q < MW) {
      const int ix = mix(lane, q);
      *z = z_s[ix];
      *a = (double)a_s[ix];
    } else {
      const int fi = pos * C32 + c32;
      *z = (double)__ldg(p + fi) + __ldg(cdr + node(base, pos));
      *a = pos < m - 1 ? (double)__ldg(wf + fi) : 0.0;
    }
  };
  int out = -1;
  const double ag = (double)__ldg(wf + (g - 1) * C32 + c32);
  if (ag == 0.0) {
    out = g * 4 + 1;  // zero-weight gate: a piece starts here for every string
  } else {
    Spec Fs{g, m, g, -1, -1, 0.0, ag, 0.0, 0.0, 0.0, 0.0, true};
    Spec Us{g, m, g, -1, -1, 0.0, -ag, 0.0, 0.0, 0.0, 0.0, true};
    int pf, tf, pu, tu;
    spec_next_bend(Fs, m, za, &pf, &tf);
    spec_next_bend(Us, m, za, &pu, &tu);
    const int lim = min(m, g + window);
    while (pf < lim || pu < lim) {
      if (pf == pu && tf == tu) {
        if (pf < m) out = pf * 4 + (tf + 1);
        break;
      }
      if (pf <= pu) {
        if (pf >= lim) break;
        spec_next_bend(Fs, m, za, &pf, &tf);
      } else {
        if (pu >= lim) break;
        spec_next_bend(Us, m, za, &pu, &tu);
      }
    }
  }
  merge[(int64_t)b * C + c] = out;
}

}  // namespace fast
}  // namespace pcb
