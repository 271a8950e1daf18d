// taut_string.cuh -- exact weighted 1D-TV prox on one chain, device side.
//
// Restates the reference taut string (_kernels.py:11-142) operation for
// operation so that, compiled with -fmad=false (no FMA contraction; numba
// compiles the reference without fastmath, _kernels.py:3-5), the output is
// bitwise equal to the reference on the same fp64 inputs.
//
// Differences in *form*, not in arithmetic:
//  * zero-weight edges end a chain piece on the fly (the reference splits
//    lines into separate chains at zero weights, decompose.py:120-139); a
//    piece restarts with fresh running sums exactly like a new chain;
//  * inputs come through an accessor (Acc::s, Acc::a) and outputs leave
//    through Acc::emit(i, fill), so one state machine serves the CSR
//    gather/scatter path, the fp64 grid path and the fused fp32 path;
//  * hull stacks live in a Hull object: the first HC entries in shared
//    memory (lane-interleaved, bank-conflict free), deeper entries in a
//    global spill region (measured depth on the BASELINE inputs is <= 7,
//    SURVEY 0.9, but adversarial weights can reach the chain length).
#pragma once
#include <cstdint>

namespace pcb {

template <int HC>
struct Hull {
  int* sx;      // shared: entry e of this thread at sx[e * ss]
  double* sy;
  int ss;
  int* gx;      // global spill: entry e >= HC at gx[(e - HC) * gs]
  double* gy;
  int64_t gs;
  __device__ __forceinline__ int x(int e) const {
    return e < HC ? sx[e * ss] : gx[(int64_t)(e - HC) * gs];
  }
  __device__ __forceinline__ double y(int e) const {
    return e < HC ? sy[e * ss] : gy[(int64_t)(e - HC) * gs];
  }
  __device__ __forceinline__ void put(int e, int xv, double yv) {
    if (e < HC) {
      sx[e * ss] = xv;
      sy[e * ss] = yv;
    } else {
      gx[(int64_t)(e - HC) * gs] = xv;
      gy[(int64_t)(e - HC) * gs] = yv;
    }
  }
};

// One chain of m nodes.  Acc provides:
//   double s(int i)           signal at node i
//   double a(int i)           weight of edge (i, i+1), i < m-1
//   void   emit(int i, double fill)   prox value of node i (called once per
//                                      node, in increasing i)
template <class Acc, class HullT>
__device__ void taut_chain(Acc& A, HullT& cH, HullT& fH, int m) {
  int i0 = 0;          // anchor gate
  double a_val = 0.0;  // string value at the anchor
  int a_t = 0;         // anchor touches: -1 floor, +1 ceiling, 0 free
  double a_S = 0.0;    // running sum at the anchor
  int pe = m;          // end gate of the current piece (lowered at zero weights)
  while (i0 < m) {
    int nc = 0, nf = 0, k = i0;
    int bk = -1, bt = 0;
    double by = 0.0;
    double sk = a_S;
    // bottom hull entries cached in registers (read on every gate)
    int c0x = 0, f0x = 0;
    double c0y = 0.0, f0y = 0.0;
    while (k < pe) {
      ++k;
      sk += A.s(k - 1);
      double rk = 0.0;
      if (k < m) {
        rk = A.a(k - 1);
        if (rk == 0.0) pe = k;  // zero weight: this gate closes the piece
      }
      // ceiling point (k, sk + rk): keep the hull convex from the anchor
      const double uy = sk + rk;
      while (nc >= 1) {
        int px;
        double py;
        if (nc >= 2) {
          px = cH.x(nc - 2);
          py = cH.y(nc - 2);
        } else {
          px = i0;
          py = a_val;
        }
        const int qx = (nc == 1) ? c0x : cH.x(nc - 1);
        const double qy = (nc == 1) ? c0y : cH.y(nc - 1);
        if ((qy - py) * (double)(k - qx) >= (uy - qy) * (double)(qx - px))
          --nc;
        else
          break;
      }
      cH.put(nc, k, uy);
      if (nc == 0) {
        c0x = k;
        c0y = uy;
      }
      ++nc;
      if (nf >= 1 && (c0y - a_val) * (double)(f0x - i0) < (f0y - a_val) * (double)(c0x - i0)) {
        bk = f0x;
        by = f0y;
        bt = -1;
        break;
      }
      // floor point (k, sk - rk): keep the hull concave from the anchor
      const double ly = sk - rk;
      while (nf >= 1) {
        int px;
        double py;
        if (nf >= 2) {
          px = fH.x(nf - 2);
          py = fH.y(nf - 2);
        } else {
          px = i0;
          py = a_val;
        }
        const int qx = (nf == 1) ? f0x : fH.x(nf - 1);
        const double qy = (nf == 1) ? f0y : fH.y(nf - 1);
        if ((qy - py) * (double)(k - qx) <= (ly - qy) * (double)(qx - px))
          --nf;
        else
          break;
      }
      fH.put(nf, k, ly);
      if (nf == 0) {
        f0x = k;
        f0y = ly;
      }
      ++nf;
      if ((f0y - a_val) * (double)(c0x - i0) > (c0y - a_val) * (double)(f0x - i0)) {
        bk = c0x;
        by = c0y;
        bt = 1;
        break;
      }
    }
    if (bk < 0) {
      // piece end: S_pe is mandatory; straight segment unless a hull point blocks it
      if (c0x != pe && (c0y - a_val) * (double)(pe - i0) < (sk - a_val) * (double)(c0x - i0)) {
        bk = c0x;
        by = c0y;
        bt = 1;
      } else if (f0x != pe && (f0y - a_val) * (double)(pe - i0) > (sk - a_val) * (double)(f0x - i0)) {
        bk = f0x;
        by = f0y;
        bt = -1;
      } else {
        bk = pe;
        by = sk;
        bt = 0;
      }
    }
    // segment [i0, bk) is constant: fresh sum plus the tube offsets at its ends
    const double ref = A.s(i0);
    double tot = 0.0;
    bool alleq = true;
    for (int j = i0; j < bk; ++j) {
      const double v = A.s(j);
      tot += v;
      alleq = alleq && (v == ref);
    }
    double corr = 0.0;
    if (bt != 0) corr += (double)bt * A.a(bk - 1);
    if (a_t != 0) corr -= (double)a_t * A.a(i0 - 1);
    const double fill = (alleq && corr == 0.0) ? ref : (tot + corr) / (double)(bk - i0);
    for (int j = i0; j < bk; ++j) A.emit(j, fill);
    i0 = bk;
    if (i0 == pe) {
      // piece finished: the next one starts like a fresh chain
      a_val = 0.0;
      a_t = 0;
      a_S = 0.0;
      pe = m;
    } else {
      a_val = by;
      a_t = bt;
      a_S = (bt == 0) ? by : by - (double)bt * A.a(bk - 1);
    }
  }
}

}  // namespace pcb
