// dual_schemes.cuh -- BCD, AP and FISTA on the exact fp64 kernels.
//
// The reference's three other dual schemes (solvers.py:212-269, 310-341)
// reuse Pi_K (the family prox sweep, here sweep_exact_sel) and Pi_L; every
// elementwise step below is the reference's expression in the reference's
// order, so the iterates y are bitwise equal to the reference's.  The
// monitors (_smooth_dual, norms) are fixed-order device reductions and match
// the reference's numpy/BLAS values to rounding.
//
// Buffers of an fp64 handle: y holds the dual iterate (so pcb_check certifies
// it directly), z holds lam (AP) or the momentum point v (FISTA), tmp holds
// the gradient point / new block iterate.
//
// Included inside paracut_b200.cu's anonymous namespace.

// s = sum_j y_j in class order (aggregate, projections.py:133-137)
__global__ void k_aggregate(const double* y, int r, int64_t n, double* s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = y[i];
    for (int j = 1; j < r; ++j) t = t + y[(int64_t)j * n + i];
    s[i] = t;
  }
}

// BCD block target: w - (s - y_j)  (solvers.py:226)
__global__ void k_bcd_target(const double* yj, const double* s, const double* w, int64_t n,
                             double* t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    t[i] = w[i] - (s[i] - yj[i]);
}

// BCD block update: diff = ynew - y_j, change += diff.diff, s += diff, y_j = ynew
// (solvers.py:229-233)
__global__ void k_bcd_apply(double* yj, const double* ynew, double* s, int64_t n, double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yn = ynew[i];
    const double d = yn - yj[i];
    acc += d * d;
    s[i] = s[i] + d;
    yj[i] = yn;
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// _smooth_dual partials (solvers.py:100-103): columns w.w and d.d, d = s - w
__global__ void k_smooth_parts(const double* s, const double* w, int64_t n, double* parts) {
  double ww = 0.0, dd = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
    const double d = s[i] - wi;
    ww += wi * wi;
    dd += d * d;
  }
  __shared__ double sh[32];
  double v = block_sum(ww, sh);
  if (threadIdx.x == 0) parts[2 * blockIdx.x] = v;
  v = block_sum(dd, sh);
  if (threadIdx.x == 0) parts[2 * blockIdx.x + 1] = v;
}

__global__ void k_smooth_final(const double* vals, double* out) {
  *out = 0.5 * vals[0] - 0.5 * vals[1];
}

// sqrt of a sum of per-family values, summed in family order (BCD change2)
__global__ void k_sum_sqrt(const double* v, int cnt, double* out) {
  double t = 0.0;
  for (int j = 0; j < cnt; ++j) t += v[j];
  *out = sqrt(t);
}

// lam = Pi_L(y) (projections.py:107-122); on a grid every class covers every
// node, so d_i = r and the support mask is 1
__global__ void k_ap_lam(const double* y, const double* w, int r, int64_t n, double* lam) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double total = y[i];
    for (int j = 1; j < r; ++j) total = total + y[(int64_t)j * n + i];
    const double corr = (w[i] - total) / (double)r;
    for (int j = 0; j < r; ++j) lam[(int64_t)j * n + i] = (y[(int64_t)j * n + i] + corr) * 1.0;
  }
}

// |a - b|^2 partials over r*n
__global__ void k_diff2(const double* a, const double* b, int64_t cnt, double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    acc += d * d;
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// FISTA gradient point: v_j - step * (sum_k v_k - w)  (solvers.py:327-328)
__global__ void k_fista_in(const double* v, const double* w, int r, int64_t n, double step,
                           double* in) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double agg = v[i];
    for (int j = 1; j < r; ++j) agg = agg + v[(int64_t)j * n + i];
    const double g = step * (agg - w[i]);
    for (int j = 0; j < r; ++j) in[(int64_t)j * n + i] = v[(int64_t)j * n + i] - g;
  }
}

// FISTA momentum (solvers.py:329-333): dy = ynew - y, v = ynew + coef * dy,
// y = ynew; partial dy.dy
__global__ void k_fista_mom(double* y, double* v, const double* ynew, int64_t cnt, double coef,
                            double* parts) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yn = ynew[i];
    const double dy = yn - y[i];
    acc += dy * dy;
    v[i] = yn + coef * dy;
    y[i] = yn;
  }
  __shared__ double sh[32];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// ---------------------------------------------------------------- host side

// _smooth_dual(w, s) into *slot (device)
int smooth_dual_dev(pcb_solver* h, const double* s, double* slot) {
  const int g = grid_for(h->n, RED_BLOCK, NODE_GRID);
  k_smooth_parts<<<g, RED_BLOCK, 0, h->stream>>>(s, h->w.p, h->n, h->parts.p);
  LAUNCH_CHECK(h);
  k_reduce_cols<<<1, 32 * 2, 0, h->stream>>>(h->parts.p, g, 2, h->vals.p + 60);
  LAUNCH_CHECK(h);
  k_smooth_final<<<1, 1, 0, h->stream>>>(h->vals.p + 60, slot);
  LAUNCH_CHECK(h);
  return 0;
}

// |a - b| over r*n into *slot (device)
int diff_norm_dev(pcb_solver* h, const double* a, const double* b, double* slot) {
  const int64_t rn = (int64_t)h->r * h->n;
  const int g = grid_for(rn, RED_BLOCK, NODE_GRID);
  k_diff2<<<g, RED_BLOCK, 0, h->stream>>>(a, b, rn, h->parts.p);
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, slot, 1);
  LAUNCH_CHECK(h);
  return 0;
}

// one BCD sweep (solvers.py:222-234); mon = _smooth_dual(w, s), stop = sqrt(change2)
int bcd_sweep(pcb_solver* h, double* mon, double* stop) {
  const int64_t n = h->n;
  double* s = h->tmp.p;           // n
  double* target = s + n;         // n
  double* ynew = target + n;      // n
  double* dots = h->vals.p + 56;  // per-family diff.diff
  const int g = grid_for(n, RED_BLOCK, NODE_GRID);
  k_aggregate<<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->r, n, s);
  LAUNCH_CHECK(h);
  for (int j = 0; j < h->r; ++j) {
    double* yj = h->y.p + (int64_t)j * n;
    k_bcd_target<<<g, RED_BLOCK, 0, h->stream>>>(yj, s, h->w.p, n, target);
    LAUNCH_CHECK(h);
    const double* src[1] = {target};
    double* dst[1] = {ynew};
    if (int e = sweep_exact_sel(h, j, j + 1, src, dst, true)) return e;
    k_bcd_apply<<<g, RED_BLOCK, 0, h->stream>>>(yj, ynew, s, n, h->parts.p);
    LAUNCH_CHECK(h);
    k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, g, dots + j, 0);
    LAUNCH_CHECK(h);
  }
  if (int e = smooth_dual_dev(h, s, mon)) return e;
  k_sum_sqrt<<<1, 1, 0, h->stream>>>(dots, h->r, stop);
  LAUNCH_CHECK(h);
  return 0;
}

// one AP step (solvers.py:257-263); mon = |y - lam|, stop = |y - yprev|
int ap_step(pcb_solver* h, double* mon, double* stop, bool want_stop) {
  const int64_t n = h->n, rn = (int64_t)h->r * n;
  const int g = grid_for(n, RED_BLOCK, NODE_GRID);
  double* lam = h->z.p;
  k_ap_lam<<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->w.p, h->r, n, lam);
  LAUNCH_CHECK(h);
  if (want_stop)
    CUDA_TRY(cudaMemcpyAsync(h->yprev.p, h->y.p, rn * sizeof(double), cudaMemcpyDeviceToDevice,
                             h->stream));
  if (int e = sweep_exact(h, lam, h->y.p, true)) return e;
  if (int e = diff_norm_dev(h, h->y.p, lam, mon)) return e;
  if (want_stop)
    if (int e = diff_norm_dev(h, h->y.p, h->yprev.p, stop)) return e;
  return 0;
}

// one FISTA step (solvers.py:326-334); mon = _smooth_dual(w, aggregate(y)),
// stop = |dy|
int fista_step(pcb_solver* h, double* mon, double* stop) {
  const int64_t n = h->n, rn = (int64_t)h->r * n;
  const int g = grid_for(n, RED_BLOCK, NODE_GRID);
  double* v = h->z.p;
  double* in = h->tmp.p;
  double* ynew = in + rn;
  const double step = 1.0 / (double)(h->r > 1 ? h->r : 1);
  k_fista_in<<<g, RED_BLOCK, 0, h->stream>>>(v, h->w.p, h->r, n, step, in);
  LAUNCH_CHECK(h);
  if (int e = sweep_exact(h, in, ynew, true)) return e;
  // momentum schedule on the host, in the reference's float arithmetic
  const double tm = h->fista_t;
  const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tm * tm));
  const double coef = (tm - 1.0) / tn;
  h->fista_t = tn;
  const int gr = grid_for(rn, RED_BLOCK, NODE_GRID);
  k_fista_mom<<<gr, RED_BLOCK, 0, h->stream>>>(h->y.p, v, ynew, rn, coef, h->parts.p);
  LAUNCH_CHECK(h);
  k_reduce_norm<<<1, 1024, 0, h->stream>>>(h->parts.p, gr, stop, 1);
  LAUNCH_CHECK(h);
  double* s = in;  // in is dead
  k_aggregate<<<g, RED_BLOCK, 0, h->stream>>>(h->y.p, h->r, n, s);
  LAUNCH_CHECK(h);
  return smooth_dual_dev(h, s, mon);
}
