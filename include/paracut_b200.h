/*
 * paracut_b200.h -- C ABI of the B200 AAR chain-prox path.
 *
 * Plain pointers and sizes only (no torch types); every function returns 0 on
 * success or a negative PCB_E* code, with a message in pcb_last_error()
 * (thread-local).  Host arrays are caller-owned and copied; device buffers
 * are owned by the opaque solver handle.  One handle = one CUDA stream; a
 * handle is not re-entrant, distinct handles may be used from distinct
 * threads.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/paracut/<file>:<line>); INTEGRATION.md shows the
 * ctypes binding a maintainer would add to the reference.
 */
#ifndef PARACUT_B200_H
#define PARACUT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCB_OK 0
#define PCB_E_ARG -1      /* invalid argument  -> ValueError in Python   */
#define PCB_E_CUDA -2     /* CUDA runtime error -> RuntimeError           */
#define PCB_E_STATE -3    /* call out of order  -> RuntimeError           */
#define PCB_E_NOMEM -4    /* device allocation failed -> MemoryError      */

/* connectivity codes, graph.py:18 CONNECTIVITIES order */
#define PCB_CONN_2D4 0
#define PCB_CONN_2D8 1
#define PCB_CONN_3D6 2

/* state precision
 * PCB_F64: AAR point z kept in fp64 and updated with the reference's exact
 *          operation order -> iterates bitwise equal to solvers.py:289-298.
 * PCB_F32: shadow p_j stored fp32, shared drift c fp64, primal x fp32;
 *          z_j = p_j + c; all prox arithmetic in fp64 (SURVEY 8(a) a6 form).
 * PCB_F64S: the PCB_F32 form with fp64 state and fp64 scans, chains split at
 *          merge points (not bitwise the reference; ~1e-12 relative). */
#define PCB_F64 0
#define PCB_F32 1
#define PCB_F64S 2

typedef struct pcb_solver pcb_solver;

const char *pcb_last_error(void);
int pcb_version(void);
int pcb_device_count(int *count);
/* Host helper (no device work): Jaccard distance 1 - |A & B| / |A | B| of two
 * np.packbits-packed labelings of nbytes bytes (0 when both are empty), the
 * trace column certify.py:68-78 / solvers.py:200-203 fill at finish. */
int pcb_jaccard_packed(const uint8_t *a, const uint8_t *b, int64_t nbytes, double *out);

/* ---- operator level ------------------------------------------------------
 * Replaces _kernels.prox_chains(node_idx, chain_ptr, edge_w, c_lo, c_hi, v,
 * out, as_projection) (_kernels.py:145-180).  Host buffers; chains
 * [c_lo, c_hi) of one CSR class; out[node_idx[..]] <- v - prox (projection)
 * or prox.  n = len(v) = len(out); edges of chain c start at
 * chain_ptr[c] - c (_kernels.py:171). */
int pcb_prox_chains(const int64_t *node_idx, const int64_t *chain_ptr, const double *edge_w,
                    int64_t c_lo, int64_t c_hi, int64_t n_nodes, int64_t n_idx,
                    int64_t n_edges, const double *v, double *out, int as_projection,
                    int device);

/* Replaces tv1d.tv1d_prox (tv1d.py:42-69) batched over a CSR of signals:
 * signal c is s[ptr[c]:ptr[c+1]], its weights a[ptr[c]-c : ptr[c+1]-c-1]. */
int pcb_tv1d_prox_batch(const double *s, const double *a, const int64_t *ptr, int64_t nchains,
                        double *x, int device);

/* Replaces projections.project_L (projections.py:107-122) for an arbitrary
 * decomposition: w[n], degree[n], support[r*n] (0/1), v[r*n] -> out[r*n],
 * lam_j = (v_j + (w - sum_k v_k) / d) * support_j.  PCB_E_ARG when w has
 * mass on a node of degree 0 (projections.py:115-117). */
int pcb_project_L(const double *w, const int64_t *degree, const uint8_t *support, int r,
                  int64_t n, const double *v, double *out, int device);

/* ---- grid solver ---------------------------------------------------------
 * Replaces GridEnergy + decompose_grid + the solve_aar loop
 * (graph.py:125-161, decompose.py:186-200, solvers.py:272-307).
 * dims: ndim = 2 or 3 sizes (C order); w: n unaries; dir_weights[k]: dense
 * per-direction arrays in graph.DIRECTIONS order with the shapes of
 * graph.direction_shape. */
int pcb_create(const int64_t *dims, int ndim, int conn, int precision, const double *w,
               const double *const *dir_weights, int device, pcb_solver **out);
/* Device ingest of a PCUT1B grid file (reference io.py:143-224 layout:
 * "PCUT1B", connectivity code u8, ndim u8, dims u64 LE, then w and each
 * direction array as LE fp64): the payload streams from the file through
 * pinned staging buffers into the handle's device arrays, with no host copy
 * of the instance.  Same handle as pcb_create; dims_out (3 entries), ndim_out
 * and conn_out (nullable) report the header.  PCB_E_ARG on a malformed file
 * (the reference's ValueError cases: bad magic, connectivity code, dimension
 * count, truncated header or payload). */
int pcb_create_from_file(const char *path, int precision, int device, pcb_solver **out,
                         int64_t *dims_out, int *ndim_out, int *conn_out);
/* Lambda path on a resident instance: every pairwise weight becomes
 * factor * (its value at creation), as scaled_pairwise (graph.py:182-187), with
 * the AAR state left in place -- the warm start of solve(g.scaled_pairwise(f),
 * warm_start=previous, force_warm=True) without re-uploading the instance. */
int pcb_scale_pairwise(pcb_solver *h, double factor);
int pcb_destroy(pcb_solver *h);
/* Device memory of destroyed handles stays mapped in a per-device pool for
 * the next handle; this returns it to the driver. */
int pcb_release_memory(int device);
/* Diagnostics: sweep counters (warp trips, lane gates, bends, tiles issued,
 * tiles retired) of a build compiled with -DPCB_COUNT; zeros otherwise. */
int pcb_debug_counters(uint64_t *out, int reset);
/* r (number of chain families) and n */
int pcb_shape(const pcb_solver *h, int *r, int64_t *n);
/* Use this CUDA stream (cudaStream_t as uintptr) for all later launches. */
int pcb_set_stream(pcb_solver *h, uintptr_t stream);
int pcb_synchronize(pcb_solver *h);

/* A second handle of the same instance in another precision, built on the
 * device from src's arrays (no host transfer), and the fused-form AAR state
 * (f32 / f64s: p_j, drift c; x = w - sum_j p_j recomputed) moved between two
 * such handles -- the f32 -> f64s hand-over of a polishing solve
 * (solvers.py:150-165 warm start, without the host round trip of get_z/set_z). */
int pcb_clone(const pcb_solver *src, int precision, pcb_solver **out);
int pcb_copy_state(pcb_solver *dst, const pcb_solver *src);
/* z0 = Pi_L(0) = w/r per class (solvers.py:284-285). */
int pcb_init_cold(pcb_solver *h);
/* Warm start / readback of the AAR point z, r*n fp64 class-major
 * (DualState.z, projections.py:28-44; solvers.py:150-165). */
int pcb_set_z(pcb_solver *h, const double *z);
int pcb_get_z(pcb_solver *h, double *z);

/* iters plain AAR iterations z <- z + Pi_L(2 Pi_K z - z) - Pi_K z
 * (solvers.py:295-298); step_norms (nullable, device-accumulated, copied
 * out at the end) receives ||z_{k+1} - z_k|| per iteration. */
int pcb_aar_run(pcb_solver *h, int64_t iters, double *step_norms);

/* Same with step flags (PCB_F32 only), for slab-sharded runs where one
 * rank's families live on two handles (include the cross-slab family on a
 * pencil handle): */
#define PCB_STEP_G_PRESET 1   /* G already holds d of other families: no FIRST role */
#define PCB_STEP_NO_UPDATE 2  /* no LAST role: drift/primal updated elsewhere      */
#define PCB_STEP_EXPORT_G 4   /* LAST stores its per-node g = sum_j d_j in G       */
#define PCB_STEP_NORM_RAW 8   /* step_norms receive sums of squares (partials)    */
int pcb_aar_step(pcb_solver *h, int64_t iters, int flags, double *step_norms);
/* Sweep only families whose bit is set (decompose_grid order). */
int pcb_set_family_mask(pcb_solver *h, unsigned mask);
/* x -= g; c += (x - g)/r on this handle's nodes, g a device pointer to n
 * floats (the exported g of the slab side, already in this handle's layout).
 * The LAST role's step-norm term sum(2 dc g + r dc^2) over the owned nodes
 * lands in norms[1] (PCB_BUF_NORMS). */
int pcb_apply_g(pcb_solver *h, uintptr_t g_dev);
/* The slab side of an overlapped sharded iteration in one pass: g = G + d_z
 * with d_z received from the pencils (device float[P][dz][cp]), applied as
 * pcb_apply_g does (norm term in norms[1]), and the new drift c written to
 * the slab -> pencil send buffer (device double[P][dz][cp], the pencils' node
 * order: they receive their drift instead of updating it).  Slabs without a
 * halo row (3D-6, 2D-4). */
int pcb_apply_g_exchange(pcb_solver *h, uintptr_t recv_dev, uintptr_t send_dev, int P, int dz,
                         int cp);
/* Nodes [n_own, n) of this handle are halo copies of nodes another shard
 * owns (2D-8 row slabs carry the next slab's first row for the zig-zag path
 * that straddles the boundary): pcb_check labels them (their edges to owned
 * nodes are this shard's) but leaves their unary / dual terms to the owner,
 * and pcb_apply_g leaves their norm term out.  n_own = n: no halo. */
int pcb_set_owned(pcb_solver *h, int64_t n_own);
/* Device pointer and element count of a handle buffer (for collectives). */
/* GPU-resident instance construction: the BASELINE synthetic
 * grid built in HBM -- image of nshapes disks / balls (centres nshapes x ndim,
 * radii, as instances.shapes_of draws them) plus the counter-based
 * N(0, 0.15^2) noise of `seed`, unaries and edge weights with the BASELINE
 * formulas, `integer` for the rounded variant, pairwise scale lam -- bit for
 * bit the arrays of paracut_b200/instances.py.  Replaces GridEnergy +
 * upload (graph.py:116-161) for generated instances. */
int pcb_create_synthetic(const int64_t* dims, int ndim, int conn, int nshapes,
                         const double* centres, const double* radii, uint64_t seed, double lam,
                         int integer, int precision, int device, pcb_solver** out);
/* The same for a box [origin, origin + extent) of the global grid gdims (a
 * rank's z-slab or pencil in a sharded run): the handle has `dims` (the box's
 * nodes in C order, possibly flattened), node values from global coordinates
 * and global noise indices, the box's internal edges for the directions in
 * dir_mask (bit k = DIRECTIONS[conn][k]) and zero weights elsewhere. */
int pcb_create_synthetic_box(const int64_t* gdims, int ndim, int conn, const int64_t* origin,
                             const int64_t* extent, const int64_t* dims, unsigned dir_mask,
                             int nshapes, const double* centres, const double* radii,
                             uint64_t seed, double lam, int integer, int precision, int device,
                             pcb_solver** out);
/* The handle's instance back on the host (w: n doubles; dir_weights[k]: the
 * direction arrays in graph.direction_shape order, as currently scaled; NULL
 * entries skipped). */
int pcb_get_instance(pcb_solver* h, double* w, double* const* dir_weights);

/* Verified sweeps of the double-buffered fp32 step:
 * per family (r entries each, NULL allowed) the current mode (1 = the next
 * plain iteration verifies last iteration's segmentation, 0 = taut-string
 * scan, -1 = family always scans), how many sweeps ran verified so far and
 * how many chains those repaired locally, how many ran as scans and in how
 * many chains those changed the segmentation.  Diagnostics; syncs the stream. */
int pcb_verify_stats(pcb_solver* h, int* modes, int64_t* sweeps, int64_t* repaired,
                     int64_t* scans, int64_t* changed);

#define PCB_BUF_G 0      /* float[n] accumulator / exported g */
#define PCB_BUF_X 1      /* float[n] primal                  */
#define PCB_BUF_C 2      /* double[n] drift                  */
#define PCB_BUF_Y 3      /* double[r*n] shadow               */
#define PCB_BUF_NORMS 4  /* double[] per-iteration norms      */
#define PCB_BUF_P 5      /* float[r*n] fp32 family state (family layout) */
#define PCB_BUF_BITS 6   /* uint8[n] last check's labels, bit t = threshold t */
int pcb_device_buffer(pcb_solver *h, int which, uintptr_t *ptr, int64_t *count);

/* Shadow y = Pi_K(z) into the handle's shadow buffer (projections.py:89-104);
 * does not change z.  y_out (nullable, r*n) and s_out (nullable, n,
 * aggregate in class order, projections.py:133-137) are copied to host. */
int pcb_shadow(pcb_solver *h, double *y_out, double *s_out);
/* Copy the current shadow (from the last pcb_shadow*) to host without
 * recomputing it (final DualState.y, solvers.py:307). */
int pcb_shadow_get(pcb_solver *h, double *y_out);
/* pcb_shadow plus *delta = ||y_new - y_prev|| against the shadow that was
 * current before the call (-1 if there was none): the dual_tol test of
 * solvers.py:300-306. */
int pcb_shadow_delta(pcb_solver *h, double *delta);
/* Apply one AAR update using the current shadow (after pcb_shadow):
 * z <- z + Pi_L(2y - z) - y; writes ||dz|| to *step_norm (nullable). */
int pcb_apply(pcb_solver *h, double *step_norm);

/* Certificates on the current shadow (solvers.py:170-182, certify.py:31-47):
 * x = w - s, labels_t = (x > thr[t]) for nthr <= 8 thresholds; per threshold
 * energy f(lab) - w.lab, gap = energy - sum min(s - w, 0); *dual_obj =
 * 0.5||w||^2 - 0.5||s - w||^2.  Labels and x stay on device ("current"). */
int pcb_check(pcb_solver *h, int nthr, const double *thr, double *energy, double *gap,
              double *dual_obj);
/* Copy the current check's labels for threshold t (uint8[n], or packed bits
 * MSB-first like np.packbits when packed=1) and x (fp64[n]) to host (each nullable). */
int pcb_get_check(pcb_solver *h, int t, uint8_t *labels, int packed, double *x);
/* Solve log (extension; replaces per-check host copies with one read at the
 * end, as solvers.py:170-209 only needs them in finish()):
 *   pcb_log_start     start logging (clears the log): pcb_aar_run / pcb_apply
 *                     called with a NULL step_norms append their step norms
 *                     to a device log instead of the handle's scratch slot
 *   pcb_log_stop      stop logging (the log stays readable)
 *   pcb_log_norms     copy min(cap, count) logged norms to out; *count = total
 *   pcb_log_labels    append the current check's packed labels for threshold
 *                     t (np.packbits order) to the device log; *slot = index
 *   pcb_log_label_get copy one logged labeling (packed, (n+7)/8 bytes) to host
 *   pcb_log_jaccard   out[i] = jaccard_distance(slot i, ref) for every slot
 *                     (certify.py:68-78 on packed bits, exact integer counts) */
int pcb_log_start(pcb_solver *h);
int pcb_log_stop(pcb_solver *h);
int pcb_log_norms(pcb_solver *h, double *out, int64_t cap, int64_t *count);
int pcb_log_labels(pcb_solver *h, int t, int64_t *slot);
int pcb_log_label_get(pcb_solver *h, int64_t slot, uint8_t *packed);
int pcb_log_jaccard(pcb_solver *h, const uint8_t *ref_packed, double *out, int64_t cap);
/* Keep the current check as the best iterate / fetch the kept one. */
int pcb_keep_best(pcb_solver *h, int t);
int pcb_get_best(pcb_solver *h, uint8_t *labels, double *x);

/* The reference's other dual schemes on the same kernels (fp64 handles;
 * iterates bitwise equal to the reference):
 *   PCB_ALG_BCD   solve_bcd   solvers.py:212-243  cyclic block projections
 *   PCB_ALG_AP    solve_ap    solvers.py:246-269  alternating projections
 *   PCB_ALG_FISTA solve_fista solvers.py:310-341  accelerated projected gradient
 * pcb_dual_init sets the iterate y (host r*n, or NULL for zeros; FISTA also
 * v = y, t = 1).  pcb_dual_run performs `iters` iterations; monitor[k]
 * (nullable) receives the reference's per-iteration monitor value (BCD and
 * FISTA: "dual_objective", AP: "ap_distance") and stop[k] (nullable) the
 * dual_tol quantity (BCD: sqrt(change2), AP: |y - yprev|, FISTA: |dy|).
 * Afterwards pcb_check / pcb_shadow_get read y, and pcb_get_z reads lam (AP)
 * or v (FISTA).  pcb_init_cold / pcb_set_z return the handle to AAR. */
#define PCB_ALG_BCD 1
#define PCB_ALG_AP 2
#define PCB_ALG_FISTA 3
int pcb_dual_init(pcb_solver *h, int alg, const double *y0);
int pcb_dual_run(pcb_solver *h, int64_t iters, double *monitor, double *stop);

/* Best level set of a TV solution (best_level_set_gap, certify.py:50-65 over
 * solvers.level_sets, solvers.py:86-97): of the labelings {x > v}, v over the
 * distinct values of x, and the all-ones labeling, the one of least energy
 * (hence least gap for any dual).  x: host fp64[n], or NULL for the x of the
 * current check.  *u receives v (-inf for all ones): the labeling is
 * x > *u, so pcb_check with threshold *u certifies it with the deterministic
 * reductions.  *energy (nullable) receives its energy from the one-sort scan
 * (fp64 atomics: exact for integer weights, last-bit rounding otherwise). */
int pcb_level_set(pcb_solver *h, const double *x, double *u, double *energy);

/* Pi_K of an arbitrary r*n host vector with this grid's decomposition
 * (project_K, projections.py:89-104); fp64 exact kernels regardless of the
 * handle precision. */
int pcb_project_K(pcb_solver *h, const double *v, double *out);

/* Plain iterations of the f32 / f64s paths replay as CUDA graphs of 8
 * iterations once the handle has run `iters` of them eagerly (default 64:
 * capture and instantiation cost about as much as the replays save over 80
 * iterations, so short solves stay eager).  0 = capture on the first block
 * (steady-state measurements).  No reference counterpart: the reference loop
 * (solvers.py:289-298) has no launch overhead to hide. */
int pcb_set_graph_after(pcb_solver *h, int64_t iters);

/* Kernel timing for the roofline: while enabled, every chain-family prox
 * launch is bracketed by CUDA events on the handle stream; pcb_profile_read
 * synchronises, returns summed milliseconds and launch counts per family
 * (r entries each, family order of decompose_grid) and clears the record. */
int pcb_set_profiling(pcb_solver *h, int on);
int pcb_profile_read(pcb_solver *h, double *ms, int64_t *launches);

/* Launch counting for the bench contract: kernels launched since the last
 * reset (our kernels only). */
int64_t pcb_launch_count(const pcb_solver *h);
void pcb_reset_launch_count(pcb_solver *h);

#ifdef __cplusplus
}
#endif
#endif
