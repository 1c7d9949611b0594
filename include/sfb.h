/*
 * sfb.h — C ABI of the B200-native BundleFusion pose solver (libsfb.so).
 *
 * The reference (scanfuse 0.1.0, /root/reference/pkg/src/scanfuse/solver.py)
 * is pure Python/NumPy and has no FFI layer of its own; its boundary is the
 * Python API of `scanfuse.solver`.  This header is what that API binds
 * through ctypes (paper_1604_01093_b200/_abi.py).  Every entry point names the
 * reference function(s) it replaces.
 *
 * Conventions
 *  - Every function returns int status: SFB_OK (0) or an SFB_E_* code.  No C++
 *    exception crosses the ABI; the message of the last failure on a handle is
 *    sfb_last_error(handle) (thread-local fallback when handle is NULL).
 *  - Host pointers are borrowed for the duration of the call only.  Device
 *    memory is owned by the handle that allocated it.
 *  - One CUDA stream per problem handle; frames in a context are read-only
 *    after upload, so problems created on one context may run concurrently
 *    (reference contract solver.py:551-552).
 *  - Frames are addressed by context slot; inside a problem, frames are
 *    addressed by their position k in frame_ids (k = 0 is the gauge anchor,
 *    variable block k-1 otherwise; reference solver.py:561-562).
 */
#ifndef SFB_H_
#define SFB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFB_ABI_VERSION 1

enum {
  SFB_OK = 0,
  SFB_E_ARG = 1,            /* invalid argument / shape                     */
  SFB_E_CUDA = 2,           /* CUDA runtime / launch failure                */
  SFB_E_OOM = 3,            /* device allocation failed                     */
  SFB_E_PCG_NONFINITE = 4,  /* PcgDivergenceError (solver.py:30-31,488-499) */
  SFB_E_STATE = 5           /* call out of order (e.g. PCG before linearize) */
};

typedef struct sfb_ctx sfb_ctx;
typedef struct sfb_problem sfb_problem;

/* One CachedFrame (reference frames.py:38-50): the planes the solver reads.
 * All planes are row-major (h, w[, c]) and C-contiguous. */
typedef struct {
  int32_t width, height;
  double fx, fy, cx, cy;          /* intrinsics_low                         */
  const uint8_t* valid_depth;     /* (h, w) bool                             */
  const uint8_t* valid_normal;    /* (h, w) bool                             */
  const float* points;            /* (h, w, 3) points_low                    */
  const float* normals;           /* (h, w, 3) normals_low                   */
  const float* grad;              /* (h, w, 2) grad_low                      */
} sfb_frame_desc;

/* EnergyWeights (solver.py:34-46) minus the ramp, which stays on the host. */
typedef struct {
  double sparse, photo, geo;
} sfb_weights;

/* SolverConfig (solver.py:56-69) fields the device path needs. */
typedef struct {
  double geo_distance_max;        /* 0.15 */
  double geo_normal_min;          /* 0.9  */
  int32_t dense_pixel_stride;     /* 1    */
  int32_t dense_bidirectional;    /* 0    */
} sfb_config;

/* Rounding conventions of the host BLAS the reference runs on (see
 * paper_1604_01093_b200/_rounding.py).  Each code is a permutation index
 * 0..5 of the 3-term FMA chain fma(a_k b_k, fma(a_j b_j, a_i b_i)); they make
 * the frame-pair filter and the association gates bit-exact with NumPy. */
typedef struct {
  int32_t matvec_c;   /* (3,3) C-contiguous @ (3,)                            */
  int32_t matvec_f;   /* (3,3) F-contiguous @ (3,)                            */
  int32_t gemm33;     /* (3,3) @ (3,3)                                        */
  int32_t apply_n;    /* (m,3) @ (3,3).T for m > 1                            */
  int32_t apply_1;    /* (1,3) @ (3,3).T                                      */
  int32_t dot3;       /* np.dot of two 3-vectors                              */
} sfb_rounding;

/* Per-GN-iteration scalars of the fused iteration (IterationRecord inputs). */
typedef struct {
  double e_sparse, e_photo, e_geo;              /* raw sums at linearization   */
  int32_t pcg_iterations;
  int32_t pcg_status;                           /* SFB_OK or SFB_E_PCG_NONFINITE */
  double pcg_relative;
  double step_norm;
  double ea_sparse, ea_photo, ea_geo;           /* frozen-association sums     */
} sfb_iter_result;

const char* sfb_last_error(const void* handle);
int sfb_abi_version(void);

/* ---- context + frame store ------------------------------------------- */
int sfb_ctx_create(int32_t device, sfb_ctx** out);
int sfb_ctx_destroy(sfb_ctx* ctx);
int sfb_ctx_set_rounding(sfb_ctx* ctx, const sfb_rounding* r);
/* Upload n CachedFrames (frames.py:38-50); one slot per frame.  Replaces the
 * per-call `.astype(np.float64)` plane reads of solver.py:219-251,268-272. */
int sfb_frames_upload(sfb_ctx* ctx, int32_t n, const sfb_frame_desc* descs,
                      int32_t* slots_out);
int sfb_frames_release(sfb_ctx* ctx, int32_t n, const int32_t* slots);

/* page-locked host memory (cudaMallocHost) for reusable staging buffers */
int sfb_host_alloc(int64_t bytes, void** ptr);
int sfb_host_free(void* ptr);

/* ---- build_cache (frames.py:75-151) on the device ---------------------- */
/* n RGB-D frames of width x height (colour (H, W, 3) uint8, depth (H, W)
 * float32; host pageable, pinned, or device pointers) -> their CachedFrame
 * planes at low_width x low_height, bit-identical to the reference's NumPy
 * float32 pipeline (block-mean luminance, block-median depth, unprojection,
 * central-difference normals, gradient).  k_low = intrinsics.scaled(low_w,
 * low_h) as (fx, fy, cx, cy); luma_order = the host's float32 BLAS FMA chain
 * order of RgbdFrame.luminance (sfb_rounding code).  The planes become
 * resident frame slots (slots_out, with intensity_low attached, as if
 * uploaded by sfb_frames_upload + sfb_frames_set_intensity) and are copied
 * to host_out: per frame 42*h*w bytes = intensity f32 | depth f32 |
 * points f32x3 | normals f32x3 | grad f32x2 | valid_depth u8 | valid_normal u8.
 * Blocks of at most 64 samples.  Synchronous. */
int sfb_build_cache(sfb_ctx* ctx, int32_t n, int32_t width, int32_t height, int32_t low_width,
                    int32_t low_height, const uint8_t* const* colors, const float* const* depths,
                    const double* k_low, int32_t luma_order, void* host_out, int32_t* slots_out);

/* ---- hashed TSDF volume (tsdf.py:55-267) ------------------------------ */
/* TsdfVolume(voxel_size, truncation, depth_weighting): 8x8x8-voxel blocks of
 * float32 accumulators (weight, weight*distance, weight*colour) in a device
 * pool; the block dictionary (key -> slot, insertion order) is host memory of
 * the handle.  Synchronous calls on the context's stream. */
typedef struct sfb_tsdf sfb_tsdf;
int sfb_tsdf_create(sfb_ctx* ctx, double voxel_size, double truncation, int32_t depth_weighting,
                    sfb_tsdf** out);
int sfb_tsdf_destroy(sfb_tsdf* t);
/* integrate (sign +1) / deintegrate (sign -1) one RGB-D frame (tsdf.py:90-160):
 * colour (H, W, 3) uint8, depth (H, W) float32, k4 = (fx, fy, cx, cy),
 * pose = camera -> world (row-major R, t) with pose_ord = NumPy's FMA order of
 * (m,3) @ R.T for its layout and m = #valid depth pixels; inv_R/inv_t =
 * pose.inverse() as NumPy computes it (C-ordered, inv_ord); tvals =
 * np.linspace(0, 1, n_samples) (_touched_blocks, :162-181).  *status: 0 ok,
 * 1 "frame has no integrated content", 2 "block err_coord missing during
 * de-integration", 3 "negative weight in block err_coord" - the reference's
 * DeintegrationMismatchError, raised at the same block with the same partial
 * update applied before it. */
int sfb_tsdf_apply(sfb_tsdf* t, int32_t sign, int32_t width, int32_t height, const uint8_t* color,
                   const float* depth, const double* k4, const double* pose_R, const double* pose_t,
                   int32_t pose_ord, const double* inv_R, const double* inv_t, int32_t inv_ord,
                   const double* tvals, int32_t n_samples, int32_t* status, int64_t* err_coord);
int sfb_tsdf_count(sfb_tsdf* t, int64_t* n_blocks);
/* all blocks in insertion order: coords (n,3) int64, weight/wdist (n,512), wcolor (n,512,3) */
int sfb_tsdf_export(sfb_tsdf* t, int64_t n, int64_t* coords, float* weight, float* wdist,
                    float* wcolor);
/* insert or overwrite blocks (TsdfVolume.allocate, load_volume) */
int sfb_tsdf_import(sfb_tsdf* t, int64_t n, const int64_t* coords, const float* weight,
                    const float* wdist, const float* wcolor);
int sfb_tsdf_get_block(sfb_tsdf* t, const int64_t* coord, int32_t* found, float* weight,
                       float* wdist, float* wcolor);

/* ---- dense_verify (filters.py:216-277) --------------------------------- */
/* Gates of FilterConfig (filters.py:41-43) and NumPy's FMA chain order of
 * (m,3) @ R.T (RigidTransform.apply, geometry.py:139-142) for a C- or
 * F-ordered rotation at m > 1 / m == 1 (sfb_rounding codes, host probe). */
typedef struct {
  double depth_max;   /* verify_depth_max  */
  double normal_min;  /* verify_normal_min */
  double color_max;   /* verify_color_max  */
  int32_t apply_n, apply_1, apply_nf, apply_1f;
} sfb_verify_config;
/* Attach CachedFrame.intensity_low ((h, w) f32, frames.py:38-50) to resident
 * slots; only dense_verify reads it, so the solver path never uploads it. */
int sfb_frames_set_intensity(sfb_ctx* ctx, int32_t n, const int32_t* slots,
                             const float* const* intensity);
/* n_items directions of dense_verify, one CTA each: item k reprojects slot
 * src_slots[k] into dst_slots[k] (_verify_one_direction, filters.py:216-250)
 * with the transform (R9[9k..] row-major rotation, t3[3k..] translation):
 * flags[k] bit 0 = use its inverse() (geometry.py:135-137, evaluated with
 * NumPy's rounding: the j -> i direction of filters.py:268), bit 1 = the
 * caller's rotation array is Fortran-ordered (selects the rounding order).
 * Outputs per item: mean_error (the NumPy pairwise sum of the good distances
 * in row-major order / count) and the count, both bit-exact.  The pass/fail
 * rule (filters.py:269-276) is host arithmetic on these.  Synchronous; source
 * frames of <= 25,600 pixels. */
int sfb_dense_verify(sfb_ctx* ctx, int32_t n_items, const int32_t* src_slots,
                     const int32_t* dst_slots, const double* R9, const double* t3,
                     const uint8_t* flags, const sfb_verify_config* cfg, double* err_out,
                     int64_t* count_out);

/* ---- problem (AlignmentProblem.__init__, solver.py:554-564) ----------- */
/* n_frames problem frames (slots may be NULL when no caches); n_sets
 * correspondence sets (CorrespondenceSet, filters.py:50-66) given as
 * problem-frame indices and offsets into the stacked (N,3) point arrays,
 * i.e. build_sparse_term (solver.py:89-111). */
int sfb_problem_create(sfb_ctx* ctx, int32_t n_frames, const int32_t* slots,
                       int32_t n_sets, const int32_t* set_frame_i,
                       const int32_t* set_frame_j, const int64_t* set_offsets,
                       const double* points_i, const double* points_j,
                       sfb_problem** out);
/* Attach the frames to a problem created with slots == NULL (the caller
 * builds the problem while the frames upload is still in flight; the same
 * state as passing the slots to sfb_problem_create).  Once only, before any
 * dense call. */
int sfb_problem_attach_frames(sfb_problem* p, const int32_t* slots);
int sfb_problem_destroy(sfb_problem* p);
int sfb_problem_stream(sfb_problem* p, void** stream_out);

/* Poses: R row-major (n,3,3), t (n,3).  f_layout[k] = 1 when the host
 * rotation array is Fortran-ordered (changes NumPy's inverse() rounding). */
int sfb_set_poses(sfb_problem* p, const double* R, const double* t,
                  const uint8_t* f_layout);
int sfb_get_poses(sfb_problem* p, double* R, double* t);
int sfb_save_best(sfb_problem* p);     /* best_poses = dict(self.poses)   */
int sfb_restore_best(sfb_problem* p);  /* self.poses = best_poses          */

/* build_dense_edges (solver.py:130-148) + view_angle_deg/frustum_overlap
 * (frames.py:154-188), bit-exact.  view_cos_min is the smallest cosine c with
 * degrees(arccos(c)) < view_angle_max_deg under NumPy (host bisection). */
int sfb_build_dense_edges(sfb_problem* p, double view_cos_min, int64_t* n_edges);
int sfb_get_dense_edges(sfb_problem* p, int32_t* pairs_out /* 2*n_edges */);
int sfb_set_dense_edges(sfb_problem* p, int64_t n_edges, const int32_t* pairs);
/* frustum_overlap(cache_a, pose_a, cache_b, pose_b) for many (a,b) pairs of
 * problem frames at the current poses: fraction in [0,1] (frames.py:154-180). */
int sfb_frustum_overlap(sfb_problem* p, int64_t n_pairs, const int32_t* pairs,
                        double* overlap_out);

/* normal_equations (solver.py:630-660): sparse state, dense association +
 * linearization, and the block system; energies are raw sums (host applies
 * the weights exactly as solver.py:646,655 do). */
int sfb_linearize(sfb_problem* p, const sfb_weights* w, double w_dense,
                  const sfb_config* cfg, double energies_out[3]);
/* pcg_solve (solver.py:463-508), scalar-Jacobi, exact recurrence. */
int sfb_pcg(sfb_problem* p, int32_t max_iterations, double tolerance,
            int32_t restart_interval, int32_t* iterations, double* relative,
            int32_t* status);
/* The PCG solution dx of the last sfb_pcg / sfb_gn_iteration (n_vars). */
int sfb_get_solution(sfb_problem* p, double* x);
/* pcg_solve on a duck-typed host system (.rhs/.diagonal/.apply, the
 * reference's test DenseSystem, test_solver.py:282-292): A is the dense
 * (n,n) row-major operator, same device recurrence as sfb_pcg. */
int sfb_pcg_dense(sfb_ctx* ctx, int32_t n, const double* A, const double* rhs,
                  const double* diagonal, int32_t max_iterations, double tolerance,
                  int32_t restart_interval, double* x_out, int32_t* iterations,
                  double* relative, int32_t* status);
/* _apply_step (solver.py:674-677): T <- exp(dx) o T for every variable frame. */
int sfb_apply_step(sfb_problem* p, double* step_norm);
/* _energy_with_frozen_associations (solver.py:662-672): raw sums. */
/* One GN iteration after a linearisation with ONE host round trip
 * (AlignmentProblem.solve, solver.py:715-750): pcg_solve -> _apply_step
 * (skipped on the device when the PCG diverged) -> the frozen energy at the
 * new poses, fused with the next linearisation (w_dense_next) when
 * relinearize != 0.  out[0] PCG iterations, [1] relative residual, [2] 1 if
 * PcgDivergenceError, [3] step norm, [4..6] energy after (sparse, photo,
 * geo raw sums), [7..9] the next linearisation's raw sums. */
int sfb_gn_step(sfb_problem* p, int32_t pcg_max_it, double pcg_tol, int32_t pcg_restart,
                const sfb_weights* w, int32_t prev_dense, int32_t relinearize,
                double w_dense_next, const sfb_config* cfg, double out[10]);
/* The same split around the sharded exchange (paper_1604_01093_b200.shard):
 * _begin enqueues everything up to the per-edge sums and reports which
 * exchange buffers (bit 0: dense edge sums, bit 1: frozen-energy sums) the
 * caller must sum across ranks on the problem's stream before _end. */
int sfb_gn_step_begin(sfb_problem* p, int32_t pcg_max_it, double pcg_tol, int32_t pcg_restart,
                      const sfb_weights* w, int32_t prev_dense, int32_t relinearize,
                      double w_dense_next, const sfb_config* cfg, int32_t* exchange);
int sfb_gn_step_end(sfb_problem* p, double out[10]);
int sfb_energy_frozen(sfb_problem* p, int32_t dense, double energies_out[3]);
/* E_after of the previous GN iteration and the next linearisation at the
 * same (current) poses in one fused pass (solver.py:662-672 then :630-660):
 * out = {E_sparse, E_photo_frozen, E_geo_frozen, E_sparse, E_photo, E_geo}. */
int sfb_energy_and_linearize(sfb_problem* p, const sfb_weights* w, int32_t prev_dense,
                             double w_dense_next, const sfb_config* cfg, double out6[6]);
/* One full GN iteration without intermediate host syncs:
 * linearize -> pcg -> step -> frozen energy (solver.py:700-724). */
int sfb_gn_iteration(sfb_problem* p, const sfb_weights* w, double w_dense,
                     const sfb_config* cfg, int32_t pcg_max_iterations,
                     double pcg_tolerance, int32_t pcg_restart_interval,
                     sfb_iter_result* out);

/* ---- host views of the linearized system (NormalEquations accessors) --- */
int sfb_system_dims(sfb_problem* p, int32_t* n_vars, int64_t* n_pairs,
                    int64_t* n_corr);
/* NormalEquations.apply (solver.py:403-410). */
int sfb_matvec(sfb_problem* p, const double* x, double* y);
/* gradient, Jacobi diagonal (solver.py:412-428). */
int sfb_get_gradient(sfb_problem* p, double* g);
int sfb_get_diagonal(sfb_problem* p, double* d);
/* block system: diag blocks (n_vars/6,6,6), pair blocks (n_pairs,6,6) with
 * their (row var, col var) ids — used by materialize() (solver.py:446-454). */
int sfb_get_blocks(sfb_problem* p, double* diag_blocks, double* pair_blocks,
                   int32_t* pair_vars);
/* world_i, world_j of the sparse state (solver.py:568-580). */
int sfb_get_sparse_world(sfb_problem* p, double* world_i, double* world_j);
/* eval_sparse residuals at current poses (solver.py:114-123), (N,3). */
int sfb_sparse_residuals(sfb_problem* p, double* res_out);
/* per-set max residual norm (max_residual_set, solver.py:765-776). */
int sfb_sparse_set_max(sfb_problem* p, double* set_max_out);

/* ---- per-edge evaluators (solver.py:216-349) ----------------------------
 * associate_photo / associate_geo (solver.py:216-260) for one directed edge
 * i->j of problem frames at the current poses.  kind 0 = photo, 1 = geo.
 * Per-source-pixel outputs (h_i*w_i, row-major), honouring the pixel stride
 * of _source_pixel_data (solver.py:158-167):
 *   sel[px] = 1 when the pixel belongs to the association
 *   tgt[px] = associated target pixel index (geo) or -1                     */
int sfb_associate(sfb_problem* p, int32_t frame_i, int32_t frame_j,
                  int32_t kind, const sfb_config* cfg, uint8_t* sel,
                  int32_t* tgt);
/* photo_residuals / photo_linearize (kind 0; aux = reference (m,2)) and
 * geo_residuals / geo_linearize (kind 1; aux = normals (m,3), targets (m,3))
 * on explicit association arrays (solver.py:263-328).  res is (m,2) or (m,);
 * jac (optional, may be NULL) is J_i as (m,2,6) or (m,6); J_j = -J_i. */
int sfb_point_eval(sfb_problem* p, int32_t frame_i, int32_t frame_j,
                   int32_t kind, int64_t m, const double* points,
                   const double* aux, const double* targets, double* res,
                   double* jac);

/* Drop correspondence sets from a live problem (solve_with_pruning,
 * solver.py:779-816, removes the worst set each round).  The surviving sets
 * keep their order and are renumbered 0..n-1 (set ids of later calls refer
 * to the compacted list); their correspondences stay resident and the block
 * structure is rebuilt on the device.  The problem is then exactly one
 * created from the surviving sets. */
int sfb_problem_drop_sets(sfb_problem* p, int64_t n, const int32_t* set_ids);

/* PCG preconditioner of this problem (every later sfb_pcg / GN step):
 * 0 = scalar Jacobi, the reference's pcg_solve (solver.py:477, default);
 * 1 = block Jacobi, the inverse of each variable's 6x6 diagonal block of A
 *     (opt-in performance mode: NOT the reference's recurrence, so results
 *     differ from the reference beyond rounding). */
int sfb_set_preconditioner(sfb_problem* p, int32_t kind);

/* ---- data-parallel sharding over frame pairs -----
 * A problem replicated on world ranks (one process per GPU) owns every
 * world-th directed dense edge and every world-th filter candidate.  The
 * two-phase calls below bracket the one collective of each step: after a
 * _begin, the caller sums the indicated exchange buffers across ranks
 * (bit 0: which=0 per-edge linearisation sums, 32 f64 per directed edge;
 * bit 1: which=1 per-edge frozen energies, 2 f64 per directed edge; the
 * filter always exchanges which=2, one u8 pass flag per candidate).  Every
 * entry has exactly one owner, so the sums are exact and every rank ends
 * with bit-identical systems; the PCG then runs replicated.
 * The single-call forms above return SFB_E_STATE on a sharded problem. */
int sfb_set_shard(sfb_problem* p, int32_t rank, int32_t world);

/* Sharded-PCG mode: mode 1 keeps each rank's system
 * PARTIAL - its own directed edges, and the correspondence sets on rank 0 -
 * instead of exchanging the per-edge sums (mode 0, default).  A
 * linearisation is then sfb_linearize_begin (exchange mask 0) ->
 * sfb_linearize_end_system -> sum exchange buffer 3 ([g | Jacobi diagonal |
 * dense energies | diagonal blocks when block-Jacobi]) -> sfb_linearize_finish,
 * and the PCG is sfb_pcg_sharded: per iteration one all-reduce of the
 * n_vars partial A.p through the caller's callback, which must sum the
 * device buffer across ranks in place, ordered on `stream`, and return 0.
 * Every rank then runs pcg_solve's scalar recurrence on identical bits. */
/* Peer-memory exchange of the per-edge sums (mode 0, ranks on one node): each
 * rank exports CUDA IPC handles of its per-edge buffer (which 0) and of a
 * 64-slot flag buffer (which 1), every rank attaches all of them (64-byte
 * handles, indexed by rank), and with sfb_set_p2p(p, 1) the edge reduction
 * stores each owned edge's sums straight into every peer's buffer, followed
 * by a device-side barrier over the flags (system-scope release/acquire):
 * no host collective for exchange buffer 0 (the _begin calls stop asking for
 * it).  Re-attach buffer 0 after every sfb_build_dense_edges_end (the buffer
 * may be reallocated). */
int sfb_ipc_export(sfb_problem* p, int32_t which, void* handle64, int64_t* bytes);
int sfb_ipc_attach(sfb_problem* p, int32_t which, int32_t world, const void* handles);
int sfb_set_p2p(sfb_problem* p, int32_t on);

typedef int (*sfb_allreduce_fn)(void* user, double* dev_buf, int64_t n, void* stream);
int sfb_set_shard_mode(sfb_problem* p, int32_t mode);
int sfb_linearize_end_system(sfb_problem* p);
int sfb_linearize_finish(sfb_problem* p, double e3[3]);
int sfb_pcg_sharded(sfb_problem* p, int32_t max_it, double tol, int32_t restart,
                    sfb_allreduce_fn fn, void* user, int32_t* iters, double* rel, int32_t* status);
int sfb_exchange_buffer(sfb_problem* p, int32_t which, void** dev_ptr, int64_t* bytes);
int sfb_build_dense_edges_begin(sfb_problem* p, double view_cos_min);
int sfb_build_dense_edges_end(sfb_problem* p, int64_t* n_edges);
int sfb_linearize_begin(sfb_problem* p, const sfb_weights* w, double w_dense,
                        const sfb_config* cfg, int32_t* exchange);
int sfb_linearize_end(sfb_problem* p, double energies_out[3]);
int sfb_energy_and_linearize_begin(sfb_problem* p, const sfb_weights* w, int32_t prev_dense,
                                   double w_dense_next, const sfb_config* cfg,
                                   int32_t* exchange);
int sfb_energy_and_linearize_end(sfb_problem* p, double out6[6]);
int sfb_energy_frozen_begin(sfb_problem* p, int32_t dense, int32_t* exchange);
int sfb_energy_frozen_end(sfb_problem* p, double energies_out[3]);

/* ---- measurement (bench.py) -------------------------------------------
 * Per-kernel-class device time measured with CUDA events on the problem's
 * stream.  Classes: 0 dense linearize, 1 frozen energy, 2 PCG, 3 pair filter,
 * 4 sparse term, 5 assembly, 6 pose update, 7 other. */
#define SFB_PROF_CLASSES 8
int sfb_profile(sfb_problem* p, int32_t enable);
int sfb_profile_read(sfb_problem* p, double* ms, int64_t* launches, int32_t reset);
/* Kernels launched by this library since load (all handles). */
int sfb_launch_count(int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* SFB_H_ */
