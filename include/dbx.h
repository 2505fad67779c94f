/*
 * dbx.h — C-ABI of the B200-native anti-reflective (AR) deblurring hot path.
 *
 * The reference (`deblur`, a header-only C++20 library under
 * /root/reference/proj/include/deblur) exposes this path as value-semantics
 * C++ functions over Eigen row-major double matrices.  This C-ABI is the
 * drop-in boundary for that path: plain pointers and sizes, opaque plan
 * handles, status codes instead of exceptions.  include/deblur_b200.hpp
 * re-creates the reference's C++ names on top of it.
 *
 * Conventions (all entry points):
 *   - arrays are FP64, row-major, ld = n2 (reference core.hpp:17-19: vec(X)
 *     is the row-major buffer); batched arrays are image-major with stride
 *     n1*n2;
 *   - every array pointer may be HOST or DEVICE memory (detected with
 *     cudaPointerGetAttributes); host arrays are staged through the plan's
 *     device buffers, device arrays are used in place;
 *   - status: DBX_OK = 0, DBX_EINVAL = 1 (reference std::invalid_argument,
 *     core.hpp:26-28), DBX_EDIVERGED = 2 (reference SolverDivergence,
 *     solver.hpp:42-44), DBX_ECUDA = 3 (device/driver error or missing
 *     sm_100a device: there is no CPU fallback);
 *   - dbx_last_error() returns the thread-local message of the last failure
 *     (the reference exception's what()).
 *   - one plan per stream; plans are independent and there is no global lock
 *     (replaces the reference's process-wide FFTW mutex, transforms.hpp:21-26).
 */
#ifndef DBX_H_
#define DBX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBX_OK 0
#define DBX_EINVAL 1
#define DBX_EDIVERGED 2
#define DBX_ECUDA 3

/* boundary.hpp:9 BoundaryCondition order {Zero, Periodic, Reflective, AntiReflective};
 * this path implements AntiReflective only. */
#define DBX_BC_REFLECTIVE 2     /* BoundaryCondition::Reflective (DCT-III algebra) */
#define DBX_BC_ANTIREFLECTIVE 3

/* transforms.hpp:17 TransformKind order {Dft, CosineIII, SineI, AntiReflective,
 * AntiReflectiveInverse}; the AR path needs the last three. */
#define DBX_KIND_COSINE3 1   /* R (cosine3_forward, transforms.hpp:88-99), reflective BCs */
#define DBX_KIND_SINEI 2
#define DBX_KIND_AR 3
#define DBX_KIND_ARINV 4

/* solver.hpp:17-32 StoppingRule::Kind order {FixedIterations, MinRre,
 * RelativeResidualBelow}. */
#define DBX_STOP_FIXED 0
#define DBX_STOP_MINRRE 1
#define DBX_STOP_RESIDUAL 2

/* Blur-apply engine selection (dbx_plan_set_conv). AUTO mirrors the
 * reference's direct/FFT cutover at q = 7 (blur.hpp:70, 79-81). */
#define DBX_CONV_AUTO 0
#define DBX_CONV_DIRECT 1
#define DBX_CONV_FFT 2
#define DBX_CONV_FFT_DENSE 3  /* FFT engine with the full 2D kernel spectrum even for a rank-1 mask */

/* AR-transform engine selection (dbx_plan_set_dst).  FFT = packed real DST-I in
 * shared memory (two lines per complex N-point DFT) whose DFT core is direct
 * (N with prime factors <= 31), Bluestein (power-of-two M >= 2N-1 up to 8192)
 * or Rader (N prime, N-1 compiled, e.g. 8191); DENSE = FP64 GEMM with the dense
 * T~/T matrices (reference dense_ar_forward / dense_ar_inverse block forms);
 * RADER = FFT with the Rader core forced where N is prime (tests).  AUTO picks
 * FFT whenever a core exists for the length. */
#define DBX_DST_AUTO 0
#define DBX_DST_DENSE 1
#define DBX_DST_FFT 2
#define DBX_DST_RADER 3

typedef struct dbx_plan dbx_plan;

/* Message of the last failing call on this thread ("" if none). */
const char* dbx_last_error(void);

/* Library version string, e.g. "dbx 0.1 sm_100a". */
const char* dbx_version(void);

/* Number of usable sm_100 devices (0 when none: every compute call then fails
 * with DBX_ECUDA — there is no CPU fallback). */
int dbx_device_count(void);

/*
 * Creates a plan for `batch` images of n1 x n2 pixels blurred by the
 * (2q1+1) x (2q2+1) mask `taps` (row-major, centre (q1,q2), host memory).
 * Replaces the construction of BlurOperator(Psf(taps), bc, n1, n2)
 * (reference blur.hpp:17-34) including Psf validation (psf.hpp:15-25: odd
 * dims, finite, >= 0, |sum-1| <= 1e-12) and check_support (boundary.hpp:66-81:
 * q <= n-2 on every axis with q > 0).  `device` selects the CUDA device.
 */
int dbx_plan_create(int n1, int n2, int batch, const double* taps, int q1, int q2, int bc,
                    int device, dbx_plan** out);
void dbx_plan_destroy(dbx_plan* plan);

/* cudaStream_t of the plan (as void*), for callers that time with CUDA events. */
void* dbx_plan_stream(dbx_plan* plan);

/* Blur engine override (DBX_CONV_*); default DBX_CONV_AUTO. */
int dbx_plan_set_conv(dbx_plan* plan, int conv);

/* AR-transform engine override (DBX_DST_*); default DBX_DST_AUTO. */
int dbx_plan_set_dst(dbx_plan* plan, int engine);

/* Fused row pipelines for the preconditioned FFT-form iteration (default 1):
 * 6 launches + finalize per iteration instead of 9 + finalize. */
int dbx_plan_set_fusion(dbx_plan* plan, int enable);

/*
 * Whether the FFT engine's column pass runs separable (*separable = 1): the
 * mask factors as w = a b^T within 1e-14 of its largest tap (axis-aligned
 * Gaussians, e.g. BASELINE C1, C3, C5), so FFT -> x H -> IFFT along each
 * column is the direct 2 q1 + 1 tap correlation of the AR-extended column
 * times one complex scale per column.  *resid = max |w - a b^T| / max |w|
 * (of the mask and its 180-degree rotation).  Diagnostic; no reference
 * equivalent (the reference correlates with the full mask, blur.hpp:39-68).
 */
int dbx_plan_separable(dbx_plan* plan, int* separable, double* resid);

/* Engines the plan will use: *conv in {DBX_CONV_DIRECT, DBX_CONV_FFT},
 * *dst in {DBX_DST_DENSE, DBX_DST_FFT}. */
int dbx_plan_engines(dbx_plan* plan, int* conv, int* dst);

/*
 * Reblurred CGLS (config 2's "CGLS-type" iteration; no
 * reference equivalent): minimises ||A x - g|| over Krylov
 * directions with the AR preconditioner D as the SPD weight
 * (use_precond = 1) or plain CGLS.  Arguments, stopping rules, histories,
 * best-iterate tracking and the divergence guard as dbx_landweber_run (the
 * residual is the recurrence's r_k = r_{k-1} - alpha q).
 */
int dbx_cgls_run(dbx_plan* plan, const double* g, const double* f_true, int max_iters, int stop_kind,
                 int fixed_iters, double resid_eps, int use_precond, double* restored, double* rre_hist,
                 double* res_hist, int* best_iter, int* iters_done, double* x_hist);

/*
 * Row-slab building blocks (one very large image split into row slabs across
 * ranks; orchestrated by paper_1211_0393_b200/slab.py with NCCL
 * halo exchange and all-to-all transposes).  The plan is created for one slab:
 * n1 = slab rows, n2 = full width, batch = 1.  Device pointers only.
 *
 * dbx_slab_blur: y = A x (adjoint = 0) or A' x on the slab's rows, from the
 *   caller-extended slab x_ext of (n1 + 2 q1) x n2 rows (q1 halo rows from the
 *   neighbours, or the global AR extension rows at the image's top/bottom);
 *   the horizontal AR extension is applied here.  g != NULL: y = g - A x and
 *   *norm2 = ||y||^2 (fixed-order sum).  Replaces apply / apply_reblur_adjoint
 *   (blur.hpp:75-90) restricted to a slab.
 * dbx_slab_rows: the AR transform `kind` along every row of the slab with an
 *   epilogue: DBX_SLAB_STORE (y = T x), DBX_SLAB_HADAMARD (y = aux o T x),
 *   DBX_SLAB_AXPY (y = aux + tau T x, norms2 = {||y||^2, ||y - f||^2}).
 * dbx_precond_block: block [r0, r0+nr) x [c0, c0+nc) of the n1g x n2g Tikhonov
 *   filter grid of the plan's symmetrised mask (transpose = 1: stored nc x nr).
 * dbx_transpose: out (cols x rows) = in (rows x cols)^T.
 * dbx_slab_extend: x_ext = [top; x; bot] ((n1 + 2 q1) x n2); top / bot = NULL
 *   at the image's first / last slab: the global AR extension rows
 *   (boundary.hpp:58-61) are synthesised from x instead.
 * dbx_slab_pack: blocks[p] = x[:, p cb : (p+1) cb] (cb = n2 / parts, each block
 *   n1 x cb contiguous) for the all-to-all transpose; unpack = 1 the inverse.
 */
#define DBX_SLAB_STORE 0
#define DBX_SLAB_HADAMARD 1
#define DBX_SLAB_AXPY 2
int dbx_slab_blur(dbx_plan* plan, const double* x_ext, double* y, int adjoint, const double* g, double* norm2);
int dbx_slab_rows(dbx_plan* plan, int kind, const double* x, double* y, int epi, const double* aux,
                  const double* f, double tau, double* norms2);
int dbx_precond_block(dbx_plan* plan, int n1g, int n2g, double alpha, int r0, int nr, int c0, int nc,
                      int transpose, double* out);
int dbx_transpose(dbx_plan* plan, const double* in, double* out, int rows, int cols);
int dbx_slab_extend(dbx_plan* plan, const double* x, const double* top, const double* bot, double* x_ext);
int dbx_slab_pack(dbx_plan* plan, const double* x, double* blocks, int parts, int unpack);

/*
 * C++ row-slab D-Landweber (the C5 config).  The loop that
 * paper_1211_0393_b200/slab.py orchestrated from Python, driven in C++ with
 * no host synchronisation inside the loop: per iteration the q-row halos go
 * through grouped ncclSend/ncclRecv with the slab neighbours (the first / last
 * slab synthesise the global AR rows on the device), the blur is the
 * separable direct pass on the halo-extended slab (FFT correlation for masks
 * that are not rank 1), the column half of D runs on column blocks obtained by
 * an all-to-all from grouped send/recv (two per iteration), and the three norms
 * are all-reduced on the device (ncclAllReduce of 3 doubles) and fed to a
 * device-side copy of the loop bookkeeping (solver.hpp:101-131).
 *
 * dbx_comm: an NCCL communicator, built here (dbx_comm_unique_id on one rank,
 *   broadcast the DBX_COMM_ID_BYTES bytes, dbx_comm_init on every rank) or
 *   wrapping the caller's ncclComm_t (dbx_comm_wrap; not owned).  libnccl.so.2
 *   is resolved at run time (the copy already loaded in the process first).
 * dbx_slab_create: slab plan of an n x n image in `parts` row slabs.  rank >= 0:
 *   this process holds slab `rank` (comm required when parts > 1); rank = -1:
 *   this process holds all `parts` slabs and the exchanges are device copies
 *   (in-process ranks, single-GPU parity tests).  alpha: the Tikhonov filter of
 *   the symmetrised mask (each process builds its own d^T column blocks).
 * dbx_slab_run: g, f (nullable), x_out are DEVICE arrays of the rows held here
 *   (slab-major, local_slabs x (n/parts) x n); histories are host arrays of
 *   max_iters; best_iter / iters_done as dbx_landweber_run.  Status as
 *   dbx_landweber_run (DBX_EDIVERGED on the divergence guard).
 */
#define DBX_COMM_ID_BYTES 128
typedef struct dbx_comm dbx_comm;
typedef struct dbx_slab dbx_slab;
int dbx_comm_unique_id(unsigned char* id);
int dbx_comm_init(int nranks, const unsigned char* id, int rank, int device, dbx_comm** comm);
int dbx_comm_wrap(void* nccl_comm, int nranks, int rank, dbx_comm** comm);
void dbx_comm_destroy(dbx_comm* comm);
int dbx_slab_create(int n, int parts, int rank, const double* taps, int q1, int q2, double alpha, dbx_comm* comm,
                    int device, dbx_slab** slab);
int dbx_slab_run(dbx_slab* slab, const double* g, const double* f, double tau, int max_iters, int stop_kind,
                 double resid_eps, double* x_out, double* rre_hist, double* res_hist, int* best_iter,
                 int* iters_done);
int dbx_slab_info(dbx_slab* slab, int* rows, int* local_slabs, int* separable, int64_t* launches);
void* dbx_slab_stream(dbx_slab* slab);
/* Tests: copy x_k (the rows held here) to buf + (k-1) * local_rows * n after
 * iteration k <= count (device buffer); buf = NULL disables. */
int dbx_slab_set_iterates(dbx_slab* slab, double* buf, int count);
void dbx_slab_destroy(dbx_slab* slab);

/*
 * Pipeline used by the last dbx_landweber_run on this plan: *fused = 1 for the
 * fused row pipelines (6 launches + finalize per preconditioned iteration,
 * fused.cu), 2 for their separable form (rank-1 mask: direct row passes in
 * the row kernels and a real column pass), 0 for the separate passes.
 * Diagnostic; no reference equivalent.
 */
int dbx_plan_pipeline(dbx_plan* plan, int* fused);

/*
 * y = A x (adjoint = 0) or y = A' x (adjoint = 1), for every image of the
 * batch.  Replaces apply (blur.hpp:75-83) and apply_reblur_adjoint
 * (blur.hpp:87-90): AR extension computed on the fly, no padded image.
 */
int dbx_blur_apply(dbx_plan* plan, const double* x, double* y, int adjoint);

/*
 * Builds D = T diag(d) T~ with d = 1/(lambda^2 + alpha), lambda the AR
 * eigenvalue grid of the SYMMETRISED mask.  Replaces build_tikhonov with
 * PreconditionerSpec{AntiReflective, alpha} (preconditioner.hpp:62-85) =
 * symmetrize (psf.hpp:71-85) + eig_antireflective (spectral.hpp:120-133) +
 * tikhonov_filter (preconditioner.hpp:37-57).  Errors like the reference:
 * alpha < 0, or alpha == 0 with a zero eigenvalue -> DBX_EINVAL.
 */
int dbx_precond_build(dbx_plan* plan, double alpha);

/* Copies the filter grid d (n1 x n2) to `d_out` (FilteredOperator::sop.eigs). */
int dbx_precond_eigs(dbx_plan* plan, double* d_out);

/* Replaces the filter grid with a caller-supplied one (SpectralOperator with
 * explicit eigs, spectral.hpp:32-39) — used for identity / constant filters. */
int dbx_precond_set_eigs(dbx_plan* plan, const double* d);

/* y = D r = T (d o (T~ r)) for every image.  Replaces precondition_apply
 * (preconditioner.hpp:88-90) -> filter_apply AR branch (spectral.hpp:161-165). */
/*
 * Alpha sweep (experiment.hpp:182-265 runs one
 * d_landweber cell per alpha): one Tikhonov filter grid per image of the
 * batch, image b filtered with alphas[b] (host array of `batch` values), so
 * the cells of a sweep run as one batched dbx_landweber_run.  A later
 * dbx_precond_build / dbx_precond_set_eigs returns to one shared grid;
 * dbx_precond_eigs reports image 0's grid.
 */
int dbx_precond_build_sweep(dbx_plan* plan, const double* alphas);

int dbx_precond_apply(dbx_plan* plan, const double* r, double* y);

/* 2D separable transform (columns then rows, transforms.hpp:179-192) of
 * kind DBX_KIND_{SINEI,AR,ARINV}; replaces tensor_apply (transforms.hpp:198-226). */
int dbx_tensor_apply(dbx_plan* plan, int kind, const double* x, double* y);

/*
 * Runs (preconditioned) Landweber for every image of the batch:
 *   x_0 = 0, x_k = x_{k-1} + tau * [D] A'(g - A x_{k-1}),
 * with the reference's bookkeeping (solver.hpp:63-132): residual_history[k-1]
 * = ||g - A x_k||, rre_history[k-1] = ||x_k - f||/||f|| (when f_true != NULL),
 * best_iteration by strict '<' (first minimum, 1-based), divergence guard
 * ||x_k|| > 1e8 ||g|| (-> DBX_EDIVERGED; the first diverging image index is
 * reported by dbx_last_error), RelativeResidualBelow breaking after recording,
 * restored = best iterate under MinRre with tracking, else the last iterate.
 * Replaces landweber (use_precond = 0) and d_landweber (use_precond = 1,
 * after dbx_precond_build) (solver.hpp:139-148).
 *
 *   g, f_true        [batch][n1][n2]   (f_true nullable: no RRE tracking)
 *   restored         [batch][n1][n2]
 *   rre_hist         [batch][H] with H = total iterations (nullable)
 *   res_hist         [batch][H]        (nullable)
 *   best_iter, iters_done  [batch]     (nullable, host memory)
 *   x_hist           [batch][H][n1][n2] every iterate (nullable; parity tests)
 *
 * H = fixed_iters for DBX_STOP_FIXED, else max_iters.
 */
int dbx_landweber_run(dbx_plan* plan, const double* g, const double* f_true, double tau,
                      int max_iters, int stop_kind, int fixed_iters, double resid_eps,
                      int use_precond, double* restored, double* rre_hist, double* res_hist,
                      int* best_iter, int* iters_done, double* x_hist);

/*
 * dbx_landweber_run over a batch split into `nplans` chunks, one plan per
 * chunk (plans[c] restores images [sum of earlier batches, + plans[c]->batch)
 * of g / f_true / restored / the histories; same n1 x n2, mask and, for
 * use_precond, a built preconditioner on every plan).  HOST arrays only
 * (page-locked for overlap): the chunks' inputs are copied up on a copy stream
 * in chunk order, each chunk's solve starts as soon as its own inputs landed
 * and the chunk two places earlier finished (two chunks solve concurrently,
 * one host thread per plan; DBX_CHUNK_DEPTH overrides the two) and its
 * restored images are copied down on its own stream, so the host<->device
 * traffic hides behind the other chunks' solves.
 * Results equal dbx_landweber_run on the whole batch (images are
 * independent).  Divergence: every chunk still runs; the first diverging image
 * (global index) is reported with DBX_EDIVERGED.  No reference equivalent (the
 * reference restores one image per call on the host).
 */
int dbx_landweber_run_chunks(dbx_plan* const* plans, int nplans, const double* g, const double* f_true,
                             double tau, int max_iters, int stop_kind, int fixed_iters, double resid_eps,
                             int use_precond, double* restored, double* rre_hist, double* res_hist,
                             int* best_iter, int* iters_done);

/*
 * Per-kernel-class device time (ms) and launch counts of the most recent
 * dbx_landweber_run made with timing enabled (dbx_plan_set_timing(plan, 1)):
 * classes 0 = blur A' (+fused epilogue), 1 = blur A (+residual), 2 = AR
 * transform passes, 3 = finalize/reductions.  Returns the number of classes.
 */
int dbx_plan_set_timing(dbx_plan* plan, int enable);
int dbx_plan_kernel_times(dbx_plan* plan, double* ms, int* launches, int max_classes);

/* Per-kernel timing of the last timed run (dbx_plan_set_timing): entry idx's
 * "kernel#class" name, total ms and launch count; returns the entry count. */
int dbx_plan_kernel_profile(dbx_plan* plan, int idx, char* name, int name_cap, double* ms, int* launches);

/* Total kernels launched by this plan since creation (launch accounting). */
int64_t dbx_plan_launch_count(dbx_plan* plan);

/* ---- input generation (host side, shared by the GPU harness and the oracle
 * tests) ---- */

/* Seeded scene: `nshapes` random ellipses / rectangles with U[0,1] intensities
 * on 0 (+ amp * smooth sinusoid when amp != 0), rows x cols, row-major. */
int dbx_gen_scene(int rows, int cols, int nshapes, double sinus_amp, uint64_t seed, double* out);

/* Gaussian mask: sigma (row, col), rotated by theta_deg (counter-clockwise,
 * columns to the right, rows down), centre offset (o1 rows, o2 cols),
 * normalised to sum 1 (generalises gaussian_portion_psf, psf.hpp:126-138). */
int dbx_gen_psf_gaussian(int q1, int q2, double sigma1, double sigma2, double theta_deg,
                         double off1, double off2, double* taps);

/* Motion mask: line of `length` px at `angle_deg` plus a one-sided exponential
 * tail of decay length `tail` px, rasterised by bilinear splatting, sum 1. */
int dbx_gen_psf_motion(int q1, int q2, double length, double angle_deg, double tail,
                       double* taps);

/* Honest data generation (experiment.hpp:71-99): centred crop offsets, direct
 * correlation of the scene (canvas rows x cols) with the mask, crop to
 * n1 x n2, then add_noise (image.hpp:72-82: mt19937_64 + Box-Muller, rescaled
 * to ||eta|| = level ||g|| exactly).  Threads: host threads used (0 = all). */
int dbx_gen_honest(const double* scene, int rows, int cols, const double* taps, int q1, int q2,
                   int n1, int n2, double noise_level, uint64_t noise_seed, int threads,
                   double* f_true, double* g);

/* add_noise alone (image.hpp:72-82). */
int dbx_add_noise(const double* g, int n1, int n2, double level, uint64_t seed, double* out);

/* Scene shape parameters in generation order (the mt19937_64 draws of
 * dbx_gen_scene), DBX_SHAPE_PARAMS doubles per shape: ellipse flag, cy, cx,
 * a, b, cos(theta), sin(theta), intensity, clipped bounding box r0, r1, c0, c1. */
#define DBX_SHAPE_PARAMS 12
int dbx_gen_scene_shapes(int rows, int cols, int nshapes, uint64_t seed, double* params);

/* The first `count` outputs of std::mt19937_64(seed) (host; test reference). */
int dbx_mt19937_64_host(uint64_t seed, uint64_t count, uint64_t* out);

/* The same stream generated on the GPU (gen_dev.cu: one CTA twists the 312-word
 * state two half-blocks at a time); `out` is host or device memory. */
int dbx_mt19937_64_device(uint64_t seed, uint64_t count, uint64_t* out, int device);

/* GPU-side Honest synthesis (experiment.hpp:71-99 + image.hpp:72-82):
 * the scene of dbx_gen_scene painted on the device (per-tile shape lists,
 * last covering shape wins — identical in/out decisions to the host painter),
 * the direct correlation with the mask over the canvas, the centred FOV crop
 * into f_true, and add_noise with the mt19937_64 stream twisted on the device
 * and Box-Muller per sample pair.  f_true (nullable) and g may be host or
 * device pointers (n1 x n2).  f_true equals the host generator's bit for bit;
 * g agrees to rounding (device libm and reduction order, <= 1e-14 relative). */
int dbx_gen_honest_device(int rows, int cols, int nshapes, double sinus_amp, uint64_t scene_seed,
                          const double* taps, int q1, int q2, int n1, int n2, double noise_level,
                          uint64_t noise_seed, double* f_true, double* g, int device);

#ifdef __cplusplus
}
#endif

#endif /* DBX_H_ */
