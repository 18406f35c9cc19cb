/*
 * gem.h — C ABI of libgem.so, the B200-native (sm_100a) GEM training step.
 *
 * GEM (arXiv 2509.25075) reconstructs a cryo-EM density V from particle
 * images I_i with known rotations, translations and CTFs (Eqs. 2-3,
 * PAPER.md:155-165) by representing V as N anisotropic 3D Gaussians with 11
 * parameters each (Eqs. 4-5), projecting them in closed form
 * (Eq. 6, App. A.2), applying the CTF and an
 * l2 loss in Fourier space (Eq. 7), thresholding to the
 * Gaussians that contribute to each ray (Eq. 8) and scattering
 * gradients only to those Gaussians.  After training the
 * density is queried on a grid (Eq. 5).
 *
 * The five calls of the method's statement are gem_init, gem_forward,
 * gem_backward, gem_step and gem_render_volume.  Conventions fixed here (the
 * paper is silent; DESIGN.md §3 lists each reading):
 *   - parallel beam along camera z, J = I; full-line integral;
 *   - exact marginal amplitude amp = rho sqrt(2 pi) sqrt(|Sigma|/|Sigma_hat|)
 *     (reading L1);
 *   - pixel (u,v) is a point sample at x = (u - D/2) px, y = (v - D/2) px;
 *     images are row-major [v][u] (x fastest);
 *   - world->camera W = P_i^T for the particle rotation P_i; the shift t_i
 *     (Angstrom) is added to the in-plane camera coordinates;
 *   - cull: the integer k-sigma AABB of each projected Gaussian (default k=3,
 *     tau=0), tile lists in ascending Gaussian id (reading L5/L6/L9);
 *   - CTF: CTFFIND form, Nyquist alias-averaged so that C(k) = C(-k) (L10, L12);
 *   - loss L = sum over particles and pixels of (I_pred - I_obs)^2 (L14);
 *   - quaternion gradients are tangent to the unit sphere (L16);
 *   - optimiser: Adam (PyTorch form) + quaternion renormalisation (L15).
 *
 * Memory: the caller owns every buffer.  All pointers are DEVICE pointers
 * unless stated otherwise, and every float4-typed array (gem_soa members) must
 * be 16-byte aligned.  libgem performs no device allocation after gem_init
 * other than cuFFT plan objects for new batch sizes (their work area comes
 * from the caller's workspace).  A context serves one thread; every call is
 * asynchronous on the given stream unless documented as synchronous.  Inside a
 * call libgem also uses internal streams (a side stream for the observations'
 * transform, the CTF constants, the loss reduction and the clearing of the
 * projections; a copy stream for GEM_MEM_HOST inputs), forked from and joined
 * back into the caller's stream: when the caller's stream has passed a call,
 * all of that call's work is done.
 *
 * Errors: arguments are validated synchronously before any launch (no
 * exceptions cross the ABI).  Device-side conditions (list overflow, non-finite
 * loss or gradient) set flags that the next gem_stats call reports.
 */
#ifndef GEM_H
#define GEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GEM_API __attribute__((visibility("default")))
#else
#define GEM_API
#endif

typedef struct gem_ctx gem_ctx;
typedef void *gem_stream_t; /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  GEM_OK = 0,
  GEM_E_INVALID = 1,   /* null pointer, bad config value                          */
  GEM_E_SHAPE = 2,     /* D odd or < 2, B > max_batch, sizes inconsistent          */
  GEM_E_ALIGN = 3,     /* a gem_soa array or the workspace is not 16/256-B aligned  */
  GEM_E_CUDA = 4,      /* a CUDA launch / copy failed                               */
  GEM_E_CUFFT = 5,     /* a cuFFT call failed                                       */
  GEM_E_CAPACITY = 6,  /* list entries exceeded list_capacity (outputs invalid)    */
  GEM_E_STATE = 7,     /* gem_backward without a live gem_forward                   */
  GEM_E_NONFINITE = 8  /* non-finite loss or gradient was produced                  */
} gem_status;

/* Host struct, copied at gem_init. */
typedef struct {
  int32_t D;              /* image edge in pixels, even, >= 2; the tile grid
                             must fit the binning's shared-memory histograms: D <= 856
                             with 8x8 tiles, D <= 1712 with 16x16 (else GEM_E_INVALID)    */
  float pixel_size;       /* Angstrom per pixel, > 0                                      */
  int64_t n_gauss;        /* N Gaussians (the paper's M), >= 1               */
  int32_t max_batch;      /* max particles per gem_forward, >= 1                          */
  float cull_k;           /* Mahalanobis radius of the AABB cull (0 -> 3)                  */
  float tau;              /* |amp| <= tau => culled (Eq. 8); >= 0            */
  int32_t tile;           /* tile edge for the per-tile lists: 8 or 16 (0 -> 8)           */
  int64_t list_capacity;  /* max (Gaussian, tile) entries per batch (0 -> derived)          */
  float lr_mean, lr_log_scale, lr_quat, lr_density; /* Adam learning rates per class       */
  float beta1, beta2, eps;                          /* Adam (0 -> 0.9, 0.999, 1e-8)         */
  uint32_t flags;         /* GEM_FLAG_* below                                              */
  int32_t wave;           /* particles per L2-resident wave in fused mode (0 = auto)        */
} gem_config;

/* gem_config.flags.  GEM_FLAG_FUSED: gem_forward processes the batch in waves
 * of `wave` particles, running splat -> cull/bin -> projection -> FFT/CTF/loss
 * -> C2R -> backward scatter per wave so that splat records, tile lists and
 * images stay resident in L2; gem_backward then only finalizes the gradient
 * from the accumulators.  Results equal the unfused path's up to the
 * summation order over waves (every path is deterministic).  In fused mode
 * gem_export_lists can only export particles of the last wave. */
/* Ablation variants of the paper's Table 5:
 * GEM_FLAG_NO_ROTATION  "No Rotation, fix R_i = I": gem_step writes q = (1, 0, 0, 0) and the
 *                       quaternion gradient from gem_backward is exactly zero.
 * GEM_FLAG_ISOTROPIC    "Isotropic Scaling": after every gem_step the three log-scales of each
 *                       Gaussian are set to their mean (S:361 reading).
 * Paper-faithful selection order ("sort the selected Gaussians along the z-axis and
 * accumulate them starting from the lowest z value"):
 * GEM_FLAG_ZSORT        every (particle, tile) list is ordered by (z_ij, j) ascending, z_ij the
 *                       camera-frame depth of Gaussian j's centre, ((W20 mx + W21 my) + W22 mz)
 *                       in fp64 without FMA (W = P_i^T); gem_export_lists returns that order.
 *                       Costs one sort kernel and a list-sized scratch buffer in the workspace. */
/* Per-pixel selection (Eq. 8 "G_j > tau" at each pixel); the pixel
 * must lie in the AABB (as always) and in addition:
 * GEM_FLAG_ELLIPSE      inside the k-sigma ellipse, Q <= cull_k^2 (not only its bounding box);
 * GEM_FLAG_PIXEL_TAU    |amp_ij| exp(-Q/2) >= tau at the pixel.
 * Both apply to the forward and, with the same masks, to the backward.  DESIGN.md §3 L26.
 * GEM_FLAG_EXACT_TILES  (with ELLIPSE and/or PIXEL_TAU) a tile lists a Gaussian only if one of
 *                       its pixels is kept (exact ellipse-tile intersection);
 *                       without it the lists stay AABB-based (a superset, rendering zeros). */
enum { GEM_FLAG_FUSED = 1, GEM_FLAG_NO_ROTATION = 2, GEM_FLAG_ISOTROPIC = 4, GEM_FLAG_ZSORT = 8,
       GEM_FLAG_ELLIPSE = 16, GEM_FLAG_PIXEL_TAU = 32, GEM_FLAG_EXACT_TILES = 64 };

/* Gaussian parameter store (a0): three float4 arrays of length N.
 *   mean_rho [N] = (mu_x, mu_y, mu_z [Angstrom], rho)
 *   log_scale[N] = (s0, s1, s2, pad)   sigma_k = exp(s_k) Angstrom; pad stays 0
 *   quat     [N] = (w, x, y, z)        normalised inside the forward
 * The same layout holds gradients and Adam moments. */
typedef struct {
  float *mean_rho;
  float *log_scale;
  float *quat;
} gem_soa;

enum { GEM_MEM_DEVICE = 0, GEM_MEM_HOST = 1 };

/* One batch of B particles with known poses and CTFs (Eq. 3). */
typedef struct {
  int32_t B;              /* 1..max_batch                                                  */
  int32_t memory;         /* GEM_MEM_DEVICE, or GEM_MEM_HOST: the four arrays are pinned
                             host memory, copied asynchronously into the workspace (an
                             internal copy stream; staging double-buffered across calls, so
                             call k + 1's copy overlaps call k's kernels), and the loss of
                             gem_forward is written to a pinned host pointer.  The host
                             arrays must stay unchanged until `stream` has passed this call
                             (e.g. an event recorded after it), as for any async copy     */
  const float *rot;       /* [B][9] row-major particle rotation P_i (world->camera = P_i^T) */
  const float *shift;     /* [B][2] in-plane translation t_i, Angstrom                      */
  const float *ctf;       /* [B][8] du, dv (A), astig angle (rad), kV, Cs (mm), amplitude
                             contrast, phase shift (rad), B-factor (A^2)                    */
  const float *observed;  /* [B][D][D] observed particle images, row-major [v][u]          */
} gem_batch;

typedef struct {
  int64_t entries;        /* (Gaussian, tile) list entries of the last gem_forward           */
  int64_t capacity;       /* list_capacity in use                                          */
  int32_t degenerate;     /* Gaussians with |q| = 0 or non-finite prep in the last forward  */
  int32_t overflow;       /* 1 if entries > capacity in any forward since the previous
                             gem_stats call (sticky; cleared by this call)                   */
  int32_t nonfinite;      /* 1 if a non-finite loss or gradient was produced                 */
  int32_t batch;          /* B of the last gem_forward                                       */
  int64_t workspace_bytes;
  int64_t pairs;          /* useful (Gaussian, pixel) pairs of the last forward: sum over
                             visible (i,j) of the AABB area (the algorithmic work unit)      */
  int32_t wave;           /* particles per wave in use                                      */
  int32_t fused;          /* 1 if GEM_FLAG_FUSED                                            */
} gem_stats_t;

/* Per-kernel device time recorded with CUDA events on the launching stream
 * while profiling is enabled (names: prep, splat_count, scan, fill,
 * render_fwd, fft_r2c, ctf_loss, fft_c2r, render_bwd, finalize, adam, volume). */
typedef struct {
  char name[24];
  int32_t launches;
  double total_ms;
} gem_kernel_time_t;

/* Bytes of device workspace gem_init needs for cfg.  Host function; creates and
 * destroys a cuFFT plan to size its work area (needs a CUDA device).
 * Returns 0 for an invalid cfg. */
GEM_API size_t gem_workspace_bytes(const gem_config *cfg);

/* Validates cfg, carves `workspace` (device, >= gem_workspace_bytes(cfg) bytes,
 * 256-B aligned, owned by the caller and borrowed until gem_destroy) and
 * creates the batched cuFFT plans for (D, max_batch).  *out receives the
 * context.  Synchronous. */
GEM_API gem_status gem_init(const gem_config *cfg, void *workspace, size_t bytes, gem_stream_t stream,
                    gem_ctx **out);

/* Releases the context and its cuFFT plans (not the workspace).  Synchronous. */
GEM_API gem_status gem_destroy(gem_ctx *ctx);

/* Forward of one step (Eqs. 6-8): Gaussian prep, per-(i,j)
 * splat + AABB cull, per-tile lists, projection I_hat, cuFFT R2C of I_hat and
 * I_obs, fused CTF / Parseval loss / gradient spectrum, cuFFT C2R -> dL/dI_hat.
 *   loss     [B+1] doubles: per-particle loss then the batch total (device,
 *            or pinned host when batch->memory == GEM_MEM_HOST).
 *   proj_out [B][D][D] nullable: the projection I_hat (Eq. 6/8).
 *   pred_out [B][D][D] nullable: I_pred = F^-1(C . F(I_hat)) (Eq. 7).
 * Leaves lists, splat records and dL/dI_hat in the workspace for the next
 * gem_backward with the same params. */
GEM_API gem_status gem_forward(gem_ctx *ctx, const gem_soa *params, const gem_batch *batch, double *loss,
                       float *proj_out, float *pred_out, gem_stream_t stream);

/* Backward of the last gem_forward: scatters dL/dI_hat only to the Gaussians
 * in each tile list, transforms per-entry partials
 * to world-frame accumulators and finalizes the 11 parameter gradients.
 * `grad` (same layout as params) is OVERWRITTEN with dL/dparams summed over
 * the batch's particles and pixels; grad->log_scale pad lanes are 0.
 * GEM_E_STATE without a live forward. */
GEM_API gem_status gem_backward(gem_ctx *ctx, const gem_soa *params, gem_soa *grad, gem_stream_t stream);

/* Fused Adam step t (1-based) on params with moments m, v (all gem_soa,
 * updated in place), per-class learning rates from the config, then
 * q <- q/|q|.  Pad lanes are never touched. */
GEM_API gem_status gem_step(gem_ctx *ctx, gem_soa *params, const gem_soa *grad, gem_soa *m, gem_soa *v, int64_t t,
                    gem_stream_t stream);

/* Density query (Eq. 5): vol[(c*Dv + b)*Dv + a] = sum_j
 * 1[voxel in k-sigma box of j] rho_j exp(-1/2 d^T Sigma_j^-1 d) at voxel centre
 * ((a-Dv/2) vs, (b-Dv/2) vs, (c-Dv/2) vs).  vol_out is a device array of Dv^3
 * floats.  Uses its own scratch carved from `scratch` (device, nullable: then
 * gem_volume_scratch_bytes(ctx, Dv) bytes must fit in the step workspace). */
GEM_API gem_status gem_render_volume(gem_ctx *ctx, const gem_soa *params, int32_t Dv, float voxel_size, float *vol_out,
                             void *scratch, size_t scratch_bytes, gem_stream_t stream);
GEM_API size_t gem_volume_scratch_bytes(const gem_ctx *ctx, int32_t Dv, float voxel_size);

/* Diagnostics (synchronous).  Copies particle `particle`'s lists of the last
 * forward: tile_off [NT+1] (NT = ceil(D/tile)^2, offsets relative to the
 * particle's first entry), ids [<= ids_cap] ascending within each tile, and
 * aabb [N][4] = (u_lo, u_hi, v_lo, v_hi) clipped to [0, D-1] (empty box
 * (1, 0, 1, 0) for culled Gaussians).  Host pointers; any may be NULL. */
GEM_API gem_status gem_export_lists(gem_ctx *ctx, int32_t particle, int32_t *tile_off, int32_t *ids, int64_t ids_cap,
                            int32_t *aabb);

/* Synchronises the context's last stream and reports counters; returns
 * GEM_E_CAPACITY / GEM_E_NONFINITE if those flags are set, else GEM_OK. */
GEM_API gem_status gem_stats(gem_ctx *ctx, gem_stats_t *out);

/* enable = 1: reset and start recording an event pair around every kernel
 * (and cuFFT exec) this context launches; enable = 0: stop recording. */
GEM_API gem_status gem_profile_enable(gem_ctx *ctx, int32_t enable);

/* Synchronises, then writes up to cap per-kernel totals of the recorded
 * launches; returns the number of distinct kernels (or -1 on error). */
GEM_API int32_t gem_profile_read(gem_ctx *ctx, gem_kernel_time_t *out, int32_t cap);

/* Number of libgem kernel launches the last forward / backward / step /
 * render_volume issued (cuFFT's own kernels are not counted). */
GEM_API int32_t gem_last_launch_count(const gem_ctx *ctx);

GEM_API const char *gem_status_string(gem_status s);

#ifdef __cplusplus
}
#endif
#endif /* GEM_H */
