// gem_internal.cuh — shared device types, workspace layout and launch helpers
// for libgem.so (sm_100a).  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include "../../include/gem.h"

namespace gem {

#ifndef GEM_KCHUNK
#define GEM_KCHUNK 4096
#endif
constexpr int kChunk = GEM_KCHUNK;    // Gaussians per binning chunk (a3)
#ifndef GEM_FILLW
#define GEM_FILLW 4
#endif
constexpr int kFillWarps = GEM_FILLW; // k_fill warps per chunk (sub-chunks with their own tile counts)
constexpr double kSqrt2Pi = 2.5066282746310002;
constexpr float kLog2e = 1.4426950408889634f;

// a1 output: fp64 covariance (6 unique) + |Sigma| + |Sigma|^1/2 + ok flag (80 B, L2-resident).
struct __align__(16) GaussPrep {
  double sig[6];   // (00, 01, 02, 11, 12, 22)  Angstrom^2
  double detS;     // |Sigma|
  double sdetS;    // |Sigma|^{1/2}
  double ok;       // 1.0 valid, 0.0 degenerate
  double pad;
};

// a1 output, fp32 rotated frame for the splat fast path (48 B): column k of R(q_hat) and
// s_k = sigma_k^2; c[0].w < 0 marks a degenerate Gaussian.
struct __align__(16) GaussPrep32 {
  float4 c[3];
};

// a2 output per (particle, Gaussian): splat in pixel units (32 B, two float4).
//   f0 = (mxr, myr, a, b)   mxr = m_x/px + D/2 - u_lo (centre relative to the box corner)
//   f1 = (c, amp, ub, vb)   ub = u_lo | u_hi << 16, vb likewise (empty box: lo > hi)
struct __align__(16) SplatRec {
  float4 f0;
  float4 f1;
};

struct Layout {  // byte offsets into the caller's workspace
  size_t prep, rec, box, hist, subcnt, base, lst, ids, proj, spec_hat, spec_obs, spec_pred, dldi, slots, acc, loss_part, ctf_par,
      stats, ticket, stage_rot, stage_shift, stage_ctf, stage_obs, stage_loss, cufft_work, cufft_work2, zs_tmp, zs_key, zs_queue, total;
  int64_t n_hist;       // B_max * NT * C
  int64_t list_cap;
  size_t cufft_bytes;
  int loss_blocks;      // CTF/loss partial blocks per particle
};

struct DevStats {      // device-side counters (zeroed per forward)
  unsigned long long entries;
  unsigned long long pairs;
  int overflow;
  int degenerate;
  int nonfinite;
  int pad;
};

struct CfgDev {        // resolved config passed by value to kernels
  int D, T, tshift, nt, NT, N, C;   // T = 1 << tshift
  unsigned flags;                   // gem_config.flags
  float px, k, tau;
  int64_t cap;
  float inv_NT, inv_nt;             // 1 / NT, 1 / nt (fast exact division, see fdivmod)
};

// q = x / d, r = x % d for 0 <= x < 2^22 with a float reciprocal and one branch-free correction
// (x and d are exact in fp32 and inv = 1/d to 1 ulp, so the truncated estimate is off by at most 1)
__device__ __forceinline__ int fdivmod(int x, int d, float inv, int &r) {
  int q = __float2int_rz((float)x * inv);
  r = x - q * d;
  q += (r >= d) - (r < 0);
  r = x - q * d;
  return q;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// List offsets (a3): base[(i C + chunk) NT + t] = start of chunk's entries in list (i, t) (the
// fill's cursors), and lst[i NT + t] = start of list (i, t), lst[B NT] = all entries: list (i, t)
// spans ids[lst[it] .. lst[it + 1]), it = i NT + t (the render, z-sort and export read lst).

}  // namespace gem

struct gem_ctx {
  gem_config cfg;
  gem::CfgDev dc;
  gem::Layout L;
  char *ws;
  size_t ws_bytes;
  cudaStream_t stream;
  // cuFFT plans keyed by batch size (small cache)
  int plan_B[8];
  cufftHandle plan_r2c[8], plan_c2r[8], plan_obs[8];   // plan_obs: R2C of the observed images (side stream)
  cufftHandle plan_il[8];   // C2C of the packed dL/dI row pairs (row path only, else 0)
  cudaStream_t side;   // internal stream: observed-image R2C overlapped with splat/bin/render
  cudaEvent_t ev_fork, ev_join, ev_ctf, ev_loss;   // side-stream fork / join points
  cudaStream_t copy = nullptr;   // host mode: the observed images' H2D, wave by wave
  cudaEvent_t *ev_obs = nullptr;   // one per wave: its images are on the device
  int n_ev_obs = 0;
  int obs_half = 0;   // the half of the double-buffered staging the next gem_forward uses
  cudaEvent_t ev_obs_free[2] = {nullptr, nullptr};   // the side stream's last reads of each half are done
  cudaEvent_t ev_sfree[2] = {nullptr, nullptr};      // the compute stream's last reads of each half are done
  cudaEvent_t ev_small = nullptr;                    // host mode: poses and CTFs are on the device
  cudaEvent_t ev_zero = nullptr;                     // the wave's projections are cleared (side stream)
  float *rot_cur = nullptr;                          // the last forward's staged rotations (gem_backward)
  int n_plans;
  int fwd_live;        // a forward's lists/records/dL/dI are valid
  int last_B;
  int W;               // particles per wave (max_batch when not fused)
  int fused;           // GEM_FLAG_FUSED
  int last_p0, last_nb;  // the last wave of the last forward
  int launches;
  // profiling (gem_profile_enable): event pairs around launches
  int prof_on;
  int prof_n, prof_cap;
  int *prof_kind;
  cudaEvent_t *prof_ev;  // 2 per record
};

namespace gem {
enum ProfKind { P_PREP, P_SPLAT, P_SCAN, P_FILL, P_RENDER_FWD, P_FFT_R2C, P_CTF_LOSS, P_FFT_C2R, P_FFT_OBS, P_RENDER_BWD,
                P_BWD_REDUCE, P_FINALIZE, P_ADAM, P_VOLUME, P_ZSORT, P_COUNT };
}

// ------------------------------------------- per-pixel selection tile test (GEM_FLAG_ELLIPSE/_PIXEL_TAU)
namespace gem {
// Q threshold of the per-pixel selection: a pixel is kept iff Q <= t,
// t = min(ELLIPSE ? k^2 : inf, PIXEL_TAU ? 2 ln(|amp| / tau) : inf)   (reading L26)
__device__ __forceinline__ float keep_q(const CfgDev &c, float amp) {
  float t = (c.flags & GEM_FLAG_ELLIPSE) ? c.k * c.k : 3.0e38f;
  if ((c.flags & GEM_FLAG_PIXEL_TAU) && c.tau > 0.f) t = fminf(t, 2.f * logf(fabsf(amp) / c.tau));
  return t;
}
// Exact ellipse-tile intersection for the lists: does the pixel block
// [c0, c1] x [r0, r1] (absolute indices, inside the AABB) hold a pixel with Q <= t?  Row by row
// the kept columns are u in [ucen + (-b dy - sqrt(disc)) / a, ucen + (-b dy + sqrt(disc)) / a],
// disc = a t - det dy^2.  Round-to-nearest intrinsics only (no contraction): the splat kernel
// (histogram) and the fill (ids) call this with the same inputs and must decide identically.
__device__ __forceinline__ bool tile_kept(float ucen, float vcen, float a, float b, float cc, float t, int c0, int c1,
                                          int r0, int r1) {
  const float det = __fsub_rn(__fmul_rn(a, cc), __fmul_rn(b, b));
  const float at = __fmul_rn(a, t), ia = __frcp_rn(a);
  for (int v = r0; v <= r1; ++v) {
    const float dy = __fsub_rn((float)v, vcen);
    const float disc = __fsub_rn(at, __fmul_rn(det, __fmul_rn(dy, dy)));
    if (!(disc >= 0.f)) continue;
    const float sq = __fsqrt_rn(disc), mb = __fmul_rn(-b, dy);
    const float lo = __fadd_rn(ucen, __fmul_rn(__fsub_rn(mb, sq), ia));
    const float hi = __fadd_rn(ucen, __fmul_rn(__fadd_rn(mb, sq), ia));
    if (fmaxf(ceilf(lo), (float)c0) <= fminf(floorf(hi), (float)c1)) return true;
  }
  return false;
}
}  // namespace gem

// ---------------------------------------------------------------- z-sort keys (GEM_FLAG_ZSORT)
namespace gem {
// camera-frame depth of Gaussian j under pose i, ((W20 mx + W21 my) + W22 mz), W = P^T, in fp64
// without contraction (w0, w1, w2 = P[2], P[5], P[8]); the z-sort key (L24)
__device__ __forceinline__ double zdepth64(float4 m, double w0, double w1, double w2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(w0, (double)m.x), __dmul_rn(w1, (double)m.y)), __dmul_rn(w2, (double)m.z));
}
// order-preserving map of an fp32 value to uint32
__device__ __forceinline__ unsigned ord32(float z) {
  const unsigned b = __float_as_uint(z);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
}  // namespace gem


// ---------------------------------------------------------------- TMA bulk copies + mbarriers
namespace gem {
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// one bulk (non-tensor) TMA copy global -> shared, completing on the barrier; bytes % 16 == 0,
// both addresses 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
}  // namespace gem

// ---------------------------------------------------------------- kernels
namespace gem {
void launch_prep(const CfgDev &c, const float4 *mean_rho, const float4 *log_scale, const float4 *quat, GaussPrep *prep,
                 DevStats *st, cudaStream_t s, int &launches);
void launch_splat_count(const CfgDev &c, int B, const GaussPrep *prep, const float4 *mean_rho, const float *rot,
                        const float *shift, SplatRec *rec, uint2 *box, unsigned short *hist, unsigned short *subcnt,
                        int *ptot, DevStats *st, cudaStream_t s, int &launches);
void launch_scan_pp(const CfgDev &c, int B, const unsigned short *hist, int *base, int *lst, const int *ptot, DevStats *st,
                    int *tk, cudaStream_t s, int &launches);
void launch_scan(const int *in, int *out, int64_t n, int *blk, int64_t nblk, DevStats *st, int64_t cap, cudaStream_t s,
                 int &launches);
void launch_fill(const CfgDev &c, int B, const uint2 *box, const int *base, const unsigned short *subcnt, int *ids,
                 const float4 *mean_rho, const float *rot, uint2 *zpair, const SplatRec *rec, cudaStream_t s,
                 int &launches);
void launch_zsort(const CfgDev &c, int B, const int *base, const float4 *mean_rho, const float *rot, int *ids,
                  const uint2 *zpair, int *tmp, int *queue, cudaStream_t s, int &launches);
void launch_render_fwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids, float *proj,
                       int *ticket, cudaStream_t s, int &launches, bool cleared);   // cleared: proj already zero
void launch_ctf_params(const CfgDev &c, int B, const float *ctf, void *ctf_par, cudaStream_t s, int &launches);
void launch_ctf_loss(const CfgDev &c, int B, const void *ctf_par, float2 *spec_hat, const float2 *spec_obs,
                     float2 *spec_pred, float2 *zout, double *loss_part, int loss_blocks, cudaStream_t s,
                     int &launches);
size_t ctf_par_bytes();
bool spectral_rows(int D);   // row-column spectral path (1D row plans + column kernel)
void launch_loss_reduce(int B, const double *loss_part, int loss_blocks, double *loss, DevStats *st, int *ticket,
                        cudaStream_t s,
                        int &launches);
int ctf_loss_blocks(int D);
void launch_dldi_pack(const CfgDev &c, int B, const float *in, float *out, cudaStream_t s, int &launches);
int bwd_chunks(int B);   // particle chunks of the backward (slots per Gaussian)
void launch_render_bwd(const CfgDev &c, int B, const SplatRec *rec, const float *dldi, const float *rot, float *slots,
                       cudaStream_t s, int &launches);
void launch_bwd_reduce(const CfgDev &c, int B, const float *slots, const float4 *mean_rho, float4 *acc, cudaStream_t s,
                       int &launches);
void launch_reduce_finalize(const CfgDev &c, int B, const float *slots, const GaussPrep *prep, const float4 *mean_rho,
                            const float4 *log_scale, const float4 *quat, float4 *g_mr, float4 *g_ls, float4 *g_q, DevStats *st, cudaStream_t s,
                            int &launches);
void launch_finalize(const CfgDev &c, const float4 *acc, const GaussPrep *prep, const float4 *mean_rho, const float4 *log_scale,
                     const float4 *quat, float4 *g_mr, float4 *g_ls, float4 *g_q, DevStats *st, cudaStream_t s,
                     int &launches);
void launch_adam(int N, float4 *p_mr, float4 *p_ls, float4 *p_q, const float4 *g_mr, const float4 *g_ls,
                 const float4 *g_q, float4 *m_mr, float4 *m_ls, float4 *m_q, float4 *v_mr, float4 *v_ls, float4 *v_q,
                 float lr_mean, float lr_ls, float lr_q, float lr_rho, float b1, float b2, float eps, float bc1,
                 float bc2, int flags, cudaStream_t s, int &launches);
size_t volume_scratch_bytes(int N, int Dv);
cudaError_t launch_volume(int N, const float4 *mean_rho, const float4 *log_scale, const float4 *quat, int Dv,
                          float vs, float k, float *vol, char *scratch, size_t scratch_bytes, cudaStream_t s,
                          int &launches, DevStats **st_out);
}  // namespace gem
