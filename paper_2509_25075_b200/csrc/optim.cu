// optim.cu — a8 pose-independent finalize and a10 fused Adam.
//
// Finalize (DESIGN.md §3 O10): from the world accumulators (L_rho, G_mu,
// G_Sigma) of each Gaussian:  dmu = G_mu, drho = L_rho,
//   ds_k = 2 sigma_k^2 (R^T G_Sigma R)_kk + rho L_rho,
//   dL/dR = 2 G_Sigma R diag(sigma^2),  dq_hat_c = <dL/dR, dR/dq_hat_c>,
//   dq = (I - q_hat q_hat^T) dq_hat / |q|   (tangent to the sphere, L16).
// Adam (reading L15, PyTorch bias-corrected form) per class lr, then
// q <- q/|q|; the log_scale pad lane is never touched.
#include "gem_internal.cuh"

namespace gem {
namespace {

// Degenerate Gaussians (the fp64 prep's flag, k_prep: the predicate of oracle O1, reading L18)
// get an exactly-zero gradient row.
__device__ __forceinline__ void finalize_j(int j, int no_rot, float4 a0, float4 a1, float4 a2,
                                           const GaussPrep *__restrict__ prep, const float4 *__restrict__ mr, const float4 *__restrict__ ls,
                                           const float4 *__restrict__ q, float4 *__restrict__ g_mr,
                                           float4 *__restrict__ g_ls, float4 *__restrict__ g_q, DevStats *st) {
  const float4 qq = q[j], ss = ls[j];
  const float rho = mr[j].w;
  const float n2 = qq.x * qq.x + qq.y * qq.y + qq.z * qq.z + qq.w * qq.w;
  if (prep[j].ok == 0.0 || !(n2 > 0.f)) {
    g_mr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    g_ls[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    g_q[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float inv = rsqrtf(n2);   // 1 / |q| (MUFU: the gradient's parity is 1e-4)
  const float w = qq.x * inv, x = qq.y * inv, y = qq.z * inv, z = qq.w * inv;
  float R[3][3];
  R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
  R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
  R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
  const float G[3][3] = {{a1.x, a1.y, a1.z}, {a1.y, a1.w, a2.x}, {a1.z, a2.x, a2.y}};
  const float s2[3] = {expf(2.f * ss.x), expf(2.f * ss.y), expf(2.f * ss.z)};
  float GR[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int k = 0; k < 3; ++k) GR[m][k] = G[m][0] * R[0][k] + G[m][1] * R[1][k] + G[m][2] * R[2][k];
  float ds[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float rgr = R[0][k] * GR[0][k] + R[1][k] * GR[1][k] + R[2][k] * GR[2][k];
    ds[k] = 2.f * s2[k] * rgr + rho * a0.x;
  }
  float dR[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int k = 0; k < 3; ++k) dR[m][k] = 2.f * GR[m][k] * s2[k];
  // <dR, dR/dq_hat_c> with dR/dq_hat from DESIGN.md §3 O10 (factor 2 folded in)
  float dw = 2.f * (-z * dR[0][1] + y * dR[0][2] + z * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]);
  float dx = 2.f * (y * dR[0][1] + z * dR[0][2] + y * dR[1][0] - 2.f * x * dR[1][1] - w * dR[1][2] + z * dR[2][0] +
                    w * dR[2][1] - 2.f * x * dR[2][2]);
  float dy = 2.f * (-2.f * y * dR[0][0] + x * dR[0][1] + w * dR[0][2] + x * dR[1][0] + z * dR[1][2] - w * dR[2][0] +
                    z * dR[2][1] - 2.f * y * dR[2][2]);
  float dz = 2.f * (-2.f * z * dR[0][0] - w * dR[0][1] + x * dR[0][2] + w * dR[1][0] - 2.f * z * dR[1][1] +
                    y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
  const float dot = dw * w + dx * x + dy * y + dz * z;
  const float4 gq = make_float4((dw - dot * w) * inv, (dx - dot * x) * inv, (dy - dot * y) * inv, (dz - dot * z) * inv);
  g_mr[j] = make_float4(a0.y, a0.z, a0.w, a0.x);
  g_ls[j] = make_float4(ds[0], ds[1], ds[2], 0.f);
  g_q[j] = no_rot ? make_float4(0.f, 0.f, 0.f, 0.f) : gq;   // GEM_FLAG_NO_ROTATION: R fixed to I
  const float chk = a0.x + a0.y + a0.z + a0.w + ds[0] + ds[1] + ds[2] + gq.x + gq.y + gq.z + gq.w;
  if (!isfinite(chk)) st->nonfinite = 1;
}

__global__ void __launch_bounds__(256) k_finalize(int N, int no_rot, const float4 *__restrict__ acc,
                                                  const GaussPrep *__restrict__ prep, const float4 *__restrict__ mr, const float4 *__restrict__ ls,
                                                  const float4 *__restrict__ q, float4 *__restrict__ g_mr,
                                                  float4 *__restrict__ g_ls, float4 *__restrict__ g_q, DevStats *st) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  finalize_j(j, no_rot, acc[3 * (size_t)j], acc[3 * (size_t)j + 1], acc[3 * (size_t)j + 2], prep, mr, ls, q, g_mr, g_ls,
             g_q, st);
}

// One batch (not fused): the backward's chunk sums [chunk][10][N] (render.cu k_render_bwd) are
// added in chunk order and finalized in the same thread (no accumulator round trip).
// One block per 32 Gaussians: warp k sums component k of the 32 Gaussians over the chunks
// (coalesced 128-byte rows, the chunks in order: the same fp32 sums as one thread per Gaussian),
// then the first warp finalizes.  (One thread per Gaussian looping over all 10 x nchunk slots left
// too few warps in flight: 196 blocks at N = 50 000.)
constexpr int kRfG = 32;
__global__ void __launch_bounds__(10 * kRfG) k_reduce_finalize(int nchunk, int N, int no_rot,
                                                              const float *__restrict__ slots,
                                                              const GaussPrep *__restrict__ prep,
                                                              const float4 *__restrict__ mr,
                                                              const float4 *__restrict__ ls,
                                                              const float4 *__restrict__ q, float4 *__restrict__ g_mr,
                                                              float4 *__restrict__ g_ls, float4 *__restrict__ g_q,
                                                              DevStats *st) {
  __shared__ float sv[10][kRfG];
  const int jj = threadIdx.x % kRfG, k = threadIdx.x / kRfG, j = blockIdx.x * kRfG + jj;
  float acc = 0.f;
  if (j < N) {
    const float *src = slots + (size_t)k * N + j;
    int ch = 0;
    for (; ch + 4 <= nchunk; ch += 4) {   // four loads in flight, added in chunk order
      const float a0 = __ldg(src + (size_t)ch * 10 * N), a1 = __ldg(src + (size_t)(ch + 1) * 10 * N);
      const float a2 = __ldg(src + (size_t)(ch + 2) * 10 * N), a3 = __ldg(src + (size_t)(ch + 3) * 10 * N);
      acc += a0; acc += a1; acc += a2; acc += a3;
    }
    for (; ch < nchunk; ++ch) acc += __ldg(src + (size_t)ch * 10 * N);
  }
  sv[k][jj] = acc;
  __syncthreads();
  if (k != 0 || j >= N) return;
  float v[10];
#pragma unroll
  for (int m = 0; m < 10; ++m) v[m] = sv[m][jj];
  const float rho = mr[j].w;
  finalize_j(j, no_rot, make_float4(rho != 0.f ? __fdividef(v[0], rho) : 0.f, v[1], v[2], v[3]),
             make_float4(v[4], v[5], v[6], v[7]), make_float4(v[8], v[9], 0.f, 0.f), prep, mr, ls, q, g_mr, g_ls, g_q,
             st);
}

// The same with 128-bit loads (N % 4 == 0): one block per 128 Gaussians, warp k sums component k
// of four Gaussians per lane (float4 rows), eight chunks in flight; then 128 threads finalize.
constexpr int kRf4 = 128;
__global__ void __launch_bounds__(320) k_reduce_finalize4(int nchunk, int N, int no_rot, const float *__restrict__ slots,
                                                         const GaussPrep *__restrict__ prep,
                                                         const float4 *__restrict__ mr, const float4 *__restrict__ ls,
                                                         const float4 *__restrict__ q, float4 *__restrict__ g_mr,
                                                         float4 *__restrict__ g_ls, float4 *__restrict__ g_q,
                                                         DevStats *st) {
  __shared__ float sv[10][kRf4];
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5, j0 = blockIdx.x * kRf4 + 4 * lane;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j0 < N) {   // (N % 4 == 0: the four Gaussians are all in range)
    const float4 *src = reinterpret_cast<const float4 *>(slots + (size_t)k * N + j0);
    const size_t cs = (size_t)10 * N / 4;   // one chunk, in float4
    int ch = 0;
    for (; ch + 8 <= nchunk; ch += 8) {   // eight loads in flight, added in chunk order
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldg(src + (size_t)(ch + u) * cs);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += a[u].x; acc.y += a[u].y; acc.z += a[u].z; acc.w += a[u].w;
      }
    }
    for (; ch < nchunk; ++ch) {
      const float4 a = __ldg(src + (size_t)ch * cs);
      acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
    }
  }
  *reinterpret_cast<float4 *>(&sv[k][4 * lane]) = acc;
  __syncthreads();
  const int jj = threadIdx.x, j = blockIdx.x * kRf4 + jj;
  if (jj >= kRf4 || j >= N) return;
  float v[10];
#pragma unroll
  for (int m = 0; m < 10; ++m) v[m] = sv[m][jj];
  const float rho = mr[j].w;
  finalize_j(j, no_rot, make_float4(rho != 0.f ? __fdividef(v[0], rho) : 0.f, v[1], v[2], v[3]),
             make_float4(v[4], v[5], v[6], v[7]), make_float4(v[8], v[9], 0.f, 0.f), prep, mr, ls, q, g_mr, g_ls, g_q,
             st);
}

// MUFU square root and reciprocal (a few ulp in the step lr m^ / (sqrt(v^) + eps): far below the
// 1e-6 parity with the fp64 optimizer, and no IEEE slow paths); ibc = 1 / (1 - beta^t) from the host
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float adam1(float p, float g, float &m, float &v, float lr, float b1, float b2, float eps,
                                       float ibc1, float ibc2) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  const float mh = m * ibc1, vh = v * ibc2;
  return p - lr * __fdividef(mh, sqrt_approx(vh) + eps);
}

struct AdamArgs {
  float4 *p[3];
  const float4 *g[3];
  float4 *m[3], *v[3];
  float lr_mean, lr_ls, lr_q, lr_rho, b1, b2, eps, bc1, bc2;   // bc1, bc2: 1 / (1 - beta^t)
  int flags;   // GEM_FLAG_NO_ROTATION / GEM_FLAG_ISOTROPIC
};

__global__ void __launch_bounds__(256) k_adam(int N, AdamArgs A) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int arr = blockIdx.y;
  if (j >= N) return;
  float4 p = A.p[arr][j], g = A.g[arr][j], m = A.m[arr][j], v = A.v[arr][j];
  if (arr == 0) {
    p.x = adam1(p.x, g.x, m.x, v.x, A.lr_mean, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.y = adam1(p.y, g.y, m.y, v.y, A.lr_mean, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.z = adam1(p.z, g.z, m.z, v.z, A.lr_mean, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.w = adam1(p.w, g.w, m.w, v.w, A.lr_rho, A.b1, A.b2, A.eps, A.bc1, A.bc2);
  } else if (arr == 1) {
    p.x = adam1(p.x, g.x, m.x, v.x, A.lr_ls, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.y = adam1(p.y, g.y, m.y, v.y, A.lr_ls, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.z = adam1(p.z, g.z, m.z, v.z, A.lr_ls, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    if (A.flags & GEM_FLAG_ISOTROPIC) {   // tie the three log-scales to their mean (Table 5)
      const float mean = (p.x + p.y + p.z) * (1.f / 3.f);
      p.x = p.y = p.z = mean;
    }
  } else if (A.flags & GEM_FLAG_NO_ROTATION) {   // R fixed to the identity (Table 5)
    p = make_float4(1.f, 0.f, 0.f, 0.f);
    m = v = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    p.x = adam1(p.x, g.x, m.x, v.x, A.lr_q, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.y = adam1(p.y, g.y, m.y, v.y, A.lr_q, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.z = adam1(p.z, g.z, m.z, v.z, A.lr_q, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    p.w = adam1(p.w, g.w, m.w, v.w, A.lr_q, A.b1, A.b2, A.eps, A.bc1, A.bc2);
    const float n2 = p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w;
    if (n2 > 0.f) {   // q / |q| (|q| = 1 to ~1e-7 after)
      const float r = rsqrtf(n2);
      p.x *= r; p.y *= r; p.z *= r; p.w *= r;
    }
  }
  A.p[arr][j] = p;
  A.m[arr][j] = m;
  A.v[arr][j] = v;
}

}  // namespace

void launch_reduce_finalize(const CfgDev &c, int B, const float *slots, const GaussPrep *prep, const float4 *mean_rho,
                            const float4 *log_scale, const float4 *quat, float4 *g_mr, float4 *g_ls, float4 *g_q, DevStats *st, cudaStream_t s,
                            int &launches) {
  const int no_rot = c.flags & GEM_FLAG_NO_ROTATION ? 1 : 0;
  if (c.N % 4 == 0)
    k_reduce_finalize4<<<(c.N + kRf4 - 1) / kRf4, 320, 0, s>>>(bwd_chunks(B), c.N, no_rot, slots, prep, mean_rho,
                                                               log_scale, quat, g_mr, g_ls, g_q, st);
  else
    k_reduce_finalize<<<(c.N + kRfG - 1) / kRfG, 10 * kRfG, 0, s>>>(bwd_chunks(B), c.N, no_rot, slots, prep,
                                                                    mean_rho, log_scale, quat, g_mr, g_ls, g_q, st);
  ++launches;
}

void launch_finalize(const CfgDev &c, const float4 *acc, const GaussPrep *prep, const float4 *mean_rho, const float4 *log_scale,
                     const float4 *quat, float4 *g_mr, float4 *g_ls, float4 *g_q, DevStats *st, cudaStream_t s,
                     int &launches) {
  k_finalize<<<(c.N + 255) / 256, 256, 0, s>>>(c.N, c.flags & GEM_FLAG_NO_ROTATION ? 1 : 0, acc, prep, mean_rho, log_scale, quat, g_mr, g_ls, g_q, st);
  ++launches;
}

void launch_adam(int N, float4 *p_mr, float4 *p_ls, float4 *p_q, const float4 *g_mr, const float4 *g_ls,
                 const float4 *g_q, float4 *m_mr, float4 *m_ls, float4 *m_q, float4 *v_mr, float4 *v_ls, float4 *v_q,
                 float lr_mean, float lr_ls, float lr_q, float lr_rho, float b1, float b2, float eps, float bc1,
                 float bc2, int flags, cudaStream_t s, int &launches) {
  AdamArgs A;
  A.flags = flags;
  A.p[0] = p_mr; A.p[1] = p_ls; A.p[2] = p_q;
  A.g[0] = g_mr; A.g[1] = g_ls; A.g[2] = g_q;
  A.m[0] = m_mr; A.m[1] = m_ls; A.m[2] = m_q;
  A.v[0] = v_mr; A.v[1] = v_ls; A.v[2] = v_q;
  A.lr_mean = lr_mean; A.lr_ls = lr_ls; A.lr_q = lr_q; A.lr_rho = lr_rho;
  A.b1 = b1; A.b2 = b2; A.eps = eps; A.bc1 = 1.f / bc1; A.bc2 = 1.f / bc2;   // (reciprocals)
  dim3 grid((N + 255) / 256, 3);
  k_adam<<<grid, 256, 0, s>>>(N, A);
  ++launches;
}

}  // namespace gem
