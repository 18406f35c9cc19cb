// ctf_loss.cu — a6: fused CTF multiply, Parseval loss and gradient spectrum.
//
// Eq. 7: I_pred = F^-1(C . F(I_hat)), L_i = ||I_pred - I_i||^2.
// With R = C . F(I_hat) - F(I_obs) on the half spectrum (cuFFT R2C layout
// [D][D/2+1]):  L_i = (1/D^2) sum_half w_k |R_k|^2  (w = 1 for k_x in {0, D/2},
// else 2), and dL/dI_hat = C2R_unnormalised((2/D^2) C . R)  (C is real and
// even; DESIGN.md §3 O7/O8).  The CTF (reading L10) is evaluated per bin with
// the phase in fp64, reduced mod 2 pi, then fp32 sincos; Nyquist bins average
// their +-1/(2 px) aliases (reading L12) so C(k) = C(-k) exactly.
#include "gem_internal.cuh"

namespace gem {
namespace {

constexpr int kCtfThreads = 256;
constexpr double kPi = 3.14159265358979323846;

struct CtfP {
  double du, dv, c2, s2a, lam, cs_A, alpha_s, alpha_c, phi, bfac;
};

__device__ __forceinline__ float ctf_raw(const CtfP &p, double fx, double fy) {
  const double s2 = fx * fx + fy * fy;
  double df = 0.5 * (p.du + p.dv);
  if (s2 > 0.0) df += 0.5 * (p.du - p.dv) * ((fx * fx - fy * fy) * p.c2 + 2.0 * fx * fy * p.s2a) / s2;
  const double lam = p.lam;
  double chi = kPi * lam * df * s2 - 0.5 * kPi * p.cs_A * lam * lam * lam * s2 * s2 + p.phi;
  chi -= 2.0 * kPi * rint(chi / (2.0 * kPi));
  float sn, cs;
  sincosf((float)chi, &sn, &cs);
  const float env = expf((float)(-p.bfac * s2 * 0.25));
  return -env * ((float)p.alpha_s * sn + (float)p.alpha_c * cs);
}

__global__ void __launch_bounds__(kCtfThreads) k_ctf_loss(CfgDev c, const float *__restrict__ ctf,
                                                          float2 *__restrict__ spec_hat,
                                                          const float2 *__restrict__ spec_obs,
                                                          float2 *__restrict__ spec_pred, double *__restrict__ part) {
  __shared__ CtfP P;
  __shared__ double red[kCtfThreads / 32];
  const int i = blockIdx.y, tid = threadIdx.x;
  if (tid == 0) {
    const float *q = ctf + 8 * i;
    const double kV = q[3], V = kV * 1000.0;
    const double h = 6.62607015e-34, m0 = 9.1093837015e-31, e = 1.602176634e-19, cl = 299792458.0;
    P.du = q[0]; P.dv = q[1];
    P.c2 = cos(2.0 * (double)q[2]); P.s2a = sin(2.0 * (double)q[2]);
    P.lam = h / sqrt(2.0 * m0 * e * V * (1.0 + e * V / (2.0 * m0 * cl * cl))) * 1e10;
    P.cs_A = (double)q[4] * 1e7;
    const double al = q[5];
    P.alpha_s = sqrt(1.0 - al * al); P.alpha_c = al;
    P.phi = q[6]; P.bfac = q[7];
  }
  __syncthreads();
  const int D = c.D, Hx = D / 2 + 1;
  const int H = D * Hx;
  const int idx = blockIdx.x * kCtfThreads + tid;
  double lsum = 0.0;
  if (idx < H) {
    const int ky = idx / Hx, kx = idx - ky * Hx;
    const double dpx = (double)D * (double)c.px, nyq = 1.0 / (2.0 * (double)c.px);
    double fx[2], fy[2];
    int nx = 1, ny = 1;
    if (2 * kx == D) { fx[0] = nyq; fx[1] = -nyq; nx = 2; } else fx[0] = kx / dpx;
    if (2 * ky == D) { fy[0] = nyq; fy[1] = -nyq; ny = 2; }
    else fy[0] = (2 * ky < D ? ky : ky - D) / dpx;
    float C = 0.f;
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < ny; ++b) C += ctf_raw(P, fx[a], fy[b]);
    C *= 1.0f / (float)(nx * ny);
    const size_t o = (size_t)i * H + idx;
    const float2 F = spec_hat[o], Ob = spec_obs[o];
    const float Rr = C * F.x - Ob.x, Ri = C * F.y - Ob.y;
    const double wgt = (kx == 0 || 2 * kx == D) ? 1.0 : 2.0;
    lsum = wgt * ((double)Rr * Rr + (double)Ri * Ri);
    const float gsc = 2.0f / ((float)D * (float)D);
    if (spec_pred) {
      const float ps = 1.0f / ((float)D * (float)D);
      spec_pred[o] = make_float2(C * F.x * ps, C * F.y * ps);
    }
    spec_hat[o] = make_float2(gsc * C * Rr, gsc * C * Ri);
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, d);
  if ((tid & 31) == 0) red[tid >> 5] = lsum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kCtfThreads / 32; ++w) s += red[w];
    part[(size_t)i * gridDim.x + blockIdx.x] = s / ((double)D * (double)D);
  }
}

// Deterministic reduction of the per-block partials: loss[i], then loss[B] = total.
__global__ void k_loss_reduce(int B, int nblk, const double *__restrict__ part, double *__restrict__ loss, DevStats *st) {
  __shared__ double li[1024];
  double tot = 0.0;
  for (int i0 = 0; i0 < B; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    if (i < B) {
      double s = 0.0;
      for (int b = 0; b < nblk; ++b) s += part[(size_t)i * nblk + b];
      loss[i] = s;
      li[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int m = min((int)blockDim.x, B - i0);
      for (int k = 0; k < m; ++k) tot += li[k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    loss[B] = tot;
    if (!isfinite(tot)) st->nonfinite = 1;
  }
}

}  // namespace

void launch_ctf_loss(const CfgDev &c, int B, const float *ctf, float2 *spec_hat, const float2 *spec_obs,
                     float2 *spec_pred, double *loss_part, int loss_blocks, double *loss, DevStats *st, cudaStream_t s,
                     int &launches) {
  dim3 grid(loss_blocks, B);
  k_ctf_loss<<<grid, kCtfThreads, 0, s>>>(c, ctf, spec_hat, spec_obs, spec_pred, loss_part);
  k_loss_reduce<<<1, 1024, 0, s>>>(B, loss_blocks, loss_part, loss, st);
  launches += 2;
}

int ctf_loss_blocks(int D) { return (D * (D / 2 + 1) + kCtfThreads - 1) / kCtfThreads; }

}  // namespace gem
