// ctf_loss.cu — a6: fused CTF multiply, Parseval loss and gradient spectrum.
//
// Eq. 7: I_pred = F^-1(C . F(I_hat)), L_i = ||I_pred - I_i||^2.
// With R = C . F(I_hat) - F(I_obs) on the half spectrum (cuFFT R2C layout
// [D][D/2+1]):  L_i = (1/D^2) sum_half w_k |R_k|^2  (w = 1 for k_x in {0, D/2},
// else 2), and dL/dI_hat = C2R_unnormalised((2/D^2) C . R)  (C is real and
// even; DESIGN.md §3 O7/O8).  The CTF (reading L10) is evaluated per bin with
// the phase in fp64 (it reaches ~420 rad at D=256), reduced mod 2 pi, then fp32
// sincos on [-pi, pi]; Nyquist bins average
// their +-1/(2 px) aliases (reading L12) so C(k) = C(-k) exactly.
#include "gem_internal.cuh"

namespace gem {
namespace {

constexpr int kCtfThreads = 256;
constexpr double kPi = 3.14159265358979323846;

// Per-particle constants: chi(f) = K1s s^2 + K1d ast(f) - K2 s^4 + phi, with
// s^2 = fx^2 + fy^2, ast = (fx^2 - fy^2) cos 2θ + 2 fx fy sin 2θ,
// K1s = π λ (du + dv)/2, K1d = π λ (du - dv)/2, K2 = π Cs λ^3 / 2 — the CTFFIND
// form of reading L10 with Δf s^2 expanded (no division by s^2).
struct CtfP {
  double K1s, K1d, K2, c2, s2a, phi;
  float alpha_s, alpha_c, bq;   // sqrt(1 - α^2), α, B/4
};

__device__ __forceinline__ float ctf_raw(const CtfP &p, double fx, double fy) {
  const double fx2 = fx * fx, fy2 = fy * fy, s2 = fx2 + fy2;
  const double ast = fma(fx2 - fy2, p.c2, 2.0 * fx * fy * p.s2a);
  double chi = fma(s2, fma(-p.K2, s2, p.K1s), fma(p.K1d, ast, p.phi));
  const double n = rint(chi * 0.15915494309189535);   // 1 / (2 pi)
  chi = fma(-n, 6.283185307179586, chi);                // reduced to [-pi, pi]
  float sn, cs;
  __sincosf((float)chi, &sn, &cs);                       // |abs err| < 4e-7 on [-pi, pi]
  const float env = p.bq > 0.f ? __expf(-p.bq * (float)s2) : 1.f;
  return -env * (p.alpha_s * sn + p.alpha_c * cs);
}

// Per-particle CTF constants (fp64: wavelength, defocus, Cs, astigmatism), once per particle.
__global__ void k_ctf_params(int B, const float *__restrict__ ctf, CtfP *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const float *q = ctf + 8 * i;
  const double kV = q[3], V = kV * 1000.0;
  const double h = 6.62607015e-34, m0 = 9.1093837015e-31, e = 1.602176634e-19, cl = 299792458.0;
  const double lam = h / sqrt(2.0 * m0 * e * V * (1.0 + e * V / (2.0 * m0 * cl * cl))) * 1e10;
  const double du = q[0], dv = q[1];
  CtfP P;
  P.K1s = kPi * lam * 0.5 * (du + dv);
  P.K1d = kPi * lam * 0.5 * (du - dv);
  P.K2 = 0.5 * kPi * ((double)q[4] * 1e7) * lam * lam * lam;
  P.c2 = cos(2.0 * (double)q[2]);
  P.s2a = sin(2.0 * (double)q[2]);
  P.phi = q[6];
  const double al = q[5];
  P.alpha_s = (float)sqrt(1.0 - al * al);
  P.alpha_c = (float)al;
  P.bq = 0.25f * q[7];
  out[i] = P;
}

__global__ void __launch_bounds__(kCtfThreads) k_ctf_loss(CfgDev c, const CtfP *__restrict__ ctfp,
                                                          float2 *__restrict__ spec_hat,
                                                          const float2 *__restrict__ spec_obs,
                                                          float2 *__restrict__ spec_pred, double *__restrict__ part) {
  __shared__ double red[kCtfThreads / 32];
  const int i = blockIdx.y, tid = threadIdx.x;
  const CtfP P = ctfp[i];
  const int D = c.D, Hx = D / 2 + 1;
  const int H = D * Hx;
  const int idx = blockIdx.x * kCtfThreads + tid;
  double lsum = 0.0;
  if (idx < H) {
    const int ky = idx / Hx, kx = idx - ky * Hx;
    const double idpx = 1.0 / ((double)D * (double)c.px), nyq = 1.0 / (2.0 * (double)c.px);
    double fx[2], fy[2];
    int nx = 1, ny = 1;
    if (2 * kx == D) { fx[0] = nyq; fx[1] = -nyq; nx = 2; } else fx[0] = kx * idpx;
    if (2 * ky == D) { fy[0] = nyq; fy[1] = -nyq; ny = 2; }
    else fy[0] = (2 * ky < D ? ky : ky - D) * idpx;
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

// Deterministic reduction of the per-block partials: block i sums particle i's partials with a
// fixed tree; the last block to finish (ticket) sums the B particle losses in order.
__global__ void __launch_bounds__(128) k_loss_reduce(int B, int nblk, const double *__restrict__ part,
                                                     double *__restrict__ loss, DevStats *st, int *ticket) {
  __shared__ double red[4];
  __shared__ int last;
  const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double s = 0.0;
  for (int b = tid; b < nblk; b += 128) s += part[(size_t)i * nblk + b];
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (tid == 0) {
    loss[i] = ((red[0] + red[1]) + red[2]) + red[3];
    __threadfence();
    last = atomicAdd(ticket, 1) == B - 1;
  }
  __syncthreads();
  if (!last || w != 0) return;
  __threadfence();
  double t = 0.0;
  for (int k = lane; k < B; k += 32) t += ((volatile double *)loss)[k];
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
  if (lane == 0) {
    loss[B] = t;
    if (!isfinite(t)) st->nonfinite = 1;
    *ticket = 0;   // self-reset for the next launch on this stream
  }
}

}  // namespace

void launch_ctf_loss(const CfgDev &c, int B, const float *ctf, void *ctf_par, float2 *spec_hat, const float2 *spec_obs,
                     float2 *spec_pred, double *loss_part, int loss_blocks, cudaStream_t s, int &launches) {
  CtfP *P = reinterpret_cast<CtfP *>(ctf_par);
  k_ctf_params<<<(B + 127) / 128, 128, 0, s>>>(B, ctf, P);
  dim3 grid(loss_blocks, B);
  k_ctf_loss<<<grid, kCtfThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, loss_part);
  launches += 2;
}

void launch_loss_reduce(int B, const double *loss_part, int loss_blocks, double *loss, DevStats *st, int *ticket,
                        cudaStream_t s, int &launches) {
  k_loss_reduce<<<B, 128, 0, s>>>(B, loss_blocks, loss_part, loss, st, ticket);
  ++launches;
}

size_t ctf_par_bytes() { return sizeof(CtfP); }

int ctf_loss_blocks(int D) { return (D * (D / 2 + 1) + kCtfThreads - 1) / kCtfThreads; }

}  // namespace gem
