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

// Per-particle constants.  With integer frequency indices (kx, ky) and idpx = 1/(D px):
//   s^2 = n2 idpx^2, n2 = kx^2 + ky^2 (exact integer), ast s^2-terms = ((kx^2 - ky^2) cos 2θ +
//   2 kx ky sin 2θ) idpx^2, so the CTFFIND phase of reading L10,
//   chi = K1s s^2 + K1d ast - K2 s^4 + phi,
// becomes chi = a n2 + b d2 + c m2 - e n2^2 + phi with d2 = kx^2 - ky^2, m2 = 2 kx ky (exact
// integers) and per-particle fp64 coefficients: 4 DFMA per bin.  The phase (up to ~420 rad at
// D = 256) is reduced mod 2 pi in fp64, then fp32 sincos on [-pi, pi].
struct CtfP {
  double a, b, c, e, phi;
  float alpha_s, alpha_c, bq;   // sqrt(1 - α^2), α, B idpx^2 / 4 (envelope exp(-bq n2))
};

__device__ __forceinline__ float ctf_raw(const CtfP &p, double n2, double d2, double m2) {
  double chi = fma(n2, fma(-p.e, n2, p.a), fma(p.b, d2, fma(p.c, m2, p.phi)));
  const double n = rint(chi * 0.15915494309189535);   // 1 / (2 pi)
  chi = fma(-n, 6.283185307179586, chi);                // reduced to [-pi, pi]
  float sn, cs;
  __sincosf((float)chi, &sn, &cs);                       // |abs err| < 4e-7 on [-pi, pi]
  const float env = p.bq > 0.f ? __expf(-p.bq * (float)n2) : 1.f;
  return -env * (p.alpha_s * sn + p.alpha_c * cs);
}

// Per-particle CTF constants (fp64: wavelength, defocus, Cs, astigmatism), once per particle.
__global__ void k_ctf_params(int B, double idpx, const float *__restrict__ ctf, CtfP *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const float *q = ctf + 8 * i;
  const double kV = q[3], V = kV * 1000.0;
  const double h = 6.62607015e-34, m0 = 9.1093837015e-31, e = 1.602176634e-19, cl = 299792458.0;
  const double lam = h / sqrt(2.0 * m0 * e * V * (1.0 + e * V / (2.0 * m0 * cl * cl))) * 1e10;
  const double du = q[0], dv = q[1];
  const double K1s = kPi * lam * 0.5 * (du + dv), K1d = kPi * lam * 0.5 * (du - dv);
  const double K2 = 0.5 * kPi * ((double)q[4] * 1e7) * lam * lam * lam;
  const double i2 = idpx * idpx;
  CtfP P;
  P.a = K1s * i2;
  P.b = K1d * cos(2.0 * (double)q[2]) * i2;
  P.c = K1d * sin(2.0 * (double)q[2]) * i2;
  P.e = K2 * i2 * i2;
  P.phi = q[6];
  const double al = q[5];
  P.alpha_s = (float)sqrt(1.0 - al * al);
  P.alpha_c = (float)al;
  P.bq = (float)(0.25 * (double)q[7] * i2);
  out[i] = P;
}

// One block per (particle, kCtfRows rows of ky); the block's Hx x kCtfRows bins are spread over
// its threads (row = floor((idx + 1/2) / Hx) in fp32, exact at these sizes).  The loss is
// summed in fp32 over a thread's few bins, then in fp64 (fixed tree) across the block.
constexpr int kCtfRows = 8;

__global__ void __launch_bounds__(kCtfThreads) k_ctf_loss(CfgDev c, const CtfP *__restrict__ ctfp,
                                                          float2 *__restrict__ spec_hat,
                                                          const float2 *__restrict__ spec_obs,
                                                          float2 *__restrict__ spec_pred, double *__restrict__ part) {
  __shared__ double red[kCtfThreads / 32];
  const int i = blockIdx.y, tid = threadIdx.x;
  const CtfP P = ctfp[i];
  const int D = c.D, Hx = D / 2 + 1, H = D * Hx;
  const float gsc = 2.0f / ((float)D * (float)D), ps = 1.0f / ((float)D * (float)D);
  float lsum = 0.f;
  const int ky0 = blockIdx.x * kCtfRows, nb = Hx * kCtfRows;
  const float invH = 1.f / (float)Hx;
  for (int idx = tid; idx < nb; idx += kCtfThreads) {
    const int r = (int)(((float)idx + 0.5f) * invH), kx = idx - r * Hx, ky = ky0 + r;
    if (ky >= D) break;
    const bool nx = 2 * kx == D, ny = 2 * ky == D;
    const int kys = 2 * ky < D ? ky : ky - D;
    // Nyquist bins average their +-1/(2 px) aliases (reading L12): sign flips of kx or ky
    float C = 0.f;
    const double kxd = kx, kyd = kys;
    for (int a = 0; a < (nx ? 2 : 1); ++a)
      for (int b2 = 0; b2 < (ny ? 2 : 1); ++b2) {
        const double fx = a ? -kxd : kxd, fy = b2 ? -kyd : kyd;
        C += ctf_raw(P, fx * fx + fy * fy, fx * fx - fy * fy, 2.0 * fx * fy);
      }
    if (nx || ny) C *= (nx && ny) ? 0.25f : 0.5f;
    const size_t o = (size_t)i * H + (size_t)ky * Hx + kx;
    const float2 F = spec_hat[o], Ob = spec_obs[o];
    const float Rr = C * F.x - Ob.x, Ri = C * F.y - Ob.y;
    const float wgt = (kx == 0 || nx) ? 1.f : 2.f;
    lsum = fmaf(wgt, fmaf(Rr, Rr, Ri * Ri), lsum);
    if (spec_pred) spec_pred[o] = make_float2(C * F.x * ps, C * F.y * ps);
    spec_hat[o] = make_float2(gsc * C * Rr, gsc * C * Ri);
  }
  double ls = lsum;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, d);
  if ((tid & 31) == 0) red[tid >> 5] = ls;
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

// ------------------------------------------------------------- row-column spectral path
// For D = R1 R2 in {32, 64, 128, 256} the 2D transforms are split (DESIGN.md §6 a6): cuFFT does
// only the row transforms (1D R2C of the projections and the observations, 1D C2R of the
// gradient), and one kernel does everything along the columns: for each half-spectrum column
// kx, the forward column FFTs of F(I_hat) and F(I_obs), the CTF / residual / Parseval loss /
// gradient spectrum per bin, and the inverse column FFT of the gradient spectrum, in place.
// Row then column = the 2D DFT (separable), so the loss and gradient are those of k_ctf_loss.
// A group of R2 threads transforms one column (length D, four-step: R1-point DFTs in registers,
// twiddles, a transpose through shared memory, R2-point DFTs); R1 values per thread.
// cos and sin of 2 pi j / 16 (the twiddles of the in-register DFTs are compile-time constants)
__device__ __forceinline__ float c16(int j) {
  constexpr float v[16] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f, 0.f,
                           -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f, -1.f,
                           -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f, 0.f,
                           0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  return v[j & 15];
}
__device__ __forceinline__ float s16(int j) { return c16(j + 12); }   // sin x = cos(x - pi/2)

template <int R>
__device__ __forceinline__ void dft_reg(float2 (&a)[R]) {
  // radix-2 decimation in frequency in registers, W_R^j = exp(-2 pi i j / R); natural-order output
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const float2 u = a[b + j], v = a[b + j + half];
        const int e = j * (16 / (2 * half));   // W_{2 half}^j = W_16^e
        const float wr = c16(e), wi = -s16(e);
        const float dx = u.x - v.x, dy = u.y - v.y;
        a[b + j] = make_float2(u.x + v.x, u.y + v.y);
        if (e == 0) a[b + j + half] = make_float2(dx, dy);
        else if (e == 4) a[b + j + half] = make_float2(dy, -dx);   // times -i
        else a[b + j + half] = make_float2(dx * wr - dy * wi, dx * wi + dy * wr);
      }
    }
  }
  float2 t[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int r = 0;
#pragma unroll
    for (int bit = 1, rb = R / 2; bit < R; bit <<= 1, rb >>= 1) r |= (k & bit) ? rb : 0;
    t[k] = a[r];
  }
#pragma unroll
  for (int k = 0; k < R; ++k) a[k] = t[k];
}

// forward (unnormalised) DFT of one column held as v[n1] = x[R2 n1 + t]; on return
// v[s R2 + k2] = X[(t S + s) + R1 k2], S = R1 / R2
template <int R1, int R2>
__device__ __forceinline__ void fft_col(float2 (&v)[R1], int t, float2 *sb, const float2 *__restrict__ tw) {
  constexpr int S = R1 / R2, P = R2 + 1;   // padded pitch: the transposed reads are conflict-free
  dft_reg<R1>(v);
  const float2 w1 = tw[t];   // W_D^(t k1) by recurrence (no bank-conflicting table lookups)
  float2 w = w1;
#pragma unroll
  for (int k1 = 1; k1 < R1; ++k1) {
    const float2 x = v[k1];
    v[k1] = make_float2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x);
    w = make_float2(w.x * w1.x - w.y * w1.y, w.x * w1.y + w.y * w1.x);
  }
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) sb[k1 * P + t] = v[k1];
  __syncwarp();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    float2 u[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) u[n2] = sb[(t * S + s) * P + n2];
    dft_reg<R2>(u);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) v[s * R2 + k2] = u[k2];
  }
  __syncwarp();
}

// inverse (unnormalised) DFT of one column held in fft_col's output order, v[s R2 + k2] =
// Y[(t S + s) + R1 k2]; on return v[n1] = y[R2 n1 + t] = sum_k Y[k] W_D^(-(R2 n1 + t) k) (natural
// order: no reordering pass).  With n = R2 n1 + n2 and k = k1 + R1 k2, W_D^(nk) = W_R1^(n1 k1)
// W_D^(n2 k1) W_R2^(n2 k2): R2-point DFTs over k2 in registers, twiddles, one transpose through
// shared memory, R1-point DFTs over k1 in registers -- the forward DFT of conj(Y), conjugated.
template <int R1, int R2>
__device__ __forceinline__ void fft_col_inv(float2 (&v)[R1], int t, float2 *sb, const float2 *__restrict__ tw) {
  constexpr int S = R1 / R2, P = R2 + 1;
  constexpr int D = R1 * R2;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    float2 u[R2];
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) u[k2] = make_float2(v[s * R2 + k2].x, -v[s * R2 + k2].y);
    dft_reg<R2>(u);   // u[n2] = sum_k2 conj(Y)[k1 + R1 k2] W_R2^(n2 k2), k1 = t S + s
    const int k1 = t * S + s;
    const float2 w1 = tw[k1 & (D - 1)];   // W_D^(k1), then W_D^(n2 k1) by recurrence
    float2 w = w1;
#pragma unroll
    for (int n2 = 1; n2 < R2; ++n2) {
      const float2 x = u[n2];
      u[n2] = make_float2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x);
      w = make_float2(w.x * w1.x - w.y * w1.y, w.x * w1.y + w.y * w1.x);
    }
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) sb[k1 * P + n2] = u[n2];
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) v[k1] = sb[k1 * P + t];
  __syncwarp();
  dft_reg<R1>(v);
#pragma unroll
  for (int n1 = 0; n1 < R1; ++n1) v[n1].y = -v[n1].y;
}

constexpr int kColThreads = 128;

template <int R1, int R2>
__global__ void __launch_bounds__(kColThreads) k_ctf_colspec(CfgDev c, const CtfP *__restrict__ ctfp,
                                                             const float2 *__restrict__ spec,
                                                             const float2 *__restrict__ sobs, float2 *__restrict__ spred,
                                                             float2 *__restrict__ zout, double *__restrict__ part) {
  constexpr int D = R1 * R2, S = R1 / R2, G = kColThreads / R2, Hx = D / 2 + 1;
  __shared__ float2 tw[D];
  __shared__ float2 sb[G][R1 * (R2 + 1)];
  __shared__ float2 so[R1][kColThreads];   // the observation's column spectrum, off the registers
  __shared__ double red[kColThreads / 32];
  for (int j = threadIdx.x; j < D; j += kColThreads) {
    float sn, cs;
    sincospif(2.0f * (float)j / (float)D, &sn, &cs);
    tw[j] = make_float2(cs, -sn);   // W_D^j = exp(-2 pi i j / D)
  }
  __syncthreads();
  const int i = blockIdx.y, g = threadIdx.x / R2, t = threadIdx.x % R2;
  const int kx0 = blockIdx.x * G + g;
  const bool act = kx0 < Hx;
  const int kx = act ? kx0 : Hx - 1;
  const size_t col = (size_t)i * D * Hx + kx;
  float2 f[R1];
  {
    float2 o[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) o[n1] = sobs[col + (size_t)(R2 * n1 + t) * Hx];
    fft_col<R1, R2>(o, t, sb[g], tw);
#pragma unroll
    for (int q = 0; q < R1; ++q) so[q][threadIdx.x] = o[q];
  }
#pragma unroll
  for (int n1 = 0; n1 < R1; ++n1) f[n1] = spec[col + (size_t)(R2 * n1 + t) * Hx];
  fft_col<R1, R2>(f, t, sb[g], tw);
  const CtfP P = ctfp[i];
  const float gsc = 2.0f / ((float)D * (float)D), ps = 1.0f / ((float)D * (float)D);
  const bool nx = 2 * kx == D;
  const float wgt = (kx == 0 || nx) ? 1.f : 2.f;
  const double kxd = kx;
  float lsum = 0.f;
#pragma unroll
  for (int q = 0; q < R1; ++q) {
    const int ky = (t * S + q / R2) + R1 * (q % R2);
    const bool ny = 2 * ky == D;
    const double kyd = 2 * ky < D ? ky : ky - D;
    // Nyquist bins average their +-1/(2 px) aliases (reading L12): sign flips of kx or ky
    float C = 0.f;
    for (int a = 0; a < (nx ? 2 : 1); ++a)
      for (int b2 = 0; b2 < (ny ? 2 : 1); ++b2) {
        const double fx = a ? -kxd : kxd, fy = b2 ? -kyd : kyd;
        C += ctf_raw(P, fx * fx + fy * fy, fx * fx - fy * fy, 2.0 * fx * fy);
      }
    if (nx || ny) C *= (nx && ny) ? 0.25f : 0.5f;
    const float2 F = f[q], Ob = so[q][threadIdx.x];
    const float Rr = C * F.x - Ob.x, Ri = C * F.y - Ob.y;
    lsum = fmaf(wgt, fmaf(Rr, Rr, Ri * Ri), lsum);
    f[q] = make_float2(gsc * C * Rr, gsc * C * Ri);
    so[q][threadIdx.x] = make_float2(C * F.x * ps, C * F.y * ps);
  }
  // inverse column DFTs in fft_col's output order (fft_col_inv): thread t ends with the rows
  // R2 n1 + t, n1 = 0 .. R1 - 1, of column kx
  // gradient: rows (2m, 2m + 1) of the row spectrum, A and B, packed as one complex row
  // Z_m = A + i B over all D columns (A[D - kx] = conj A[kx]); the inverse C2C of Z_m is then
  // (g[2m][u], g[2m + 1][u]) interleaved: the layout k_render_bwd reads.  The imaginary parts
  // at kx = 0 and D/2 are dropped (what a C2R of the Hermitian half spectrum computes).  Row
  // R2 n1 + t pairs with row R2 n1 + (t ^ 1), held by lane t ^ 1 of the group.
  {
    fft_col_inv<R1, R2>(f, t, sb[g], tw);
    float2 *zi = zout + (size_t)i * (D / 2) * D;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const float2 mine = f[n1];
      const float2 other = make_float2(__shfl_xor_sync(0xffffffffu, mine.x, 1), __shfl_xor_sync(0xffffffffu, mine.y, 1));
      if (act && !(t & 1)) {
        const int m = (R2 * n1 + t) >> 1;   // A = row 2m (mine), B = row 2m + 1 (other)
        if (kx == 0 || nx) {
          zi[(size_t)m * D + kx] = make_float2(mine.x, other.x);
        } else {
          zi[(size_t)m * D + kx] = make_float2(mine.x - other.y, mine.y + other.x);
          zi[(size_t)m * D + (D - kx)] = make_float2(mine.x + other.y, other.x - mine.y);
        }
      }
    }
  }
  if (spred) {
#pragma unroll
    for (int q = 0; q < R1; ++q) f[q] = so[q][threadIdx.x];
    fft_col_inv<R1, R2>(f, t, sb[g], tw);
    if (act) {
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) spred[col + (size_t)(R2 * n1 + t) * Hx] = f[n1];
    }
  }
  double ls = act ? (double)lsum : 0.0;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ls;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < kColThreads / 32; ++w) sum += red[w];
    part[(size_t)i * gridDim.x + blockIdx.x] = sum / ((double)D * (double)D);
  }
}

template <int R1, int R2>
int colspec_blocks() { return (R1 * R2 / 2 + 1 + kColThreads / R2 - 1) / (kColThreads / R2); }

}  // namespace

void launch_ctf_params(const CfgDev &c, int B, const float *ctf, void *ctf_par, cudaStream_t s, int &launches) {
  k_ctf_params<<<(B + 127) / 128, 128, 0, s>>>(B, 1.0 / ((double)c.D * (double)c.px), ctf,
                                                reinterpret_cast<CtfP *>(ctf_par));
  ++launches;
}

bool spectral_rows(int D) { return D == 32 || D == 64 || D == 128 || D == 256; }

void launch_ctf_loss(const CfgDev &c, int B, const void *ctf_par, float2 *spec_hat, const float2 *spec_obs,
                     float2 *spec_pred, float2 *zout, double *loss_part, int loss_blocks, cudaStream_t s,
                     int &launches) {
  const CtfP *P = reinterpret_cast<const CtfP *>(ctf_par);
  dim3 grid(loss_blocks, B);
  switch (spectral_rows(c.D) ? c.D : 0) {
    case 32: k_ctf_colspec<8, 4><<<grid, kColThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, zout, loss_part); break;
    case 64: k_ctf_colspec<8, 8><<<grid, kColThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, zout, loss_part); break;
    case 128: k_ctf_colspec<16, 8><<<grid, kColThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, zout, loss_part); break;
    case 256: k_ctf_colspec<16, 16><<<grid, kColThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, zout, loss_part); break;
    default: k_ctf_loss<<<grid, kCtfThreads, 0, s>>>(c, P, spec_hat, spec_obs, spec_pred, loss_part);
  }
  ++launches;
}

void launch_loss_reduce(int B, const double *loss_part, int loss_blocks, double *loss, DevStats *st, int *ticket,
                        cudaStream_t s, int &launches) {
  k_loss_reduce<<<B, 128, 0, s>>>(B, loss_blocks, loss_part, loss, st, ticket);
  ++launches;
}

size_t ctf_par_bytes() { return sizeof(CtfP); }

int ctf_loss_blocks(int D) {
  switch (spectral_rows(D) ? D : 0) {
    case 32: return colspec_blocks<8, 4>();
    case 64: return colspec_blocks<8, 8>();
    case 128: return colspec_blocks<16, 8>();
    case 256: return colspec_blocks<16, 16>();
    default: return (D + kCtfRows - 1) / kCtfRows;
  }
}

}  // namespace gem
