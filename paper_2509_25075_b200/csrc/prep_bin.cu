// prep_bin.cu — a1 Gaussian prep, a2 splat preprocess + per-chunk tile
// histogram, device-wide exclusive scan, a3 stable per-tile list fill.
//
// Geometry follows App. A.2 (J = I for parallel rays, the
// exact marginal amplitude of P:500-501) and the Eq. 8 selection (PAPER.md:
// 219-225) realised as the integer k-sigma AABB (readings
// L1/L5/L6).  Every bound-relevant quantity is computed in fp64 with explicit
// round-to-nearest intrinsics (no FMA contraction) in the canonical op order of
// DESIGN.md §3 O3, so the cull lists are a bit-exact function of the fp32
// inputs.  Lists are emitted in ascending Gaussian id per tile (reading L9).
#include "gem_internal.cuh"

namespace gem {
namespace {

// MUFU.RSQ (rel. error < 2^-22): bound error ~1e-6 px, far inside the 1e-3 px exactness margin
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {   // 1 ulp: the amplitude and conic only
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Rounding on the FMA/ALU pipes instead of the XU (FRND / F2I run at 16 lanes/clk/SM): for
// |x| < 2^22, x + 1.5 * 2^23 rounds x to the nearest integer in the low mantissa bits.
constexpr float kMagicF = 12582912.f;      // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;
__device__ __forceinline__ float rint_fma(float x) { return __fsub_rn(__fadd_rn(x, kMagicF), kMagicF); }
__device__ __forceinline__ int iround_fma(float x) { return __float_as_int(__fadd_rn(x, kMagicF)) - kMagicBits; }
// exact int -> double (|i| < 2^31) by the 2^52 + 2^51 magic: one DADD, no I2F.F64
__device__ __forceinline__ double i2d_magic(int i) {
  return __dsub_rn(__hiloint2double(0x43380000, i ^ 0x80000000), 6755401588539392.0);   // 2^52 + 2^51 + 2^31
}

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsb(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

// ----------------------------------------------------------------- a1 prep
// q_hat = q/|q|, R(q_hat), sigma^2 = exp(2 s), Sigma = R diag(sigma^2) R^T,
// |Sigma| = exp(2 (s0+s1+s2))   (Eq. 4).  Degenerate (reading L18: skipped
// in every pair, zero gradient row, counted): |q| = 0, or q, Sigma, |Sigma|, mu or rho non-finite.
__global__ void __launch_bounds__(256) k_prep(int N, const float4 *__restrict__ mr, const float4 *__restrict__ ls,
                                              const float4 *__restrict__ q, GaussPrep *__restrict__ prep,
                                              DevStats *st) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  float4 qq = q[j], ss = ls[j];
  const float4 m4 = mr[j];
  double w = qq.x, x = qq.y, y = qq.z, z = qq.w;
  double n = sqrt(da(da(da(dm(w, w), dm(x, x)), dm(y, y)), dm(z, z)));
  GaussPrep p;
  bool ok = (n > 0.0) && isfinite(n);
  if (ok) {
    w = dv(w, n); x = dv(x, n); y = dv(y, n); z = dv(z, n);
    double R[9];
    R[0] = dsb(1.0, dm(2.0, da(dm(y, y), dm(z, z))));
    R[1] = dm(2.0, dsb(dm(x, y), dm(w, z)));
    R[2] = dm(2.0, da(dm(x, z), dm(w, y)));
    R[3] = dm(2.0, da(dm(x, y), dm(w, z)));
    R[4] = dsb(1.0, dm(2.0, da(dm(x, x), dm(z, z))));
    R[5] = dm(2.0, dsb(dm(y, z), dm(w, x)));
    R[6] = dm(2.0, dsb(dm(x, z), dm(w, y)));
    R[7] = dm(2.0, da(dm(y, z), dm(w, x)));
    R[8] = dsb(1.0, dm(2.0, da(dm(x, x), dm(y, y))));
    double s0 = ss.x, s1 = ss.y, s2 = ss.z;
    double e0 = exp(dm(2.0, s0)), e1 = exp(dm(2.0, s1)), e2 = exp(dm(2.0, s2));
    const int K[6] = {0, 0, 0, 1, 1, 2}, Lx[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      int k = K[e], l = Lx[e];
      p.sig[e] = da(da(dm(dm(R[3 * k + 0], e0), R[3 * l + 0]), dm(dm(R[3 * k + 1], e1), R[3 * l + 1])),
                    dm(dm(R[3 * k + 2], e2), R[3 * l + 2]));
    }
    p.detS = exp(dm(2.0, da(da(s0, s1), s2)));
    p.sdetS = exp(da(da(s0, s1), s2));   // |Sigma|^{1/2} (amplitude only, not bound-critical)
    ok = isfinite(p.detS) && isfinite(p.sig[0]) && isfinite(p.sig[3]) && isfinite(p.sig[5]) && isfinite(m4.x) &&
         isfinite(m4.y) && isfinite(m4.z) && isfinite(m4.w);
  }
  if (!ok) {
#pragma unroll
    for (int e = 0; e < 6; ++e) p.sig[e] = 0.0;
    p.detS = 0.0;
    p.sdetS = 0.0;
    atomicAdd(&st->degenerate, 1);
  }
  p.ok = ok ? 1.0 : 0.0;
  prep[j] = p;
  // fp32 rotated frame (splat fast path)
  GaussPrep32 f;
  if (ok) {
    const float fw = qq.x, fx = qq.y, fy = qq.z, fz = qq.w;
    const float inv = rsqrtf(((fw * fw + fx * fx) + fy * fy) + fz * fz);
    const float w2 = fw * inv, x2 = fx * inv, y2 = fy * inv, z2 = fz * inv;
    const float Rf[9] = {1.f - 2.f * (y2 * y2 + z2 * z2), 2.f * (x2 * y2 - w2 * z2), 2.f * (x2 * z2 + w2 * y2),
                         2.f * (x2 * y2 + w2 * z2), 1.f - 2.f * (x2 * x2 + z2 * z2), 2.f * (y2 * z2 - w2 * x2),
                         2.f * (x2 * z2 - w2 * y2), 2.f * (y2 * z2 + w2 * x2), 1.f - 2.f * (x2 * x2 + y2 * y2)};
    const float sk[3] = {expf(2.f * ss.x), expf(2.f * ss.y), expf(2.f * ss.z)};
#pragma unroll
    for (int k = 0; k < 3; ++k) f.c[k] = make_float4(Rf[k], Rf[3 + k], Rf[6 + k], sk[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) f.c[k] = make_float4(0.f, 0.f, 0.f, -1.f);
  }
  reinterpret_cast<GaussPrep32 *>(prep + N)[j] = f;
}

__device__ __forceinline__ int clip_d(double v, int lo, int hi) {
  if (!(v >= (double)lo)) return lo;
  if (v > (double)hi) return hi;
  return (int)v;
}

// --------------------------------------------------- a2 splat + histogram
// Per (particle i, Gaussian j): m = W mu + t, Sigma_hat = [W Sigma W^T]_2x2,
// det2, conic, amp = rho sqrt(2 pi) sqrt(|Sigma|/det2) (App. A.2), integer
// k-sigma AABB; visible => count one entry per touched tile in a per-CTA
// smem histogram; hist layout [i][t][chunk] so that one flat exclusive scan
// yields every list's start (t-major) and each chunk's sub-offset.
// Canonical O3 chain in fp64: bit-identical to the oracle.  Used only for the
// Gaussians whose fp32 bounds lie within 1e-3 px of an integer (or look degenerate).
__device__ __noinline__ bool splat_exact(const GaussPrep &g, const double *W, double tx, double ty, float4 m4,
                                         const CfgDev &c, double px, double ipx, double half, double kk, double tau,
                                         int &ulo, int &uhi, int &vlo, int &vhi, float &mxp, float &myp, float &aa,
                                         float &bb, float &cc2, float &ampf) {
  const double mu0 = m4.x, mu1 = m4.y, mu2 = m4.z, rho = m4.w;
  const double mxc = da(da(da(dm(W[0], mu0), dm(W[1], mu1)), dm(W[2], mu2)), tx);
  const double myc = da(da(da(dm(W[3], mu0), dm(W[4], mu1)), dm(W[5], mu2)), ty);
  const double S00 = g.sig[0], S01 = g.sig[1], S02 = g.sig[2], S11 = g.sig[3], S12 = g.sig[4], S22 = g.sig[5];
  const double v00 = da(da(dm(S00, W[0]), dm(S01, W[1])), dm(S02, W[2]));
  const double v01 = da(da(dm(S01, W[0]), dm(S11, W[1])), dm(S12, W[2]));
  const double v02 = da(da(dm(S02, W[0]), dm(S12, W[1])), dm(S22, W[2]));
  const double v10 = da(da(dm(S00, W[3]), dm(S01, W[4])), dm(S02, W[5]));
  const double v11 = da(da(dm(S01, W[3]), dm(S11, W[4])), dm(S12, W[5]));
  const double v12 = da(da(dm(S02, W[3]), dm(S12, W[4])), dm(S22, W[5]));
  const double A = da(da(dm(W[0], v00), dm(W[1], v01)), dm(W[2], v02));
  const double Bc = da(da(dm(W[0], v10), dm(W[1], v11)), dm(W[2], v12));
  const double Cc = da(da(dm(W[3], v10), dm(W[4], v11)), dm(W[5], v12));
  const double det2 = dsb(dm(A, Cc), dm(Bc, Bc));
  const double ampc = dm(rho, dm(kSqrt2Pi, sqrt(dv(g.detS, det2))));
  const bool ok = g.ok != 0.0 && isfinite(mxc) && isfinite(myc) && isfinite(A) && isfinite(Cc) && isfinite(det2) &&
                  det2 > 0.0 && isfinite(ampc);
  ulo = 1; uhi = 0; vlo = 1; vhi = 0;
  if (!ok) return false;
  const double rx = dm(kk, sqrt(A)), ry = dm(kk, sqrt(Cc));
  ulo = clip_d(ceil(da(dv(dsb(mxc, rx), px), half)), 0, c.D);
  uhi = clip_d(floor(da(dv(da(mxc, rx), px), half)), -1, c.D - 1);
  vlo = clip_d(ceil(da(dv(dsb(myc, ry), px), half)), 0, c.D);
  vhi = clip_d(floor(da(dv(da(myc, ry), px), half)), -1, c.D - 1);
  if (!(fabs(ampc) > tau && ulo <= uhi && vlo <= vhi)) return false;
  const double mx = fma(W[0], mu0, fma(W[1], mu1, fma(W[2], mu2, tx)));
  const double my = fma(W[3], mu0, fma(W[4], mu1, fma(W[5], mu2, ty)));
  mxp = (float)(fma(mx, ipx, half) - (double)ulo);
  myp = (float)(fma(my, ipx, half) - (double)vlo);
  const double px2 = px * px;
  aa = (float)(Cc / det2 * px2);
  bb = (float)(-Bc / det2 * px2);
  cc2 = (float)(A / det2 * px2);
  ampf = (float)ampc;
  return true;
}

constexpr int kSplatThreads = 256;
#ifndef GEM_FILL_BOXCS
#define GEM_FILL_BOXCS 0
#endif
#ifndef GEM_SPLAT_PF
#define GEM_SPLAT_PF 1
#endif
constexpr int kSub = kChunk / kFillWarps;   // Gaussians per k_fill warp

template <bool PM>
__global__ void __launch_bounds__(kSplatThreads, 4) k_splat_count(CfgDev c, const GaussPrep *__restrict__ prep,
                                                               const float4 *__restrict__ mr,
                                                               const float *__restrict__ rot,
                                                               const float *__restrict__ shift,
                                                               SplatRec *__restrict__ rec, uint2 *__restrict__ box,
                                                               unsigned short *__restrict__ hist,
                                                               unsigned short *__restrict__ subcnt,
                                                               int *__restrict__ ptot, DevStats *__restrict__ st) {
  // [kFillWarps][NT] tile histograms of the chunk's kFillWarps sub-chunks (one per k_fill warp),
  // then the exact-path queue [kChunk]
  extern __shared__ int shist[];
  int *queue = shist + kFillWarps * c.NT;
  __shared__ int qn;
  const int i = blockIdx.y, ch = blockIdx.x, tid = threadIdx.x;
  const GaussPrep32 *__restrict__ prep32 = reinterpret_cast<const GaussPrep32 *>(prep + c.N);
  for (int t = tid; t < kFillWarps * c.NT; t += blockDim.x) shist[t] = 0;
  if (tid == 0) qn = 0;
  double W[9];
  float Wf[6];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) W[3 * r + cc] = (double)rot[9 * i + 3 * cc + r];
#pragma unroll
  for (int k = 0; k < 6; ++k) Wf[k] = (float)W[k];
  const double tx = shift[2 * i], ty = shift[2 * i + 1];
  const double px = c.px, half = (double)(c.D / 2), kk = c.k, tau = c.tau, ipx = 1.0 / px;
  const float kf = c.k, ipxf = (float)ipx, px2f = c.px * c.px, Df = (float)c.D, tauf = (float)tau;
  unsigned pairs = 0;
  constexpr bool pixmask = PM;
  __syncthreads();
  auto emit = [&](int j, bool vis, int ulo, int uhi, int vlo, int vhi, float mxp, float myp, float aa, float bb,
                  float cc2, float ampf) {
    SplatRec o;
    if (vis) {
      o.f0 = make_float4(mxp, myp, aa, bb);
      o.f1 = make_float4(cc2, ampf, __int_as_float((ulo & 0xffff) | (uhi << 16)),
                         __int_as_float((vlo & 0xffff) | (vhi << 16)));
      pairs += (unsigned)((uhi - ulo + 1) * (vhi - vlo + 1));
      const int tu0 = (ulo >> c.tshift), tu1 = (uhi >> c.tshift), tv0 = (vlo >> c.tshift), tv1 = (vhi >> c.tshift);
      int *sub = shist + ((j - ch * kChunk) / kSub) * c.NT;
      if (!pixmask) {
        if (tu1 - tu0 <= 1 && tv1 - tv0 <= 1) {   // the usual case: a 1x1 .. 2x2 tile rectangle
          int *h0 = sub + tv0 * c.nt + tu0;
          atomicAdd(h0, 1);
          if (tu1 > tu0) atomicAdd(h0 + 1, 1);
          if (tv1 > tv0) {
            atomicAdd(h0 + c.nt, 1);
            if (tu1 > tu0) atomicAdd(h0 + c.nt + 1, 1);
          }
        } else {
          for (int tv = tv0; tv <= tv1; ++tv)
            for (int tu = tu0; tu <= tu1; ++tu) atomicAdd(&sub[tv * c.nt + tu], 1);
        }
      } else {   // per-pixel selection: only tiles holding a kept pixel (exact ellipse-tile test)
        const float tq = keep_q(c, ampf), ucen = (float)ulo + mxp, vcen = (float)vlo + myp;
        for (int tv = tv0; tv <= tv1; ++tv)
          for (int tu = tu0; tu <= tu1; ++tu)
            if (tile_kept(ucen, vcen, aa, bb, cc2, tq, max(ulo, tu << c.tshift), min(uhi, (tu << c.tshift) + c.T - 1),
                          max(vlo, tv << c.tshift), min(vhi, (tv << c.tshift) + c.T - 1)))
              atomicAdd(&sub[tv * c.nt + tu], 1);
      }
    } else {
      ulo = 1; uhi = 0; vlo = 1; vhi = 0;
      o.f0 = make_float4(0.f, 0.f, 0.f, 0.f);
      o.f1 = make_float4(0.f, 0.f, __int_as_float(1), __int_as_float(1));
    }
    const size_t ij = (size_t)i * c.N + j;
    rec[ij] = o;
    box[ij] = make_uint2((unsigned)(ulo & 0xffff) | ((unsigned)uhi << 16), (unsigned)(vlo & 0xffff) | ((unsigned)vhi << 16));
  };
#if GEM_SPLAT_PF
  // the next Gaussian's parameters are loaded one iteration ahead (L2 latency off the chain)
  float4 m4n = make_float4(0.f, 0.f, 0.f, 0.f);
  GaussPrep32 g32n;
  {
    const int j = ch * kChunk + tid;
    if (j < c.N) { m4n = mr[j]; g32n = prep32[j]; }
  }
#endif
  for (int r = 0; r < kChunk / kSplatThreads; ++r) {
    const int j = ch * kChunk + r * kSplatThreads + tid;
    if (j >= c.N) break;
#if GEM_SPLAT_PF
    const float4 m4 = m4n;
    const GaussPrep32 g32 = g32n;
    if (r + 1 < kChunk / kSplatThreads && j + kSplatThreads < c.N) {
      m4n = mr[j + kSplatThreads];
      g32n = prep32[j + kSplatThreads];
    }
#else
    const float4 m4 = mr[j];
    const GaussPrep32 g32 = prep32[j];
#endif
    // centre in fp64 (the record stores it relative to the box corner to ~1e-7 px)
    const double mx = fma(W[0], (double)m4.x, fma(W[1], (double)m4.y, fma(W[2], (double)m4.z, tx)));
    const double my = fma(W[3], (double)m4.x, fma(W[4], (double)m4.y, fma(W[5], (double)m4.z, ty)));
    const double mxd = fma(mx, ipx, half), myd = fma(my, ipx, half);
    // fp32 fast path: Sigma_hat from the rotated frame as sums of positive terms (no
    // cancellation): A = sum s_k p_k^2, C = sum s_k q_k^2, B = sum s_k p_k q_k, and by
    // Cauchy-Binet det2 = sum_{k<l} s_k s_l (p_k q_l - p_l q_k)^2, p_k = W_0 . r_k, q_k = W_1 . r_k.
    float p[3], q[3], s3[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float4 ck = g32.c[k];
      p[k] = fmaf(Wf[0], ck.x, fmaf(Wf[1], ck.y, Wf[2] * ck.z));
      q[k] = fmaf(Wf[3], ck.x, fmaf(Wf[4], ck.y, Wf[5] * ck.z));
      s3[k] = ck.w;
    }
    const float Af = fmaf(s3[0], p[0] * p[0], fmaf(s3[1], p[1] * p[1], s3[2] * p[2] * p[2]));
    const float Cf = fmaf(s3[0], q[0] * q[0], fmaf(s3[1], q[1] * q[1], s3[2] * q[2] * q[2]));
    const float Bf = fmaf(s3[0], p[0] * q[0], fmaf(s3[1], p[1] * q[1], s3[2] * p[2] * q[2]));
    const float x01 = fmaf(p[0], q[1], -p[1] * q[0]), x02 = fmaf(p[0], q[2], -p[2] * q[0]),
                x12 = fmaf(p[1], q[2], -p[2] * q[1]);
    const float d2f = fmaf(s3[0] * s3[1], x01 * x01, fmaf(s3[0] * s3[2], x02 * x02, s3[1] * s3[2] * x12 * x12));
    const float ampf = m4.w * 2.5066282746310002f * rsqrt_approx(d2f * rcp_approx(s3[0] * s3[1] * s3[2]));
    const float cx = (float)mxd, cy = (float)myd;
    const float rxp = kf * (Af * rsqrt_approx(Af)) * ipxf, ryp = kf * (Cf * rsqrt_approx(Cf)) * ipxf;
    const float fu0 = cx - rxp, fu1 = cx + rxp, fv0 = cy - ryp, fv1 = cy + ryp;
    // fp32 error of a bound (pixel units): the fp64 centre rounded to fp32 and the sums carry
    // <= ~4 ulp of |bound| (2.4e-7 |f|); the half-width k sqrt(A) / px carries <= k dp sqrt(tr Sigma)
    // / px with dp ~ 1.5e-6 the error of the fp32 projected axes (A = sum s p^2 with positive
    // terms: Cauchy-Schwarz), bounded with sqrt(x) <= (x + 1) / 2.  A floor/ceil is certain unless
    // the bound lies within e = 1e-4 + 2.4e-7 |f| + 5e-6 (tr Sigma / px^2 + 1) / 2 px of an integer
    // (or anything looks degenerate) -> exact queue.  (e grows with D and with the Gaussian.)
    const float trs = 2.5e-6f * fmaf(s3[0] + s3[1] + s3[2], ipxf * ipxf, 1.f);
    auto nearint = [&](float f, float r) { return fabsf(f - r) < fmaf(2.4e-7f, fabsf(f), 1e-4f + trs); };
    // |bounds| < 2^21 keeps the magic-number rounding exact (the clip below goes to [-1, D])
    const bool okf = s3[0] >= 0.f && d2f > 0.f && fabsf(ampf) < 3e38f && fabsf(fu0) < 2e6f && fabsf(fu1) < 2e6f &&
                     fabsf(fv0) < 2e6f && fabsf(fv1) < 2e6f;
    const float ru0 = rint_fma(fu0), ru1 = rint_fma(fu1), rv0 = rint_fma(fv0), rv1 = rint_fma(fv1);
    // (bitwise ORs: one predicate chain, no short-circuit branches)
    const bool near = nearint(fu0, ru0) | nearint(fu1, ru1) | nearint(fv0, rv0) | nearint(fv1, rv1) |
                      (tau > 0.0 && fabsf(fabsf(ampf) - tauf) <= 1e-4f * tauf);
    if (s3[0] >= 0.f && (!okf || near)) {   // deferred to the exact pass (compact, no warp divergence)
      queue[atomicAdd(&qn, 1)] = j;
      continue;
    }
    // not near an integer: ceil(x) = rint(x) + (rint(x) < x), floor(x) = rint(x) - (rint(x) > x);
    // clip as the canonical chain does: lo to [0, D], hi to [-1, D-1]
    const float cu0 = ru0 + (ru0 < fu0 ? 1.f : 0.f), fu1f = ru1 - (ru1 > fu1 ? 1.f : 0.f);
    const float cv0 = rv0 + (rv0 < fv0 ? 1.f : 0.f), fv1f = rv1 - (rv1 > fv1 ? 1.f : 0.f);
    const int ulo = iround_fma(fminf(fmaxf(cu0, 0.f), Df));
    const int uhi = iround_fma(fmaxf(fminf(fu1f, Df - 1.f), -1.f));
    const int vlo = iround_fma(fminf(fmaxf(cv0, 0.f), Df));
    const int vhi = iround_fma(fmaxf(fminf(fv1f, Df - 1.f), -1.f));
    const bool vis = okf && fabsf(ampf) > tauf && ulo <= uhi && vlo <= vhi;
    const float id2 = px2f * rcp_approx(d2f);   // (d2f > 0 and ampf finite on this path)
    emit(j, vis, ulo, uhi, vlo, vhi, (float)__dsub_rn(mxd, i2d_magic(ulo)), (float)__dsub_rn(myd, i2d_magic(vlo)),
         Cf * id2, -Bf * id2, Af * id2, ampf);
  }
  __syncthreads();
  for (int k = tid; k < qn; k += blockDim.x) {   // exact pass over the deferred Gaussians
    const int j = queue[k];
    int ulo, uhi, vlo, vhi;
    float mxp = 0.f, myp = 0.f, aa = 0.f, bb = 0.f, cc2 = 0.f, ampf = 0.f;
    const bool vis = splat_exact(prep[j], W, tx, ty, mr[j], c, px, ipx, half, kk, tau, ulo, uhi, vlo, vhi, mxp, myp,
                                 aa, bb, cc2, ampf);
    emit(j, vis, ulo, uhi, vlo, vhi, mxp, myp, aa, bb, cc2, ampf);
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, d);
  if ((tid & 31) == 0 && pairs) atomicAdd(&st->pairs, (unsigned long long)pairs);
  __syncthreads();
  unsigned short *sc = subcnt + ((size_t)i * c.C + ch) * kFillWarps * c.NT;   // (counts <= kChunk: 16 bits)
  int ctot = 0;   // the chunk's entries, added to the particle's total (k_scan_pp's starts)
  for (int t = tid; t < c.NT; t += blockDim.x) {
    int tot = 0;
#pragma unroll
    for (int w = 0; w < kFillWarps; ++w) {
      const int v = shist[w * c.NT + t];
      sc[w * c.NT + t] = (unsigned short)v;
      tot += v;
    }
    hist[((size_t)i * c.C + ch) * c.NT + t] = (unsigned short)tot;   // [i][chunk][t]: coalesced
    ctot += tot;
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) ctot += __shfl_xor_sync(0xffffffffu, ctot, d);
  if ((tid & 31) == 0 && ctot) atomicAdd(ptot + i, ctot);
}

// ------------------------------------------------------------------- scan
// Device-wide exclusive scan of int32 (3 phases; each block scans 4096 items).
constexpr int kScanThreads = 1024, kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_excl_scan(int v, int *smem_warp, int &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) smem_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? smem_warp[lane] : 0;
    int si = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, si, d);
      if (lane >= d) si += y;
    }
    if (lane < nw) smem_warp[lane] = si - s;
    if (lane == 31) smem_warp[32] = si;
  }
  __syncthreads();
  total = smem_warp[32];
  int r = incl - v + smem_warp[wid];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_local(const int *__restrict__ in, int *__restrict__ out,
                                                             int64_t n, int *__restrict__ blk) {
  __shared__ int sw[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems], s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0;
    s += v[k];
  }
  int total;
  int e = block_excl_scan(s, sw, total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = e;
    e += v[k];
  }
  if (threadIdx.x == 0) blk[blockIdx.x] = total;
}

// single block: exclusive scan of the block totals; writes out[n] = total.
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(int *__restrict__ blk, int64_t nblk, int *__restrict__ out,
                                                              int64_t n, DevStats *st, int64_t cap) {
  __shared__ int sw[33];
  int carry = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += kScanThreads) {
    int64_t b = b0 + threadIdx.x;
    int v = b < nblk ? blk[b] : 0;
    int total;
    int e = block_excl_scan(v, sw, total);
    if (b < nblk) blk[b] = e + carry;
    carry += total;
  }
  if (threadIdx.x == 0) {   // totals accumulate over the waves of one forward
    out[n] = carry;
    st->entries += (unsigned long long)carry;
    if ((int64_t)carry > cap) st->overflow = 1;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(int *__restrict__ out, int64_t n, const int *__restrict__ blk) {
  const int add = blk[blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  for (int k = threadIdx.x; k < kScanTile; k += kScanThreads)
    if (base + k < n) out[base + k] += add;
}

// List offsets, one CTA per particle, with no inter-block dependency: the splat kernel added each
// chunk's entry count to ptot[i], so CTA i starts its particle at pbase = sum_{i' < i} ptot[i']
// (a block reduction) and writes pbase + the exclusive scan, in (tile, chunk) order, of its own
// counts: the global exclusive scan of the whole array in (i, t, chunk) order, stored in the
// [i][chunk][t] layout the splat writes and the fill reads coalesced (list_bounds for the
// readers) plus each list's start in lst[i NT + t] (the last CTA writes lst[B NT] = all entries).  Entries beyond the capacity set the overflow
// flags (the fill never writes past the buffer; the step's outputs are then invalid, include/gem.h).
constexpr int kPpThreads = 1024;

__global__ void __launch_bounds__(kPpThreads) k_scan_pp(const unsigned short *__restrict__ hist, int *__restrict__ base,
                                                        int *__restrict__ lst, int NT, int C, int B,
                                                        const int *__restrict__ ptot, int64_t cap, DevStats *st,
                                                        int *tk) {
  __shared__ int sw[33];
  const int i = blockIdx.x, seg = NT * C;
  // this particle's start: the entries of the particles before it
  int pb = 0;
  for (int b = threadIdx.x; b < i; b += kPpThreads) pb += __ldg(ptot + b);
  int pbase;
  block_excl_scan(pb, sw, pbase);
  const unsigned short *in = hist + (size_t)i * seg;
  int *out = base + (size_t)i * seg;
  // scan order (t, chunk) over the [chunk][t] layout: thread tau owns tile t = t0 + tau of a
  // block of kPpThreads tiles and its C chunk counts (coalesced across the threads for each
  // chunk, all loads in flight); one block scan of the tiles' totals per block of tiles, the
  // running total carried between blocks; the chunk starts re-read from L1
  int carry = pbase;
  for (int t0 = 0; t0 < NT; t0 += kPpThreads) {
    const int t = t0 + threadIdx.x;
    int sum = 0;
    if (t < NT) {
#pragma unroll 8
      for (int ch = 0; ch < C; ++ch) sum += __ldg(in + (size_t)ch * NT + t);
    }
    int total;
    int run = carry + block_excl_scan(sum, sw, total);
    if (t < NT) {
      lst[(size_t)i * NT + t] = run;   // the list's own start (chunk 0)
#pragma unroll 8
      for (int ch = 0; ch < C; ++ch) {
        out[(size_t)ch * NT + t] = run;
        run += __ldg(in + (size_t)ch * NT + t);
      }
    }
    carry += total;
  }
  if (threadIdx.x == 0 && i == B - 1) {   // totals accumulate over the waves of one forward
    lst[(size_t)B * NT] = carry;
    st->entries += (unsigned long long)carry;
    if ((int64_t)carry > cap) { st->overflow = 1; tk[4] = 1; }   // tk[4]: sticky until gem_stats
  }
}

// --------------------------------------------------------------- a3 fill
// One CTA of 4 warps per (particle, chunk of kChunk Gaussians); warp w owns the sub-chunk w.
// The splat kernel counted each sub-chunk's entries per tile; those counts, seeded with the
// chunk's global offset (the device scan), give each warp its per-tile cursors; the warp then
// visits its Gaussians 32 per step (consecutive ids) and emits each step's entries per tile in
// lane order.  Chunks, sub-chunks and steps are in id order, so every tile's list is in
// ascending Gaussian id: the oracle's O4 list, element by element.


// ZK (GEM_FLAG_ZSORT): entries are written as (id, z-sort key ord32(fp32(z_ij))) pairs to
// zpair[slot] instead of ids[slot] -- one 8-byte store costs the same DRAM sectors as the 4-byte
// id -- with the key computed once per Gaussian from a coalesced read of mean_rho; the sort
// kernel reads the pairs and writes the sorted ids.
template <bool ZK, bool PM>
__global__ void __launch_bounds__(kFillWarps * 32) k_fill(CfgDev c, const uint2 *__restrict__ box,
                                                          const int *__restrict__ base,
                                                          const unsigned short *__restrict__ subcnt, int *__restrict__ ids,
                                                          const float4 *__restrict__ mean_rho,
                                                          const float *__restrict__ rot, uint2 *__restrict__ zpair,
                                                          const SplatRec *__restrict__ rec) {
  extern __shared__ int cnt[];   // [kFillWarps][NT] cursors
  __shared__ unsigned smask[kFillWarps * 64];   // per warp: lane sets of the step's tiles
  const int i = blockIdx.y, ch = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < kFillWarps * 64; t += blockDim.x) smask[t] = 0u;
  int *mine = cnt + w * c.NT;
  const int jsub = ch * kChunk + w * kSub;
  const uint2 *boxi = box + (size_t)i * c.N;
  // cursors: the chunk's offset of each tile plus the counts of the preceding sub-chunks (the
  // splat kernel counted each sub-chunk's entries per tile)
  const unsigned short *sc = subcnt + ((size_t)i * c.C + ch) * kFillWarps * c.NT;
  for (int t = threadIdx.x; t < c.NT; t += blockDim.x) {
    int run = base[((size_t)i * c.C + ch) * c.NT + t];
#pragma unroll
    for (int ww = 0; ww < kFillWarps; ++ww) {
      cnt[ww * c.NT + t] = run;
      run += sc[ww * c.NT + t];
    }
  }
  __syncthreads();
  constexpr bool pixmask = PM;
  const unsigned lt = (1u << lane) - 1u;
  double w0 = 0.0, w1 = 0.0, w2 = 0.0;
  if (ZK) { w0 = (double)rot[9 * i + 2]; w1 = (double)rot[9 * i + 5]; w2 = (double)rot[9 * i + 8]; }
  uint2 bnext = make_uint2(1u, 0u);   // the next step's box, loaded one step ahead
#if GEM_FILL_BOXCS   // the boxes are read once: evict-first
#define LDBOX(p_) __ldcs(p_)
#else
#define LDBOX(p_) (*(p_))
#endif
  if (jsub + lane < c.N) bnext = LDBOX(boxi + jsub + lane);
  for (int step = 0; step < kSub / 32; ++step) {     // pass 2: deterministic fill
    const int j0 = jsub + step * 32;
    if (j0 >= c.N) break;
    const int j = j0 + lane;
    const uint2 bcur = bnext;
    if (step + 1 < kSub / 32 && j + 32 < c.N) bnext = LDBOX(boxi + j + 32);
    int tu0 = 0, tv0 = 0, ntu = 0, ntv = 0;
    if (j < c.N) {
      const uint2 b = bcur;
      const int ulo = (int)(b.x & 0xffff), uhi = (int)(b.x >> 16), vlo = (int)(b.y & 0xffff), vhi = (int)(b.y >> 16);
      if (ulo <= uhi && vlo <= vhi) {
        tu0 = ulo >> c.tshift; tv0 = vlo >> c.tshift;
        ntu = (uhi >> c.tshift) - tu0 + 1; ntv = (vhi >> c.tshift) - tv0 + 1;
      }
    }
    unsigned key = 0;
    if (ZK && ntu > 0) key = ord32(__double2float_rn(zdepth64(__ldg(mean_rho + j), w0, w1, w2)));
    // per-pixel selection: the same exact tile test as the splat kernel's histogram
    float ucen = 0.f, vcen = 0.f, ca = 0.f, cb = 0.f, cc = 0.f, tq = 0.f;
    int ulo = 0, uhi = -1, vlo = 0, vhi = -1;
    if (pixmask && ntu > 0) {
      const SplatRec r = rec[(size_t)i * c.N + j];
      ulo = (int)(__float_as_uint(r.f1.z) & 0xffff); uhi = (int)(__float_as_uint(r.f1.z) >> 16);
      vlo = (int)(__float_as_uint(r.f1.w) & 0xffff); vhi = (int)(__float_as_uint(r.f1.w) >> 16);
      ucen = (float)ulo + r.f0.x; vcen = (float)vlo + r.f0.y;
      ca = r.f0.z; cb = r.f0.w; cc = r.f1.x; tq = keep_q(c, r.f1.y);
    }
    // Ascending Gaussian id within each tile (O4 order, reading L9): the step's 32 Gaussians are
    // consecutive ids, so a tile's entries from this step go in lane order.  Each lane keeps a
    // bit mask of the cells of its tile rectangle still to be emitted; per round the first lane
    // with work names its first pending tile, a ballot of the lanes whose rectangle holds that
    // tile gives each its rank, and the tile's cursor advances once (rounds = distinct tiles the
    // step touches).  Rectangles wider than 8 or taller than 4 tiles (huge boxes) send the step to a serial
    // path: lanes one after the other, the warp spreading each rectangle over its 32 lanes.
    const bool act = ntu > 0;
    auto kept = [&](int tu, int tv) {
      return !pixmask || tile_kept(ucen, vcen, ca, cb, cc, tq, max(ulo, tu << c.tshift),
                                   min(uhi, (tu << c.tshift) + c.T - 1), max(vlo, tv << c.tshift),
                                   min(vhi, (tv << c.tshift) + c.T - 1));
    };
    auto put = [&](int slot, int jj, unsigned kk) {
      if ((int64_t)slot < c.cap) {
        if (ZK) zpair[slot] = make_uint2((unsigned)jj, kk);
        else ids[slot] = jj;
      }
    };
    // Usual case: the union of the step's rectangles spans <= 64 tiles.  Each lane ORs its lane
    // bit into a per-warp shared word per tile of its rectangle; a tile's word is then the set
    // of the step's lanes holding it: rank = lanes below, and the lowest lane advances the
    // cursor and clears the word.
    const int ux0 = __reduce_min_sync(0xffffffffu, act ? tu0 : 0x7fffffff);
    if (ux0 == 0x7fffffff) continue;   // no visible Gaussian in this step
    const int vy0 = __reduce_min_sync(0xffffffffu, act ? tv0 : 0x7fffffff);
    const int uw = (int)__reduce_max_sync(0xffffffffu, act ? (unsigned)(tu0 + ntu) : 0u) - ux0;
    const int uh = (int)__reduce_max_sync(0xffffffffu, act ? (unsigned)(tv0 + ntv) : 0u) - vy0;
    if (uw * uh <= 64 && !__any_sync(0xffffffffu, ntu > 2 || ntv > 2)) {
      // every rectangle within 2 x 2 tiles: the three phases unrolled over the four cells
      unsigned *sm = smask + 64 * w;
      const int cbase = (tv0 - vy0) * uw + (tu0 - ux0);
      bool val[4];
      int cell[4], tt[4], cur[4];
      unsigned m[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int du = q & 1, dv = q >> 1;
        val[q] = act && du < ntu && dv < ntv && kept(tu0 + du, tv0 + dv);
        cell[q] = cbase + dv * uw + du;
        tt[q] = (tv0 + dv) * c.nt + tu0 + du;
        if (val[q]) atomicOr(&sm[cell[q]], 1u << lane);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (val[q]) { m[q] = sm[cell[q]]; cur[q] = mine[tt[q]]; }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (val[q]) {
          put(cur[q] + __popc(m[q] & lt), j, key);
          if (!(m[q] & lt)) {   // the tile's lowest lane advances the cursor and clears the word
            mine[tt[q]] = cur[q] + __popc(m[q]);
            sm[cell[q]] = 0u;
          }
        }
      __syncwarp();
    } else if (uw * uh <= 64) {
      unsigned *sm = smask + 64 * w;
      const int cbase = (tv0 - vy0) * uw + (tu0 - ux0);
      if (act)
        for (int dv = 0; dv < ntv; ++dv)
          for (int du = 0; du < ntu; ++du)
            if (kept(tu0 + du, tv0 + dv)) atomicOr(&sm[cbase + dv * uw + du], 1u << lane);
      __syncwarp();
      if (act)
        for (int dv = 0; dv < ntv; ++dv)
          for (int du = 0; du < ntu; ++du) {
            const unsigned m = sm[cbase + dv * uw + du];
            if ((m >> lane) & 1u) put(mine[(tv0 + dv) * c.nt + tu0 + du] + __popc(m & lt), j, key);
          }
      __syncwarp();
      if (act)
        for (int dv = 0; dv < ntv; ++dv)
          for (int du = 0; du < ntu; ++du) {
            const int cc_ = cbase + dv * uw + du;
            const unsigned m = sm[cc_];
            if (((m >> lane) & 1u) && !(m & lt)) {
              mine[(tv0 + dv) * c.nt + tu0 + du] += __popc(m);
              sm[cc_] = 0u;
            }
          }
      __syncwarp();
    } else if (!__any_sync(0xffffffffu, act && (ntu > 8 || ntv > 4))) {
      // cells (du, dv) of the rectangle at bit 8 dv + du: rectangles up to 8 x 4 tiles
      unsigned pend = 0;
      if (act) {
        const unsigned row = (0x1feu << (ntu - 1)) >> 8;   // the ntu low bits
        for (int r = 0; r < ntv; ++r) pend |= row << (8 * r);
      }
      if (pixmask)
        for (int n = 0; n < 32; ++n)
          if (((pend >> n) & 1u) && !kept(tu0 + (n & 7), tv0 + (n >> 3))) pend &= ~(1u << n);
      for (;;) {
        const unsigned lead = __ballot_sync(0xffffffffu, pend != 0);
        if (!lead) break;
        const int L = __ffs(lead) - 1;
        const int cl = __ffs(pend) - 1;   // the leader's first pending cell (garbage elsewhere)
        const int tup = __shfl_sync(0xffffffffu, tu0 + (cl & 7), L);
        const int tvp = __shfl_sync(0xffffffffu, tv0 + (cl >> 3), L);
        const unsigned du = (unsigned)(tup - tu0), dv = (unsigned)(tvp - tv0);
        const int cell = (int)(8 * dv + du);
        const bool in = act && du < (unsigned)ntu && dv < (unsigned)ntv && ((pend >> cell) & 1u);
        const unsigned m = __ballot_sync(0xffffffffu, in);
        const int t = tvp * c.nt + tup;
        const int cur = mine[t];
        if (in) {
          put(cur + __popc(m & lt), j, key);
          pend &= ~(1u << cell);
        }
        __syncwarp();
        if (lane == L) mine[t] = cur + __popc(m);
        __syncwarp();
      }
    } else {
      unsigned todo = __ballot_sync(0xffffffffu, act);
      while (todo) {
        const int L = __ffs(todo) - 1;
        todo &= todo - 1;
        const int a0 = __shfl_sync(0xffffffffu, tu0, L), b0 = __shfl_sync(0xffffffffu, tv0, L);
        const int na_ = __shfl_sync(0xffffffffu, ntu, L), nb_ = __shfl_sync(0xffffffffu, ntv, L);
        const unsigned kL = __shfl_sync(0xffffffffu, key, L);
        const float pu = __shfl_sync(0xffffffffu, ucen, L), pv = __shfl_sync(0xffffffffu, vcen, L);
        const float pa = __shfl_sync(0xffffffffu, ca, L), pb = __shfl_sync(0xffffffffu, cb, L);
        const float pc = __shfl_sync(0xffffffffu, cc, L), pt = __shfl_sync(0xffffffffu, tq, L);
        const int plo = __shfl_sync(0xffffffffu, ulo, L), phi = __shfl_sync(0xffffffffu, uhi, L);
        const int qlo = __shfl_sync(0xffffffffu, vlo, L), qhi = __shfl_sync(0xffffffffu, vhi, L);
        for (int n = lane; n < na_ * nb_; n += 32) {
          const int tv = b0 + n / na_, tu = a0 + n % na_;
          if (pixmask && !tile_kept(pu, pv, pa, pb, pc, pt, max(plo, tu << c.tshift), min(phi, (tu << c.tshift) + c.T - 1),
                                    max(qlo, tv << c.tshift), min(qhi, (tv << c.tshift) + c.T - 1)))
            continue;
          const int t = tv * c.nt + tu;
          put(mine[t]++, j0 + L, kL);
        }
        __syncwarp();
      }
    }
  }
}

}  // namespace

void launch_prep(const CfgDev &c, const float4 *mean_rho, const float4 *log_scale, const float4 *quat, GaussPrep *prep,
                 DevStats *st, cudaStream_t s, int &launches) {
  k_prep<<<(c.N + 255) / 256, 256, 0, s>>>(c.N, mean_rho, log_scale, quat, prep, st);
  ++launches;
}

void launch_splat_count(const CfgDev &c, int B, const GaussPrep *prep, const float4 *mean_rho, const float *rot,
                        const float *shift, SplatRec *rec, uint2 *box, unsigned short *hist, unsigned short *subcnt,
                        int *ptot, DevStats *st,
                        cudaStream_t s, int &launches) {
  dim3 grid(c.C, B);
  const size_t smem = (kFillWarps * c.NT + kChunk) * sizeof(int);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_splat_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_splat_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    init = true;
  }
  if (c.flags & GEM_FLAG_EXACT_TILES)
    k_splat_count<true><<<grid, kSplatThreads, smem, s>>>(c, prep, mean_rho, rot, shift, rec, box, hist, subcnt, ptot, st);
  else
    k_splat_count<false><<<grid, kSplatThreads, smem, s>>>(c, prep, mean_rho, rot, shift, rec, box, hist, subcnt, ptot,
                                                           st);
  ++launches;
}

void launch_scan(const int *in, int *out, int64_t n, int *blk, int64_t nblk, DevStats *st, int64_t cap, cudaStream_t s,
                 int &launches) {
  k_scan_local<<<(unsigned)nblk, kScanThreads, 0, s>>>(in, out, n, blk);
  k_scan_blocks<<<1, kScanThreads, 0, s>>>(blk, nblk, out, n, st, cap);
  k_scan_add<<<(unsigned)nblk, kScanThreads, 0, s>>>(out, n, blk);
  launches += 3;
}

void launch_scan_pp(const CfgDev &c, int B, const unsigned short *hist, int *base, int *lst, const int *ptot, DevStats *st,
                    int *tk, cudaStream_t s, int &launches) {
  k_scan_pp<<<B, kPpThreads, 0, s>>>(hist, base, lst, c.NT, c.C, B, ptot, c.cap, st, tk);
  ++launches;
}


void launch_fill(const CfgDev &c, int B, const uint2 *box, const int *base, const unsigned short *subcnt, int *ids,
                 const float4 *mean_rho, const float *rot, uint2 *zpair, const SplatRec *rec, cudaStream_t s,
                 int &launches) {
  dim3 grid(c.C, B);
  const size_t smem = (size_t)kFillWarps * c.NT * sizeof(int);
  const bool pm = (c.flags & GEM_FLAG_EXACT_TILES) != 0;
  auto kern = zpair ? (pm ? k_fill<true, true> : k_fill<true, false>) : (pm ? k_fill<false, true> : k_fill<false, false>);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kFillWarps * 32, smem, s>>>(c, box, base, subcnt, ids, mean_rho, rot, zpair, rec);
  ++launches;
}

}  // namespace gem
