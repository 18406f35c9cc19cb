// render.cu — a5 forward evaluate/project and a7 backward scatter over the
// per-tile lists.
//
// Forward (Eq. 6 with the Eq. 8 selection):
//   I_hat(u,v) = sum_{j in list(tile(u,v)), (u,v) in AABB_j} amp_j exp(-Q_j/2),
//   Q = a dx^2 + 2 b dx dy + c dy^2 (pixel units).
// One CTA (4 warps) per (particle, T x T tile); see k_render_fwd below for the
// warp-per-entry scheme (lanes over the pixels of one entry's box, warp-private
// smem accumulators, fixed-order reduction: bitwise deterministic).
//
// Backward ("gradient computation restricted to the Gaussians contributing to
// each pixel"): one thread per list entry loops over the
// pixels of AABB_j inside the tile (dL/dI_hat staged in smem), accumulating four
// per-row sums from which the six partials (L_amp, L_mx, L_my, L_a, L_b, L_c)
// follow algebraically; it then transforms them to
// world-frame accumulators (L_rho, G_mu, G_Sigma; DESIGN.md §3 O9) and adds
// them with three vector reductions red.global.add.v4.f32.
#include "gem_internal.cuh"

namespace gem {
namespace {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void red_add_v4(float4 *addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}


// Warp-per-entry forward.  Each warp takes batches of 32 consecutive list
// entries (batch b -> warp b % kFwdWarps), stages them in its own smem slot,
// and for each entry enumerates the pixels of AABB_j ∩ tile linearly over its
// 32 lanes (pixel p = pass*32 + lane -> row q = p / w, col r = p % w, computed
// exactly in fp32 with a round-to-nearest magic constant).  Values are added
// into a warp-private tile accumulator in smem: within a warp the lanes of one
// pass touch distinct pixels and entries are processed in order, so no atomics
// are needed; the kFwdWarps copies are summed in a fixed order at the end
// (bitwise deterministic).  Lane utilisation = |box ∩ tile| / 32 per pass.
constexpr int kFwdWarps = 4;

template <int T>
__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                                const int *__restrict__ base,
                                                                const int *__restrict__ ids,
                                                                float *__restrict__ proj) {
  constexpr int S = T + 8;                     // accumulator row stride (floats)
  __shared__ float acc[kFwdWarps][T * S];
  __shared__ float4 st0[kFwdWarps][32];        // (mx' + 1/2, my', A, B); mx' relative to the box∩tile corner
  __shared__ float4 st1[kFwdWarps][32];        // (C, amp, 1/w, w)
  __shared__ int2 st2[kFwdWarps][32];          // (npix, corner index | (S - w) << 16)
  const int t = blockIdx.x, i = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int u0 = (t % c.nt) * T, v0 = (t / c.nt) * T;
  const size_t hidx = ((size_t)i * c.NT + t) * c.C;
  int s = base[hidx], e = base[hidx + c.C];
  if ((int64_t)e > c.cap) e = (int)c.cap;
  if ((int64_t)s > c.cap) s = (int)c.cap;
  if (s >= e) {  // empty tile: the projection is zero there
    for (int pp = tid; pp < T * T; pp += kFwdWarps * 32) {
      const int u = u0 + pp % T, v = v0 + pp / T;
      if (u < c.D && v < c.D) proj[((size_t)i * c.D + v) * c.D + u] = 0.f;
    }
    return;
  }
  for (int k = lane; k < T * S; k += 32) acc[w][k] = 0.f;
  const SplatRec *reci = rec + (size_t)i * c.N;
  const float kA = -0.5f * kLog2e, kB = -kLog2e;
  const float laneh = (float)lane + 0.5f;
  const float M = 12582912.f;                   // 1.5 * 2^23: x + M rounds x to an integer
  float *accw = acc[w] + lane;
  __syncwarp();
  for (int b0 = s + 32 * w; b0 < e; b0 += 32 * kFwdWarps) {
    const int n = min(32, e - b0);
    if (lane < n) {
      const int id = ids[b0 + lane];
      const SplatRec r = reci[id];
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      const int bu0 = max(ulo - u0, 0), bu1 = min(uhi - u0, T - 1);
      const int bv0 = max(vlo - v0, 0), bv1 = min(vhi - v0, T - 1);
      const int wd = bu1 - bu0 + 1, ht = bv1 - bv0 + 1;
      st0[w][lane] = make_float4((float)(ulo - u0 - bu0) + r.f0.x + 0.5f, (float)(vlo - v0 - bv0) + r.f0.y,
                                 kA * r.f0.z, kB * r.f0.w);
      st1[w][lane] = make_float4(kA * r.f1.x, r.f1.y, 1.0f / (float)wd, (float)wd);
      st2[w][lane] = make_int2(wd * ht, (bv0 * S + bu0) | ((S - wd) << 16));
    }
    __syncwarp();
    for (int k = 0; k < n; ++k) {
      const float4 E0 = st0[w][k];
      const float4 E1 = st1[w][k];
      const int2 E2 = st2[w][k];
      const int npix = E2.x, corner = E2.y & 0xffff, sw = E2.y >> 16;
      float pfh = laneh;   // pixel index + 1/2
      int p0 = 0;
#pragma unroll 1
      do {
        const float xm = fmaf(pfh, E1.z, -0.5f) + M;          // round((p + 1/2)/w - 1/2) = p div w
        const float qf = xm - M;
        const int qi = __float_as_int(xm) - 0x4B400000;
        const float dx = fmaf(-qf, E1.w, pfh) - E0.x;            // (p mod w) - mx'
        const float dy = qf - E0.y;
        const float q = fmaf(fmaf(E0.z, dx, E0.w * dy), dx, E1.x * dy * dy);
        const float ev = ex2(q);
        if (p0 + lane < npix) {
          float *a = accw + corner + p0 + qi * sw;
          *a = fmaf(E1.y, ev, *a);
        }
        p0 += 32;
        pfh += 32.f;
      } while (p0 < npix);
    }
    __syncwarp();
  }
  __syncthreads();
  for (int pp = tid; pp < T * T; pp += kFwdWarps * 32) {
    const int pu = pp % T, pv = pp / T;
    float sum = 0.f;
#pragma unroll
    for (int ww = 0; ww < kFwdWarps; ++ww) sum += acc[ww][pv * S + pu];
    const int u = u0 + pu, v = v0 + pv;
    if (u < c.D && v < c.D) proj[((size_t)i * c.D + v) * c.D + u] = sum;
  }
}

// Backward: one thread per list entry.  A warp's time is set by its largest
// box ∩ tile, so each 256-entry chunk is first counting-sorted in smem by its
// (height, width) class: threads of a warp then loop over near-equal boxes.
constexpr int kBwdThreads = 256;
constexpr int kBwdKeys = 144;   // (min(h,12)-1)*12 + min(w,12)-1

template <int T>
__global__ void __launch_bounds__(kBwdThreads) k_render_bwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                             const int *__restrict__ base, const int *__restrict__ ids,
                                                             const float *__restrict__ dldi,
                                                             const float4 *__restrict__ mean_rho,
                                                             const float *__restrict__ rot, float4 *__restrict__ acc) {
  __shared__ float gs[T][T + 1];
  __shared__ float4 sr0[kBwdThreads], sr1[kBwdThreads];
  __shared__ int sid[kBwdThreads];
  __shared__ int hist[kBwdKeys];
  __shared__ int order[kBwdThreads];
  __shared__ int warp_tot[kBwdThreads / 32 + 1];
  const int t = blockIdx.x, i = blockIdx.y, tid = threadIdx.x;
  const int u0 = (t % c.nt) * T, v0 = (t / c.nt) * T;
  const size_t hidx = ((size_t)i * c.NT + t) * c.C;
  int s = base[hidx], e = base[hidx + c.C];
  if ((int64_t)e > c.cap) e = (int)c.cap;
  if ((int64_t)s > c.cap) s = (int)c.cap;
  if (s >= e) return;  // empty tile: no Gaussian touches it
  for (int pp = tid; pp < T * T; pp += kBwdThreads) {
    const int pu = pp % T, pv = pp / T, u = u0 + pu, v = v0 + pv;
    gs[pv][pu] = (u < c.D && v < c.D) ? dldi[((size_t)i * c.D + v) * c.D + u] : 0.f;
  }
  // W = P^T: W[r][k] = P[3k + r]; only rows 0 and 1 of W are needed.
  float W0[3], W1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    W0[k] = rot[9 * i + 3 * k];
    W1[k] = rot[9 * i + 3 * k + 1];
  }
  const float inv_px = 1.f / c.px, inv_px2 = inv_px * inv_px;
  const float nh = -0.5f * kLog2e;
  const SplatRec *reci = rec + (size_t)i * c.N;
  const int lane = tid & 31, wid = tid >> 5;
  for (int cs = s; cs < e; cs += kBwdThreads) {
    const int n = min(kBwdThreads, e - cs);
    for (int k = tid; k < kBwdKeys; k += kBwdThreads) hist[k] = 0;
    __syncthreads();
    int key = 0;
    if (tid < n) {
      const int id = ids[cs + tid];
      const SplatRec r = reci[id];
      sid[tid] = id;
      sr0[tid] = r.f0;
      sr1[tid] = r.f1;
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int wd = min(ub >> 16, u0 + T - 1) - max(ub & 0xffff, u0) + 1;
      const int ht = min(vb >> 16, v0 + T - 1) - max(vb & 0xffff, v0) + 1;
      key = (min(ht, 12) - 1) * 12 + (min(wd, 12) - 1);
      atomicAdd(&hist[key], 1);
    }
    __syncthreads();
    // exclusive scan of the key histogram (one value per thread, kBwdKeys <= 256)
    int hv = tid < kBwdKeys ? hist[tid] : 0, incl = hv;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int woff = 0;
    for (int ww = 0; ww < wid; ++ww) woff += warp_tot[ww];
    __syncthreads();
    if (tid < kBwdKeys) hist[tid] = woff + incl - hv;
    __syncthreads();
    if (tid < n) order[atomicAdd(&hist[key], 1)] = tid;
    __syncthreads();
    if (tid < n) {
      const int slot = order[tid];
      const int id = sid[slot];
      const float4 f0 = sr0[slot], f1 = sr1[slot];
      const int ub = __float_as_int(f1.z), vb = __float_as_int(f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      const float mxr = f0.x, myr = f0.y, a = f0.z, b = f0.w, cc = f1.x, amp = f1.y;
      const int ua = max(ulo, u0), ubnd = min(uhi, u0 + T - 1), va = max(vlo, v0), vbnd = min(vhi, v0 + T - 1);
      // Per row (dy fixed) accumulate T0 = sum g e, T1 = sum g e dx, T2 = sum g e dx^2; since
      // h = amp g e, the six partials are L_amp = sum T0 and, over rows,
      // L_mx = amp (a sum T1 + b sum dy T0), L_my = amp (b sum T1 + c sum dy T0),
      // L_a = -amp/2 sum T2, L_b = -amp sum dy T1, L_c = -amp/2 sum dy^2 T0.
      const float na = nh * a, nb2 = 2.f * nh * b, nc = nh * cc;
      float A0 = 0.f, A1 = 0.f, A2 = 0.f, Ay0 = 0.f, Ay1 = 0.f, Ayy0 = 0.f;
      const float dx0 = (float)(ua - ulo) - mxr;
      float dy = (float)(va - vlo) - myr;
      const float *grow = &gs[va - v0][ua - u0];
      const int nu = ubnd - ua;
#pragma unroll 1
      for (int v = va; v <= vbnd; ++v, dy += 1.f, grow += T + 1) {
        const float t1 = nb2 * dy, t2 = nc * dy * dy;
        float dx = dx0, T0 = 0.f, T1 = 0.f, T2 = 0.f;
        const float *gp = grow;
#pragma unroll 1
        for (int uu = 0; uu <= nu; ++uu, dx += 1.f, ++gp) {
          const float ge = *gp * ex2(fmaf(fmaf(na, dx, t1), dx, t2));
          const float gdx = ge * dx;
          T0 += ge;
          T1 += gdx;
          T2 = fmaf(gdx, dx, T2);
        }
        A0 += T0;
        A1 += T1;
        A2 += T2;
        Ay0 = fmaf(dy, T0, Ay0);
        Ay1 = fmaf(dy, T1, Ay1);
        Ayy0 = fmaf(dy * dy, T0, Ayy0);
      }
      const float La = A0;
      const float Lmx = amp * fmaf(a, A1, b * Ay0), Lmy = amp * fmaf(b, A1, cc * Ay0);
      float Lpa = amp * A2, Lpb = amp * Ay1, Lpc = amp * Ayy0;
      Lpa *= -0.5f; Lpb = -Lpb; Lpc *= -0.5f;
      // G_Sigma_hat (pixel units) = -K Gk K - 1/2 L_amp amp K, Gk = [[Lpa, Lpb/2],[Lpb/2, Lpc]]
      const float g01 = 0.5f * Lpb;
      const float KG00 = a * Lpa + b * g01, KG01 = a * g01 + b * Lpc;
      const float KG10 = b * Lpa + cc * g01, KG11 = b * g01 + cc * Lpc;
      const float hl = 0.5f * La * amp;
      float G00 = -(KG00 * a + KG01 * b) - hl * a;
      float G01 = -(KG00 * b + KG01 * cc) - hl * b;
      float G11 = -(KG10 * b + KG11 * cc) - hl * cc;
      G00 *= inv_px2; G01 *= inv_px2; G11 *= inv_px2;   // -> Angstrom units
      const float lmx = Lmx * inv_px, lmy = Lmy * inv_px;
      const float rho = mean_rho[id].w;
      float4 o0, o1, o2;
      o0.x = La * (amp / rho);
      o0.y = lmx * W0[0] + lmy * W1[0];
      o0.z = lmx * W0[1] + lmy * W1[1];
      o0.w = lmx * W0[2] + lmy * W1[2];
      // G_Sigma_kl = sum_ab W[a][k] G[a][b] W[b][l]
      float M[3][3];
  #pragma unroll
      for (int kk = 0; kk < 3; ++kk)
  #pragma unroll
        for (int ll = kk; ll < 3; ++ll)
          M[kk][ll] = W0[kk] * (G00 * W0[ll] + G01 * W1[ll]) + W1[kk] * (G01 * W0[ll] + G11 * W1[ll]);
      o1 = make_float4(M[0][0], M[0][1], M[0][2], M[1][1]);
      o2 = make_float4(M[1][2], M[2][2], 0.f, 0.f);
      float4 *dst = acc + 3 * (size_t)id;
      red_add_v4(dst, o0);
      red_add_v4(dst + 1, o1);
      red_add_v4(dst + 2, o2);
    }
    __syncthreads();
  }
}

}  // namespace

void launch_render_fwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids, float *proj,
                       cudaStream_t s, int &launches) {
  dim3 grid(c.NT, B);
  if (c.T == 16) k_render_fwd<16><<<grid, kFwdWarps * 32, 0, s>>>(c, rec, base, ids, proj);
  else k_render_fwd<8><<<grid, kFwdWarps * 32, 0, s>>>(c, rec, base, ids, proj);
  ++launches;
}

void launch_render_bwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids,
                       const float *dldi, const float4 *mean_rho, const float *rot, float4 *acc, cudaStream_t s,
                       int &launches) {
  dim3 grid(c.NT, B);
  if (c.T == 16) k_render_bwd<16><<<grid, kBwdThreads, 0, s>>>(c, rec, base, ids, dldi, mean_rho, rot, acc);
  else k_render_bwd<8><<<grid, kBwdThreads, 0, s>>>(c, rec, base, ids, dldi, mean_rho, rot, acc);
  ++launches;
}

}  // namespace gem
