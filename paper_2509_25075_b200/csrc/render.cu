// render.cu — a5 forward evaluate/project and a7 backward scatter over the
// per-tile lists.
//
// Forward (Eq. 6 with the Eq. 8 selection):
//   I_hat(u,v) = sum_{j in list(tile(u,v)), (u,v) in AABB_j} amp_j exp(-Q_j/2),
//   Q = a dx^2 + 2 b dx dy + c dy^2 (pixel units).
// One CTA per (particle, T x T tile).  List entries are staged into shared
// memory (gathering the 32-B splat records by id); each warp owns an 8x4
// pixel sub-tile, ballot-compacts the entries whose AABB meets it, and
// accumulates in fp32 per pixel in ascending list (= ascending j) order, so the
// forward is bitwise deterministic.
//
// Backward ("gradient computation restricted to the Gaussians contributing to
// each pixel"): one thread per list entry loops over the
// pixels of AABB_j inside the tile (dL/dI_hat staged in smem), reduces the six
// partials (L_amp, L_mx, L_my, L_a, L_b, L_c) in registers, transforms them to
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

__device__ __forceinline__ int clamp_i(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <int T>
__global__ void __launch_bounds__(T *T) k_render_fwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                      const int *__restrict__ base, const int *__restrict__ ids,
                                                      float *__restrict__ proj) {
  constexpr int NTH = T * T;
  __shared__ float4 e0[NTH];   // (mx, my) tile-local centre, (A, B) prescaled conic
  __shared__ float2 e1[NTH];   // (C prescaled, amp)
  __shared__ int4 eb[NTH];     // tile-local box (ulo, uhi, vlo, vhi), clamped to [-1, T]
  const int t = blockIdx.x, i = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int u0 = (t % c.nt) * T, v0 = (t / c.nt) * T;
  const int su0 = (T == 16) ? (w & 1) * 8 : 0, sv0 = (T == 16) ? (w >> 1) * 4 : w * 4;
  const int pu = su0 + (lane & 7), pv = sv0 + (lane >> 3);
  const float puf = (float)pu, pvf = (float)pv;
  const size_t hidx = ((size_t)i * c.NT + t) * c.C;
  int s = base[hidx], e = base[hidx + c.C];
  if ((int64_t)e > c.cap) e = (int)c.cap;
  if ((int64_t)s > c.cap) s = (int)c.cap;
  const SplatRec *reci = rec + (size_t)i * c.N;
  float acc = 0.f;
  const float kA = -0.5f * kLog2e, kB = -kLog2e;
  for (int cs = s; cs < e; cs += NTH) {
    const int n = min(NTH, e - cs);
    __syncthreads();
    if (tid < n) {
      const int id = ids[cs + tid];
      const SplatRec r = reci[id];
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      e0[tid] = make_float4((float)(ulo - u0) + r.f0.x, (float)(vlo - v0) + r.f0.y, kA * r.f0.z, kB * r.f0.w);
      e1[tid] = make_float2(kA * r.f1.x, r.f1.y);
      eb[tid] = make_int4(clamp_i(ulo - u0, -1, T), clamp_i(uhi - u0, -1, T), clamp_i(vlo - v0, -1, T),
                          clamp_i(vhi - v0, -1, T));
    }
    __syncthreads();
    for (int g = 0; g < n; g += 32) {
      const int k = g + lane;
      bool hit = false;
      if (k < n) {
        const int4 b = eb[k];
        hit = b.x <= su0 + 7 && b.y >= su0 && b.z <= sv0 + 3 && b.w >= sv0;
      }
      unsigned m = __ballot_sync(0xffffffffu, hit);
      while (m) {
        const int kk = g + __ffs(m) - 1;
        m &= m - 1;
        const float4 E = e0[kk];
        const float2 F = e1[kk];
        const int4 b = eb[kk];
        const bool inside = (unsigned)(pu - b.x) <= (unsigned)(b.y - b.x) && (unsigned)(pv - b.z) <= (unsigned)(b.w - b.z);
        const float dx = puf - E.x, dy = pvf - E.y;
        const float q = fmaf(fmaf(E.z, dx, E.w * dy), dx, F.x * dy * dy);
        const float ev = ex2(q);
        if (inside) acc = fmaf(F.y, ev, acc);
      }
    }
  }
  const int u = u0 + pu, v = v0 + pv;
  if (u < c.D && v < c.D) proj[((size_t)i * c.D + v) * c.D + u] = acc;
}

template <int T>
__global__ void __launch_bounds__(T *T) k_render_bwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                      const int *__restrict__ base, const int *__restrict__ ids,
                                                      const float *__restrict__ dldi,
                                                      const float4 *__restrict__ mean_rho, const float *__restrict__ rot,
                                                      float4 *__restrict__ acc) {
  constexpr int NTH = T * T;
  __shared__ float gs[T][T + 1];
  const int t = blockIdx.x, i = blockIdx.y, tid = threadIdx.x;
  const int u0 = (t % c.nt) * T, v0 = (t / c.nt) * T;
  {
    const int pu = tid % T, pv = tid / T, u = u0 + pu, v = v0 + pv;
    gs[pv][pu] = (u < c.D && v < c.D) ? dldi[((size_t)i * c.D + v) * c.D + u] : 0.f;
  }
  const size_t hidx = ((size_t)i * c.NT + t) * c.C;
  int s = base[hidx], e = base[hidx + c.C];
  if ((int64_t)e > c.cap) e = (int)c.cap;
  if ((int64_t)s > c.cap) s = (int)c.cap;
  // W = P^T: W[r][k] = P[3k + r]; only rows 0 and 1 of W are needed.
  float W0[3], W1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    W0[k] = rot[9 * i + 3 * k];
    W1[k] = rot[9 * i + 3 * k + 1];
  }
  const float inv_px = 1.f / c.px, inv_px2 = inv_px * inv_px;
  const float nh = -0.5f * kLog2e;
  __syncthreads();
  const SplatRec *reci = rec + (size_t)i * c.N;
  for (int k = s + tid; k < e; k += NTH) {
    const int id = ids[k];
    const SplatRec r = reci[id];
    const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
    const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
    const float mxr = r.f0.x, myr = r.f0.y, a = r.f0.z, b = r.f0.w, cc = r.f1.x, amp = r.f1.y;
    const int ua = max(ulo, u0), ubnd = min(uhi, u0 + T - 1), va = max(vlo, v0), vbnd = min(vhi, v0 + T - 1);
    float La = 0.f, Lmx = 0.f, Lmy = 0.f, Lpa = 0.f, Lpb = 0.f, Lpc = 0.f;
    for (int v = va; v <= vbnd; ++v) {
      const float dy = (float)(v - vlo) - myr;
      for (int u = ua; u <= ubnd; ++u) {
        const float dx = (float)(u - ulo) - mxr;
        const float adbd = fmaf(a, dx, b * dy), bdcd = fmaf(b, dx, cc * dy);
        const float Q = fmaf(adbd, dx, bdcd * dy);
        const float ev = ex2(nh * Q);
        const float ge = gs[v - v0][u - u0] * ev;
        const float h = ge * amp;
        La += ge;
        Lmx = fmaf(h, adbd, Lmx);
        Lmy = fmaf(h, bdcd, Lmy);
        Lpa = fmaf(h, dx * dx, Lpa);
        Lpb = fmaf(h, dx * dy, Lpb);
        Lpc = fmaf(h, dy * dy, Lpc);
      }
    }
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
}

}  // namespace

void launch_render_fwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids, float *proj,
                       cudaStream_t s, int &launches) {
  dim3 grid(c.NT, B);
  if (c.T == 16) k_render_fwd<16><<<grid, 256, 0, s>>>(c, rec, base, ids, proj);
  else k_render_fwd<8><<<grid, 64, 0, s>>>(c, rec, base, ids, proj);
  ++launches;
}

void launch_render_bwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids,
                       const float *dldi, const float4 *mean_rho, const float *rot, float4 *acc, cudaStream_t s,
                       int &launches) {
  dim3 grid(c.NT, B);
  if (c.T == 16) k_render_bwd<16><<<grid, 256, 0, s>>>(c, rec, base, ids, dldi, mean_rho, rot, acc);
  else k_render_bwd<8><<<grid, 64, 0, s>>>(c, rec, base, ids, dldi, mean_rho, rot, acc);
  ++launches;
}

}  // namespace gem
