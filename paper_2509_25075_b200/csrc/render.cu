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

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
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

// Entries are processed in pairs with packed fp32 (FFMA2 / FADD2 / FMUL2):
// the staging layout stores each field of a pair as one float2 so a pass needs
// no register shuffling.

template <int T>
__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                                const int *__restrict__ base,
                                                                const int *__restrict__ ids,
                                                                float *__restrict__ proj) {
  constexpr int S = T + 8;                     // accumulator row stride (floats)
  __shared__ float acc[kFwdWarps][T * S];
  __shared__ float2 sf[kFwdWarps][8][17];      // [field][pair] = (entry a, entry b): mx'+1/2, my', A, B, C, amp, 1/w, -w
  __shared__ int4 si[kFwdWarps][17];           // (npix_a, npix_b, byte offset a, byte offset b)
  __shared__ int2 ssw[kFwdWarps][17];          // (4 (S - w_a), 4 (S - w_b)): byte stride correction per row
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
  const float M = 12582912.f;                   // 1.5 * 2^23: x + M rounds x to an integer
  const uint32_t accb = smem_u32(&acc[w][lane]);
  float2(*F)[17] = sf[w];
  __syncwarp();
  // software pipeline: the next batch's record is loaded while this batch renders
  int b0 = s + 32 * w;
  SplatRec nr;
  if (b0 + lane < e) nr = reci[ids[b0 + lane]];
  for (; b0 < e; b0 += 32 * kFwdWarps) {
    const int n = min(32, e - b0);
    const SplatRec r = nr;
    const bool have = lane < n;
    const int nb = b0 + 32 * kFwdWarps + lane;
    if (nb < e) nr = reci[ids[nb]];
    int npix = 0, boff = 0, bsw = 0;
    float f[8];
    if (have) {
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      const int bu0 = max(ulo - u0, 0), bv0 = max(vlo - v0, 0);
      const int wd = min(uhi - u0, T - 1) - bu0 + 1;
      npix = wd * (min(vhi - v0, T - 1) - bv0 + 1);
      bsw = 4 * (S - wd);
      // byte offset of the box corner, pre-biased so that offset + bits(xm) * bsw
      // addresses row q = bits(xm) - bits(M) (wrap-around arithmetic)
      boff = 4 * (bv0 * S + bu0) - 0x4B400000 * bsw;
      f[0] = (float)(ulo - u0 - bu0) + r.f0.x + 0.5f;   // mx' + 1/2 (pixel index + 1/2 is enumerated)
      f[1] = (float)(vlo - v0 - bv0) + r.f0.y;          // my'
      f[2] = kA * r.f0.z;
      f[3] = kB * r.f0.w;
      f[4] = kA * r.f1.x;
      f[5] = r.f1.y;
      f[6] = 1.0f / (float)wd;
      f[7] = -(float)wd;
    }
    // stage single-pass entries (npix <= 32) first so paired entries need equal passes
    const unsigned big = __ballot_sync(0xffffffffu, have && npix > 32);
    const unsigned small = __ballot_sync(0xffffffffu, have && npix <= 32);
    const unsigned lt = (1u << lane) - 1u;
    if (have) {
      const int slot = npix > 32 ? __popc(small) + __popc(big & lt) : __popc(small & lt);
      const int pr = slot >> 1, ab = slot & 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) reinterpret_cast<float *>(&F[q][pr])[ab] = f[q];
      int *sip = (int *)&si[w][pr];
      sip[ab] = npix;
      sip[2 + ab] = boff;
      reinterpret_cast<int *>(&ssw[w][pr])[ab] = bsw;
    }
    if (lane == 0 && (n & 1)) {   // dummy partner for an odd count
      int *sip = (int *)&si[w][n >> 1];
      sip[1] = 0;
      sip[3] = 0;
      reinterpret_cast<int *>(&ssw[w][n >> 1])[1] = 0;
    }
    __syncwarp();
    const int npairs = (n + 1) >> 1;
    const float laneh = (float)lane + 0.5f;
    for (int pr = 0; pr < npairs; ++pr) {   // two entries per pass, packed fp32 (FFMA2)
      const int4 I = si[w][pr];
      const int2 SW = ssw[w][pr];
      const float2 mx = F[0][pr], my = F[1][pr], A2 = F[2][pr], B2 = F[3][pr];
      const float2 C2 = F[4][pr], amp = F[5][pr], iw = F[6][pr], nw = F[7][pr];
      const int npm = max(I.x, I.y);
      float2 pfh = make_float2(laneh, laneh);
      float2 dxo = __fadd2_rn(pfh, make_float2(-mx.x, -mx.y));
      uint32_t pa = accb + (uint32_t)I.z, pb = accb + (uint32_t)I.w;
      int p = lane;
#pragma unroll 1
      do {
        const float2 xm = __fadd2_rn(__ffma2_rn(pfh, iw, make_float2(-0.5f, -0.5f)), make_float2(M, M));
        const float2 qf = __fadd2_rn(xm, make_float2(-M, -M));
        const float2 dx = __ffma2_rn(qf, nw, dxo);
        const float2 dy = __fadd2_rn(qf, make_float2(-my.x, -my.y));
        const float2 q = __ffma2_rn(__ffma2_rn(A2, dx, __fmul2_rn(B2, dy)), dx, __fmul2_rn(__fmul2_rn(C2, dy), dy));
        const float ea = ex2(q.x), eb = ex2(q.y);
        if (p < I.x) {
          const uint32_t a = pa + (uint32_t)__float_as_int(xm.x) * (uint32_t)SW.x;
          sts_f32(a, fmaf(amp.x, ea, lds_f32(a)));
        }
        if (p < I.y) {
          const uint32_t b = pb + (uint32_t)__float_as_int(xm.y) * (uint32_t)SW.y;
          sts_f32(b, fmaf(amp.y, eb, lds_f32(b)));
        }
        p += 32;
        pa += 128;
        pb += 128;
        pfh = __fadd2_rn(pfh, make_float2(32.f, 32.f));
        dxo = __fadd2_rn(dxo, make_float2(32.f, 32.f));
      } while (p - lane < npm);
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
// box ∩ tile, so the tile's whole list (up to kBwdMax entries per round) is first
// counting-sorted in smem by the class (min(h,8), min(ceil(w/2),4)) of its box:
// consecutive entries — one warp's — then have near-equal loop trip counts.
constexpr int kBwdThreads = 256;
constexpr int kBwdKeys = 32;
constexpr int kBwdMax = 4096;

template <int T>
__global__ void __launch_bounds__(kBwdThreads) k_render_bwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                             const uint2 *__restrict__ box,
                                                             const int *__restrict__ base, const int *__restrict__ ids,
                                                             const float *__restrict__ dldi,
                                                             const float4 *__restrict__ mean_rho,
                                                             const float *__restrict__ rot, float4 *__restrict__ acc) {
  __shared__ float gs[T + 1][T + 1];   // one spare row: the paired loop may read one past a row
  __shared__ unsigned char skey[kBwdMax];
  __shared__ unsigned short order[kBwdMax];
  __shared__ int hist[kBwdKeys];
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
  const uint2 *boxi = box + (size_t)i * c.N;
  for (int cs = s; cs < e; cs += kBwdMax) {
    const int n = min(kBwdMax, e - cs);
    if (tid < kBwdKeys) hist[tid] = 0;
    __syncthreads();
    for (int k = tid; k < n; k += kBwdThreads) {
      const uint2 b = boxi[ids[cs + k]];
      const int wd = min((int)(b.x >> 16), u0 + T - 1) - max((int)(b.x & 0xffff), u0) + 1;
      const int ht = min((int)(b.y >> 16), v0 + T - 1) - max((int)(b.y & 0xffff), v0) + 1;
      const int key = (min(ht, 8) - 1) * 4 + min((wd + 1) >> 1, 4) - 1;
      skey[k] = (unsigned char)key;
      atomicAdd(&hist[key], 1);
    }
    __syncthreads();
    if (tid < 32) {   // exclusive scan of the 32 class counts
      const int hv = hist[tid];
      int incl = hv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, d);
        if (tid >= d) incl += y;
      }
      hist[tid] = incl - hv;
    }
    __syncthreads();
    for (int k = tid; k < n; k += kBwdThreads) order[atomicAdd(&hist[skey[k]], 1)] = (unsigned short)k;
    __syncthreads();
    for (int kk = tid; kk < n; kk += kBwdThreads) {
      const int id = ids[cs + order[kk]];
      const SplatRec r = reci[id];
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      const float mxr = r.f0.x, myr = r.f0.y, a = r.f0.z, b = r.f0.w, cc = r.f1.x, amp = r.f1.y;
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
    const int nu = ubnd - ua;                 // row length - 1
    const float2 na2 = make_float2(na, na), two = make_float2(2.f, 2.f);
#pragma unroll 1
    for (int v = va; v <= vbnd; ++v, dy += 1.f, grow += T + 1) {
      const float t1 = nb2 * dy, t2 = nc * dy * dy;
      const float2 t12 = make_float2(t1, t1), t22 = make_float2(t2, t2);
      float2 dx = make_float2(dx0, dx0 + 1.f);
      float2 T0 = make_float2(0.f, 0.f), T1 = T0, T2 = T0;
      const float *gp = grow;
#pragma unroll 1
      for (int uu = 0; uu <= nu; uu += 2, gp += 2) {   // two pixels per iteration (FFMA2)
        const float2 arg = __ffma2_rn(__ffma2_rn(na2, dx, t12), dx, t22);
        const float2 g2 = make_float2(gp[0], uu < nu ? gp[1] : 0.f);
        const float2 ge = __fmul2_rn(g2, make_float2(ex2(arg.x), ex2(arg.y)));
        const float2 gdx = __fmul2_rn(ge, dx);
        T0 = __fadd2_rn(T0, ge);
        T1 = __fadd2_rn(T1, gdx);
        T2 = __ffma2_rn(gdx, dx, T2);
        dx = __fadd2_rn(dx, two);
      }
      const float s0 = T0.x + T0.y, s1 = T1.x + T1.y, s2 = T2.x + T2.y;
      A0 += s0;
      A1 += s1;
      A2 += s2;
      Ay0 = fmaf(dy, s0, Ay0);
      Ay1 = fmaf(dy, s1, Ay1);
      Ayy0 = fmaf(dy * dy, s0, Ayy0);
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

void launch_render_bwd(const CfgDev &c, int B, const SplatRec *rec, const uint2 *box, const int *base, const int *ids,
                       const float *dldi, const float4 *mean_rho, const float *rot, float4 *acc, cudaStream_t s,
                       int &launches) {
  dim3 grid(c.NT, B);
  if (c.T == 16) k_render_bwd<16><<<grid, kBwdThreads, 0, s>>>(c, rec, box, base, ids, dldi, mean_rho, rot, acc);
  else k_render_bwd<8><<<grid, kBwdThreads, 0, s>>>(c, rec, box, base, ids, dldi, mean_rho, rot, acc);
  ++launches;
}

}  // namespace gem
