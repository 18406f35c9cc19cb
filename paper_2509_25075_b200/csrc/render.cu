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


// Row-owner forward.  Each warp takes batches of 32 list entries strided over the
// tile's list (batch j -> warp j % kFwdWarps) and stages them in smem.  Lane l owns tile
// row q = l % T of accumulator copy l / T (32/T private copies per warp), and
// walks the row segments AABB_k ∩ row q of the batch's entries of its copy
// (entry k -> copy k % (32/T)) in ascending k: for one segment it evaluates
// amp exp(-Q/2) along the row, two columns per iteration with packed fp32
// (FFMA2).  All lanes of a round work on distinct (copy, row) accumulators, so
// there are no write conflicts and no atomics; the per-warp copies are summed in
// a fixed order at the end (bitwise deterministic).  Lane utilisation is the
// fraction of rows with a segment in the round times mean/max segment width.
constexpr int kFwdWarps = 4;

template <int T>
__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(CfgDev c, const SplatRec *__restrict__ rec,
                                                                const int *__restrict__ base,
                                                                const int *__restrict__ ids,
                                                                float *__restrict__ proj) {
  constexpr int S = T + 1;                    // accumulator row stride (floats)
  constexpr int NCP = 32 / T;                 // accumulator copies per warp (one lane per row each)
  constexpr int COPY = T * S;
  __shared__ float acc[kFwdWarps][NCP * COPY];
  __shared__ float4 st0[kFwdWarps][32];       // (bu0 - mx', my', na, nb2)  tile-local, pre-scaled conic
  __shared__ float4 st1[kFwdWarps][32];       // (nc, amp, bu0 | w << 8, -)
  const int t = blockIdx.x, i = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int q = lane % T, cp = lane / T;
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
  for (int k = lane; k < NCP * COPY; k += 32) acc[w][k] = 0.f;
  const SplatRec *reci = rec + (size_t)i * c.N;
  const float nh = -0.5f * kLog2e;
  const uint32_t rowb = smem_u32(&acc[w][cp * COPY + q * S]);
  const unsigned csel = (NCP == 2 ? 0x55555555u : (NCP == 4 ? 0x11111111u : 0x01010101u)) << cp;
  const float qf = (float)q;
  __syncwarp();
  // Batch j (j = 0 .. nbat-1, warp j % kFwdWarps) holds entries s + j + nbat * l, l = 0..31:
  // strided over the whole (spatially ordered) list, so a batch's boxes spread over all
  // rows of the tile and the per-row segment counts stay balanced across lanes.
  const int nlist = e - s, nbat = (nlist + 31) >> 5;
  int j = w;
  SplatRec nr;
  if (j < nbat && j + nbat * lane < nlist) nr = reci[ids[s + j + nbat * lane]];
  for (; j < nbat; j += kFwdWarps) {
    const bool have = j + nbat * lane < nlist;
    const SplatRec r = nr;
    const int jn = j + kFwdWarps;
    if (jn < nbat && jn + nbat * lane < nlist) nr = reci[ids[s + jn + nbat * lane]];
    int bv0 = T, bv1 = -1;
    if (have) {
      const int ub = __float_as_int(r.f1.z), vb = __float_as_int(r.f1.w);
      const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
      const int bu0 = max(ulo - u0, 0), wd = min(uhi - u0, T - 1) - bu0 + 1;
      bv0 = max(vlo - v0, 0);
      bv1 = min(vhi - v0, T - 1);
      const float mx = (float)(ulo - u0) + r.f0.x, my = (float)(vlo - v0) + r.f0.y;
      st0[w][lane] = make_float4((float)bu0 - mx, my, nh * r.f0.z, 2.f * nh * r.f0.w);
      st1[w][lane] = make_float4(nh * r.f1.x, r.f1.y, __int_as_float(bu0 | (wd << 8)), 0.f);
    }
    unsigned mine = 0;   // entries of this batch whose box covers my row, of my copy
#pragma unroll
    for (int rr = 0; rr < T; ++rr) {
      const unsigned m = __ballot_sync(0xffffffffu, bv0 <= rr && rr <= bv1);
      if (rr == q) mine = m;
    }
    mine &= csel;
    __syncwarp();
#pragma unroll 1
    while (__any_sync(0xffffffffu, mine != 0)) {
      int wd = 0;
      float4 E0 = make_float4(0.f, 0.f, 0.f, 0.f), E1 = E0;
      if (mine) {
        const int k = __ffs(mine) - 1;
        mine &= mine - 1;
        E0 = st0[w][k];
        E1 = st1[w][k];
        wd = __float_as_int(E1.z) >> 8;
      }
      const int wmax = __reduce_max_sync(0xffffffffu, wd);
      const float dy = qf - E0.y;
      const float t1 = E0.w * dy, t2 = E1.x * dy * dy;
      const float2 na2 = make_float2(E0.z, E0.z), t12 = make_float2(t1, t1), t22 = make_float2(t2, t2);
      float2 dx = make_float2(E0.x, E0.x + 1.f);
      const uint32_t a0 = rowb + 4u * (uint32_t)(__float_as_int(E1.z) & 0xff);
      const float amp = E1.y;
#pragma unroll 1
      for (int cc = 0; cc < wmax; cc += 2) {
        const float2 arg = __ffma2_rn(__ffma2_rn(na2, dx, t12), dx, t22);
        const float ea = ex2(arg.x), eb = ex2(arg.y);
        const uint32_t a = a0 + 4u * (uint32_t)cc;
        if (cc < wd) sts_f32(a, fmaf(amp, ea, lds_f32(a)));
        if (cc + 1 < wd) sts_f32(a + 4u, fmaf(amp, eb, lds_f32(a + 4u)));
        dx = __fadd2_rn(dx, make_float2(2.f, 2.f));
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int pp = tid; pp < T * T; pp += kFwdWarps * 32) {
    const int pu = pp % T, pv = pp / T;
    float sum = 0.f;
#pragma unroll
    for (int ww = 0; ww < kFwdWarps; ++ww)
#pragma unroll
      for (int k = 0; k < NCP; ++k) sum += acc[ww][k * COPY + pv * S + pu];
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
