// render.cu — a5 forward evaluate/project, a7 backward over the per-tile lists, and the
// per-Gaussian reduction of the backward's image-space partials.
//
// Forward (Eq. 6 with the Eq. 8 selection):
//   I_hat(u,v) = sum_{j in list(tile(u,v)), (u,v) in AABB_j} amp_j exp(-Q_j/2),
//   Q = a dx^2 + 2 b dx dy + c dy^2 (pixel units).
// Backward: per (particle, Gaussian), the moments of dL/dI_hat * exp(-Q/2)
// over AABB_ij give the six 2D partials; see k_render_bwd and k_bwd_reduce.
// Both use multiplicative recurrences instead of one exp per pixel (see the forward's comment).
#include "gem_internal.cuh"

#ifndef GEM_FWD_IDCS
#define GEM_FWD_IDCS 0
#endif
#if GEM_FWD_IDCS   // the tile lists' ids stream through once: evict-first loads
#define LDID(p_) __ldcs(p_)
#else
#define LDID(p_) (*(p_))
#endif

namespace gem {
namespace {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Forward.  Recurrences: in pixel units, with f = log2 of the kernel, f(dx, dy) = na dx^2 +
// nb2 dx dy + nc dy^2 (na = -log2(e) a / 2, nb2 = -log2(e) b, nc = -log2(e) c / 2), f is quadratic
// along a row and along a column, so the values on the pixel grid obey exact multiplicative
// recurrences:
//   along a row                  e_{k+1} = e_k R_k,  R_{k+1} = R_k S,  S  = 2^{2 na}
//   down the box's first column  e_{r+1} = e_r V_r,  V_{r+1} = V_r W,  W  = 2^{2 nc}
//   and the row ratio            R(r+1) = R(r) Kb,                     Kb = 2^{nb2}.
// One (Gaussian x tile) entry costs 6 exps plus two multiplies per pixel instead of one exp per
// pixel (MUFU: 16/clk/SM vs 128 FMA lanes/clk/SM; tools/microbench.cu).  Rounding: a pixel k
// columns and r rows from the box corner carries ~(k^2 + r^2)/4 ulp relative to its own value.
// Safety: f <= 0, so values never overflow; the recurrences stay exact only while their factors
// are normal numbers, so an entry whose first-column values fall below 2^-100 amp (needle-like
// Gaussians at far AABB corners), whose corner row ratio is below 2^-120, or whose W, Kb leave the
// normal range is evaluated directly (exp per pixel).  The amplitude's sign only multiplies
// (negative densities take the fast path too).
constexpr int kFwdWarps = 2;       // warps per CTA (independent)
constexpr int kCH = 64;            // list entries staged per chunk per warp

__device__ __forceinline__ int next_item(int *ticket, int lane) {
  int item = 0;
  if (lane == 0) item = atomicAdd(ticket, 1);
  return __shfl_sync(0xffffffffu, item, 0);
}
// the last warp out resets the two ticket words for the next launch on this stream
__device__ __forceinline__ void retire(int *ticket, int lane) {
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)(gridDim.x * (blockDim.x >> 5)) - 1) {
      ticket[0] = 0;
      ticket[1] = 0;
    }
  }
}

// Forward kernel for 16 x 16 tiles (8 x 8 tiles use k_render_fwd_le below).  Register
// accumulators: lane L owns row pair p = L / NCP of the tile (NCP = 32 / NP lanes per pair)
// and keeps a private copy of that pair-row, T columns x 2 rows,
// in registers.  Per chunk of <= kCH entries, each lane takes one entry (records prefetched one
// 32-entry group ahead, ids two), stores its per-entry constants once in shared memory and
// appends the entry's index to the bin of every row pair its box covers (ballots, in list
// order: deterministic).  Then the NCP lanes of pair p take the segments of bin p round-robin:
// a lane evaluates its segment's start values directly (e and the row ratio R at the first
// column of rows 2p and 2p+1: four exps) and renders the segment with a fully unrolled,
// predicated T-column recurrence into its registers: no shared-memory read-modify-write and no
// divergence from box widths.  At the end the NCP copies of each pair-row are summed by a fixed
// butterfly of shuffles (bitwise deterministic).
template <int T>
struct FwdSmem {
  static constexpr int NP = T / 2;
  float4 eA[kCH];                // (my, nb2, nc, amp)           tile-local pixel units, log2 scale
  float4 eB[kCH];                // (Fx, Gx, D0, S = 2^{2 na})   f(dx0, dy) = Fx + dy (Gx + nc dy)
  float2 eC[kCH];                // (na, bits)  bits = cu0 | cu1 << 8 | cv0 << 16 | cv1 << 24 | slow << 31
  float thr[kCH];                // MK: per-pixel keep threshold on |amp e|
  unsigned char bin[NP][kCH];    // entry indices per row pair
};

// Per-pixel selection variants (reading L26; GEM_FLAG_ELLIPSE / _PIXEL_TAU): a
// pixel inside the AABB is kept only if Q <= k^2 and/or |amp| e >= tau, i.e. |amp e| >= thr with
// thr = max(ELLIPSE ? |amp| exp(-k^2/2) : 0, PIXEL_TAU ? tau : 0), tested on the value the
// recurrence produces (forward) or on e >= thr / |amp| (backward).
__device__ __forceinline__ float keep_thr(const CfgDev &c, float amp, float eK) {
  float t = (c.flags & GEM_FLAG_ELLIPSE) ? fabsf(amp) * eK : 0.f;
  if (c.flags & GEM_FLAG_PIXEL_TAU) t = fmaxf(t, c.tau);
  return t;
}

template <int T, bool MK>
__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(CfgDev c, int B, const SplatRec *__restrict__ rec,
                                                                const int *__restrict__ base,
                                                                const int *__restrict__ ids,
                                                                float *__restrict__ proj, int *ticket) {
  using SM = FwdSmem<T>;
  constexpr int NP = T / 2, NCP = 32 / NP;
  constexpr float nh = -0.5f * kLog2e;
  const float eK = MK ? ex2(nh * c.k * c.k) : 0.f;
  extern __shared__ __align__(16) unsigned char fwd_dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SM &sm = reinterpret_cast<SM *>(fwd_dsm)[w];
  const unsigned lt = (1u << lane) - 1u;
  const int mp = lane / NCP, cp = lane % NCP;
  const float pyA = (float)(2 * mp);
  const int items = B * c.NT;
  // item pipeline: the next item's ticket and list bounds are fetched while the current item is
  // processed (hides the global atomic and the two dependent loads)
  auto bounds = [&](int it, int &s_, int &e_) {
    s_ = 0; e_ = 0;
    if (it < items) {
      s_ = base[it];   // base = lst here (list starts, see list_bounds' comment)
      e_ = base[it + 1];
    }
  };
  int nitem = next_item(ticket, lane), ns, ne;
  bounds(nitem, ns, ne);
  for (;;) {
    const int item = nitem;
    if (item >= items) break;
    int s = ns, e = ne;
    nitem = next_item(ticket, lane);
    bounds(nitem, ns, ne);
    const int i = item / c.NT, t = item - i * c.NT;
    const int u0 = (t % c.nt) * T, v0 = (t / c.nt) * T;
    if ((int64_t)e > c.cap) e = (int)c.cap;
    if ((int64_t)s > c.cap) s = (int)c.cap;
    float *out = proj + (size_t)i * c.D * c.D;
    if (s >= e) {   // empty tile: the projection is zero there
      for (int p = lane; p < T * T; p += 32) {
        const int u = u0 + p % T, v = v0 + p / T;
        if (u < c.D && v < c.D) out[(size_t)v * c.D + u] = 0.f;
      }
      continue;
    }
    float2 acc[T];
#pragma unroll
    for (int k = 0; k < T; ++k) acc[k] = make_float2(0.f, 0.f);
    const SplatRec *reci = rec + (size_t)i * c.N;
    // software pipeline over 32-entry groups: ids two groups ahead, records one group ahead
    const int nall = e - s;
    int id1 = lane < nall ? ids[s + lane] : 0;
    int id2 = 32 + lane < nall ? ids[s + 32 + lane] : 0;
    SplatRec nxt;
    if (lane < nall) nxt = reci[id1];
    int blen = 0;   // length of bin mp in the current chunk (lanes of pair pp hold bin pp's length)
    for (int g0 = 0; g0 < nall; g0 += 32) {
      const int q = g0 + lane, qc = g0 % kCH + lane;   // list position, index within the chunk
      const SplatRec rr = nxt;
      if (q + 32 < nall) nxt = reci[id2];
      if (q + 64 < nall) id2 = LDID(ids + s + q + 64);
      int pr0 = NP, pr1 = -1;
      if (q < nall) {
        const int ub = __float_as_int(rr.f1.z), vb = __float_as_int(rr.f1.w);
        const int ulo = (ub & 0xffff) - u0, uhi = (ub >> 16) - u0, vlo = (vb & 0xffff) - v0, vhi = (vb >> 16) - v0;
        const int cu0 = max(ulo, 0), cu1 = min(uhi, T - 1), cv0 = max(vlo, 0), cv1 = min(vhi, T - 1);
        pr0 = cv0 >> 1;
        pr1 = cv1 >> 1;
        const float na = nh * rr.f0.z, nb2 = 2.f * nh * rr.f0.w, nc = nh * rr.f1.x;
        const float mx = (float)ulo + rr.f0.x, my = (float)vlo + rr.f0.y;
        const float dx0 = (float)cu0 - mx;
        const float Fx = na * dx0 * dx0, Gx = nb2 * dx0, D0 = na * fmaf(2.f, dx0, 1.f);
        // the recurrence needs its factors normal: first-column values and the row ratio at the
        // covered rows (f concave, ratio linear in dy: check the end rows)
        const float d0 = (float)cv0 - my, d1 = (float)cv1 - my;
        const float f0 = fmaf(d0, fmaf(nc, d0, Gx), Fx), f1 = fmaf(d1, fmaf(nc, d1, Gx), Fx);
        const float r0 = fmaf(nb2, d0, D0), r1 = fmaf(nb2, d1, D0);
        const bool slow = !(fminf(f0, f1) >= -100.f && fminf(r0, r1) >= -120.f);
        sm.eA[qc] = make_float4(my, nb2, nc, rr.f1.y);
        sm.eB[qc] = make_float4(Fx, Gx, D0, ex2(2.f * na));
        sm.eC[qc] = make_float2(na, __int_as_float(cu0 | (cu1 << 8) | (cv0 << 16) | (cv1 << 24) |
                                                   (slow ? (int)0x80000000 : 0)));
        if (MK) sm.thr[qc] = keep_thr(c, rr.f1.y, eK);
      }
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const bool in = pr0 <= pp && pp <= pr1;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const int before = __shfl_sync(0xffffffffu, blen, pp * NCP);
        if (in) sm.bin[pp][before + __popc(bal & lt)] = (unsigned char)qc;
        if (mp == pp) blen += __popc(bal);
      }
      if ((g0 + 32) % kCH != 0 && g0 + 32 < nall) continue;   // the chunk's bins are not full yet
      __syncwarp();
      // render: lanes of pair mp take segments cp, cp + NCP, ... of bin mp
#pragma unroll 1
      for (int sg = cp; __any_sync(0xffffffffu, sg < blen); sg += NCP) {
        if (sg >= blen) continue;
        const int qe = sm.bin[mp][sg];
        const float4 A = sm.eA[qe], Bq = sm.eB[qe];
        const float2 Cq = sm.eC[qe];
        const int bits = __float_as_int(Cq.y);
        const int k0 = bits & 0xff, k1 = (bits >> 8) & 0xff, cv0 = (bits >> 16) & 0xff, cv1 = (bits >> 24) & 0x7f;
        const bool vA = 2 * mp >= cv0, vB = 2 * mp + 1 <= cv1;
        const float dyA = pyA - A.x, dyB = dyA + 1.f, nb2 = A.y, nc = A.z, amp = A.w;
        const float fA = fmaf(dyA, fmaf(nc, dyA, Bq.y), Bq.x), fB = fmaf(dyB, fmaf(nc, dyB, Bq.y), Bq.x);
        const float gA = fmaf(nb2, dyA, Bq.z), gB = gA + nb2;   // log2 R at the first column
        const float th = MK ? sm.thr[qe] : 0.f;
        if (bits >= 0) {
          float2 E2 = make_float2(vA ? amp * ex2(fA) : 0.f, vB ? amp * ex2(fB) : 0.f);
          float2 R2 = make_float2(vA ? ex2(gA) : 0.f, vB ? ex2(gB) : 0.f);
          const float2 S2 = make_float2(Bq.w, Bq.w);
#pragma unroll
          for (int k = 0; k < T; ++k) {
            if (k >= k0 && k <= k1) {
              if (MK) {
                acc[k].x += fabsf(E2.x) >= th ? E2.x : 0.f;
                acc[k].y += fabsf(E2.y) >= th ? E2.y : 0.f;
              } else {
                acc[k] = __fadd2_rn(acc[k], E2);
              }
              E2 = __fmul2_rn(E2, R2);
              R2 = __fmul2_rn(R2, S2);
            }
          }
        } else {   // direct evaluation: f = f0 + kk g0 + kk (kk - 1) na, kk = k - k0
          const float na = Cq.x;
#pragma unroll
          for (int k = 0; k < T; ++k) {
            if (k >= k0 && k <= k1) {
              const float kf = (float)(k - k0), kq = kf * (kf - 1.f) * na;
              if (MK) {
                const float xa = amp * ex2(fmaf(kf, gA, fA) + kq), xb = amp * ex2(fmaf(kf, gB, fB) + kq);
                if (vA && fabsf(xa) >= th) acc[k].x += xa;
                if (vB && fabsf(xb) >= th) acc[k].y += xb;
              } else {
                if (vA) acc[k].x = fmaf(amp, ex2(fmaf(kf, gA, fA) + kq), acc[k].x);
                if (vB) acc[k].y = fmaf(amp, ex2(fmaf(kf, gB, fB) + kq), acc[k].y);
              }
            }
          }
        }
      }
      blen = 0;
      __syncwarp();
    }
    // sum the NCP copies of each pair-row (fixed butterfly), lane cp writes columns cp, cp + NCP, ...
#pragma unroll
    for (int k = 0; k < T; ++k) {
#pragma unroll
      for (int d = 1; d < NCP; d <<= 1) {
        acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, d);
        acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, d);
      }
    }
    const int v = v0 + 2 * mp;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      if (k % NCP == cp) {
        const int u = u0 + k;
        if (u < c.D && v < c.D) out[(size_t)v * c.D + u] = acc[k].x;
        if (u < c.D && v + 1 < c.D) out[(size_t)(v + 1) * c.D + u] = acc[k].y;
      }
    }
  }
  retire(ticket, lane);
}

// Forward for 8x8 tiles, lane per entry.  Every lane keeps a private copy of the whole tile in
// registers (4 row pairs x 8 columns, packed fp32x2 = 64 floats) and renders whole list entries,
// lane l taking entries l, l + 32, ... of the tile (records prefetched one round ahead, ids two):
// no binning, no shared memory, no idle lanes except in a tile's last round.  An entry walks the
// row pairs its box covers (predicated, fully unrolled) with the recurrences of the forward
// comment extended down the column in pairs: with E2 = (e_r, e_r+1) at the first column,
//   E2 <- E2 (V_r^2 W, V_r^2 W^3),  (V_r^2 W, V_r^2 W^3) <- (.) W^4,  R2 <- R2 Kb^2  per row pair,
// so an entry costs 6 exps.  The 32 private copies are summed by a fixed reduce-scatter of
// shuffles (halving 64 -> 2 values per lane; lane L ends with row pair L / 8, column L % 8):
// bitwise deterministic.  The row-pair recurrence squares V, so entries with |log2 V| > 60 at
// an end row take the direct path too.
constexpr int kLeWarps = 2, kLeBatch = 4, kLePitch = 68;   // kLePitch: the reduction buffer's row pitch
#ifndef GEM_FWD_L2PF
#define GEM_FWD_L2PF 0
#endif

template <bool MK>
__global__ void __launch_bounds__(kLeWarps * 32, 8) k_render_fwd_le(CfgDev c, int B, const SplatRec *__restrict__ rec,
                                                                    const int *__restrict__ base,
                                                                    const int *__restrict__ ids,
                                                                    float *__restrict__ proj, int *ticket,
                                                                    int zero_empty) {
  constexpr int T = 8;
  constexpr float nh = -0.5f * kLog2e;
  __shared__ __align__(16) float le_smem[kLeWarps * 32 * kLePitch];
  const float eK = MK ? ex2(nh * c.k * c.k) : 0.f;
  const int lane = threadIdx.x & 31;
  const int items = B * c.NT;
  // items (particle, tile) are taken kLeBatch at a time from the ticket; the next item's list
  // bounds are fetched while the current one is rendered
  auto bounds = [&](int it, int &s_, int &e_) {
    s_ = 0; e_ = 0;
    if (it < items) {
      s_ = base[it];   // base = lst here: list (i, t) = ids[lst[it] .. lst[it + 1]), it = i NT + t
      e_ = base[it + 1];
    }
  };
  int bat = kLeBatch * next_item(ticket, lane), pos = 0;
  auto take = [&]() {
    if (pos == kLeBatch) { bat = kLeBatch * next_item(ticket, lane); pos = 0; }
    return bat + pos++;
  };
  int nitem = take(), ns, ne;
  bounds(nitem, ns, ne);
  for (;;) {
    const int item = nitem;
    if (item >= items) break;
    int s = ns, e = ne;
    nitem = take();
    bounds(nitem, ns, ne);
    int t, tu;
    const int i = fdivmod(item, c.NT, c.inv_NT, t);
    const int tv = fdivmod(t, c.nt, c.inv_nt, tu);
    const int u0 = tu * T, v0 = tv * T;
#if GEM_FWD_L2PF
    // the warp that takes a particle's first tile has the records of the particle GEM_FWD_L2PF
    // ahead prefetched into L2 by one bulk (TMA-engine) prefetch: the first gather of each
    // record then hits L2 instead of HBM
    if (t == 0 && lane == 0 && i + GEM_FWD_L2PF < B) {
      const SplatRec *pf = rec + (size_t)(i + GEM_FWD_L2PF) * c.N;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"((unsigned)(c.N * sizeof(SplatRec)))
                   : "memory");
    }
#endif
    if ((int64_t)e > c.cap) e = (int)c.cap;
    if ((int64_t)s > c.cap) s = (int)c.cap;
    float *out = proj + (size_t)i * c.D * c.D;
    if (s >= e) {   // empty tile: the projection is zero there (or already cleared: zero_empty = 0)
      if (zero_empty) {
        for (int p = lane; p < T * T; p += 32) {
          const int u = u0 + p % T, v = v0 + p / T;
          if (u < c.D && v < c.D) out[(size_t)v * c.D + u] = 0.f;
        }
      }
      continue;
    }
    float2 acc[4][T];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int k = 0; k < T; ++k) acc[p][k] = make_float2(0.f, 0.f);
    const SplatRec *reci = rec + (size_t)i * c.N;
    const int nall = e - s;
#if GEM_FWD_DPF
    // records two rounds ahead, ids three
    int id3 = 64 + lane < nall ? LDID(ids + s + 64 + lane) : 0;
    SplatRec nxt, nxt2;
    if (lane < nall) nxt = reci[LDID(ids + s + lane)];
    if (32 + lane < nall) nxt2 = reci[LDID(ids + s + 32 + lane)];
    for (int g0 = 0; g0 < nall; g0 += 32) {
      const int q = g0 + lane;
      const SplatRec rr = nxt;
      nxt = nxt2;
      if (q + 64 < nall) nxt2 = reci[id3];
      if (q + 96 < nall) id3 = LDID(ids + s + q + 96);
#else
    int id2 = 32 + lane < nall ? LDID(ids + s + 32 + lane) : 0;
    SplatRec nxt;
    if (lane < nall) nxt = reci[LDID(ids + s + lane)];
    for (int g0 = 0; g0 < nall; g0 += 32) {
      const int q = g0 + lane;
      const SplatRec rr = nxt;
      if (q + 32 < nall) nxt = reci[id2];
      if (q + 64 < nall) id2 = LDID(ids + s + q + 64);
#endif
      if (q >= nall) continue;
      const int ub = __float_as_int(rr.f1.z), vb = __float_as_int(rr.f1.w);
      const int ulo = (ub & 0xffff) - u0, uhi = (ub >> 16) - u0, vlo = (vb & 0xffff) - v0, vhi = (vb >> 16) - v0;
      const int cu0 = max(ulo, 0), cu1 = min(uhi, T - 1), cv0 = max(vlo, 0), cv1 = min(vhi, T - 1);
      const int p0 = cv0 >> 1, p1 = cv1 >> 1;
      const unsigned cm = (0xffu << cu0) & (0xffu >> (T - 1 - cu1));   // covered columns
      const float na = nh * rr.f0.z, nb2 = 2.f * nh * rr.f0.w, nc = nh * rr.f1.x, amp = rr.f1.y;
      const float mx = (float)ulo + rr.f0.x, my = (float)vlo + rr.f0.y;
      const float dx0 = (float)cu0 - mx, dyS = (float)(2 * p0) - my, dyE = (float)(2 * p1 + 1) - my;
      // log2 of: e at (cu0, dy); R = e(k+1)/e(k) at cu0; V = e(r+1)/e(r) at cu0
      const float Fx = na * dx0 * dx0, Gx = nb2 * dx0;
      const float fS = fmaf(dyS, fmaf(nc, dyS, Gx), Fx), fE = fmaf(dyE, fmaf(nc, dyE, Gx), Fx);
      const float D0 = na * fmaf(2.f, dx0, 1.f);
      const float gS = fmaf(nb2, dyS, D0), gE = fmaf(nb2, dyE, D0);
      const float hS = fmaf(nc, fmaf(2.f, dyS, 1.f), Gx), hE = fmaf(nc, fmaf(2.f, dyE, 1.f), Gx);
      const bool slow = !(fminf(fS, fE) >= -100.f && fminf(gS, gE) >= -120.f && fmaxf(fabsf(hS), fabsf(hE)) <= 60.f &&
                          nc >= -30.f && fabsf(nb2) <= 60.f);
      const float th = MK ? keep_thr(c, amp, eK) : 0.f;
      if (!slow) {
        const float EA = amp * ex2(fS), VA = ex2(hS), RA = ex2(gS);
        const float W = ex2(2.f * nc), Kb = ex2(nb2), S = ex2(2.f * na);
        float2 E2 = make_float2(EA, EA * VA), R2 = make_float2(RA, RA * Kb);
        const float VVW = VA * VA * W, W2 = W * W;
        float2 VV2 = make_float2(VVW, VVW * W2);
        const float2 W42 = make_float2(W2 * W2, W2 * W2), Kb22 = make_float2(Kb * Kb, Kb * Kb), S2 = make_float2(S, S);
        // all four row pairs run predicated (no branches: the pairs' column chains are
        // independent and interleave); pairs outside [p0, p1] add zeros, and the row-pair
        // recurrence only advances inside [p0, p1], so every factor stays finite
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const bool inr = p >= p0 && p <= p1;
          float2 Em = make_float2(inr && 2 * p >= cv0 ? E2.x : 0.f, inr && 2 * p + 1 <= cv1 ? E2.y : 0.f);
          float2 Rc = R2;
#pragma unroll
          for (int k = 0; k < T; ++k) {
            if (cm & (1u << k)) {
              if (MK) {
                acc[p][k].x += fabsf(Em.x) >= th ? Em.x : 0.f;
                acc[p][k].y += fabsf(Em.y) >= th ? Em.y : 0.f;
              } else {
                acc[p][k] = __fadd2_rn(acc[p][k], Em);
              }
              Em = __fmul2_rn(Em, Rc);
              Rc = __fmul2_rn(Rc, S2);
            }
          }
          if (p >= p0 && p < p1) {   // advance only between covered pairs: no overflow
            E2 = __fmul2_rn(E2, VV2);
            VV2 = __fmul2_rn(VV2, W42);
            R2 = __fmul2_rn(R2, Kb22);
          }
        }
      } else {   // direct evaluation, exp per pixel
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          if (p >= p0 && p <= p1) {
            const float dyA = (float)(2 * p) - my, dyB = dyA + 1.f;
            const bool vA = 2 * p >= cv0, vB = 2 * p + 1 <= cv1;
#pragma unroll
            for (int k = 0; k < T; ++k) {
              if (k >= cu0 && k <= cu1) {
                const float dx = (float)k - mx;
                const float fa = fmaf(dx, fmaf(na, dx, nb2 * dyA), nc * dyA * dyA);
                const float fb = fmaf(dx, fmaf(na, dx, nb2 * dyB), nc * dyB * dyB);
                const float xa = amp * ex2(fa), xb = amp * ex2(fb);
                if (vA && (!MK || fabsf(xa) >= th)) acc[p][k].x += xa;
                if (vB && (!MK || fabsf(xb) >= th)) acc[p][k].y += xb;
              }
            }
          }
        }
      }
    }
    // sum of the 32 private tiles (flattened index n = 16 p + 2 k + (0: .x, 1: .y)) through the
    // warp's shared buffer: lane L stores its copy as row L (16 x 128-bit stores; row pitch 68
    // floats: 4-way, i.e. conflict-free, 128-bit stores), then sums column pair (2L, 2L + 1) over
    // the 32 rows in lane order (32 x 64-bit loads, conflict-free): lane L ends with row pair L / 8,
    // column L % 8.  Fixed order: bitwise deterministic.
    float *buf = le_smem + (threadIdx.x >> 5) * (32 * kLePitch);
    __syncwarp();   // the previous item's reads are done
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int k = 0; k < T; k += 2)
        *reinterpret_cast<float4 *>(buf + lane * kLePitch + 16 * p + 2 * k) =
            make_float4(acc[p][k].x, acc[p][k].y, acc[p][k + 1].x, acc[p][k + 1].y);
    __syncwarp();
    float2 sum = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 32; ++r) sum = __fadd2_rn(sum, *reinterpret_cast<const float2 *>(buf + r * kLePitch + 2 * lane));
    const int u = u0 + (lane & 7), vr = v0 + 2 * (lane >> 3);
    if (u < c.D && vr < c.D) out[(size_t)vr * c.D + u] = sum.x;
    if (u < c.D && vr + 1 < c.D) out[(size_t)(vr + 1) * c.D + u] = sum.y;
  }
  retire(ticket, lane);
}

// Backward ("gradient computation restricted to the Gaussians contributing to each pixel",
// PAPER.md:108, :117), Gaussian-parallel: one thread per (Gaussian j, chunk of kBwdP particles)
// walks the whole box of (i, j) for each particle i of its chunk in turn (no tiles, no lists)
// with the forward's recurrences, two rows at a time (packed fp32), reading g = dL/dI_hat
// through L1/L2 (ids are in Morton order, so the 32 boxes of a warp are spatial neighbours and
// their reads share cache lines).  Per row pair it accumulates packed running sums of h = g e
// (C, Q, Z below: the zeroth to second column moments without forming h k, h k^2), folds them
// with dy into six moments, from which the six 2D
// partials (L_amp, L_mx, L_my, L_a, L_b, L_c) follow algebraically and reduce to the
// image-space gradient (q0 = L_amp amp, l_mx, l_my, G_hat 00/01/11, in Angstrom units).  That is
// transformed to the world frame with W_i = P_i^T and summed over the chunk in particle order:
//   G_mu += W^T (l_mx, l_my, 0),  G_Sigma += W^T [G_hat 0; 0 0] W,  L_rho += q0 / rho,
// (the ten running sums live in shared memory, which keeps the two-row-pair walk below within 64
// registers), and the chunk's ten sums go to slot (chunk, j) (coalesced, one writer); k_bwd_reduce adds the
// chunks in a fixed order: deterministic, no atomics, 10 floats per (chunk, j) of traffic
// instead of 6 per (i, j).
#ifndef GEM_BWD_UNROLL4
#define GEM_BWD_UNROLL4 0
#endif
#ifndef GEM_BWD_RPF
#define GEM_BWD_RPF 0
#endif
#ifndef GEM_BWD_CS
#define GEM_BWD_CS 1
#endif
#ifndef GEM_BWD_TMA
#define GEM_BWD_TMA 0
#endif
#ifndef GEM_BWD_MINB
#define GEM_BWD_MINB 4
#endif
constexpr int kBwdBlock = 256, kBwdP = 8;   // threads per block, particles per thread

template <bool MK, int DT>   // DT: the image edge as a compile-time constant (0: c.D at run time)
__global__ void __launch_bounds__(kBwdBlock, GEM_BWD_MINB) k_render_bwd(CfgDev c, int B, const SplatRec *__restrict__ rec,
                                                          const float *__restrict__ dldi,
                                                          const float *__restrict__ rot, float *__restrict__ slots) {
  constexpr float nh = -0.5f * kLog2e;
  __shared__ float sW[kBwdP][6];   // rows 0 and 1 of W_i = P_i^T for the chunk's particles
  const int j = blockIdx.x * blockDim.x + threadIdx.x, chunk = blockIdx.y;
  const int i0 = chunk * kBwdP, np = min(kBwdP, B - i0);
  if (threadIdx.x < 6 * np) {
    const int p = threadIdx.x / 6, e = threadIdx.x % 6;
    sW[p][e] = rot[9 * (i0 + p) + 3 * (e % 3) + e / 3];   // W[row][col] = P[3 col + row], row = e / 3
  }
#if GEM_BWD_TMA
  // measured variant (not kept: 442.6 vs 433 us): each warp's 32 records of particle
  // i0 + p (one contiguous 1 KB run) staged in shared memory by TMA bulk copies two particles
  // ahead, per-warp double buffer and mbarriers
  __shared__ __align__(128) SplatRec srec[kBwdBlock / 32][2][32];
  __shared__ __align__(8) unsigned long long sbar[kBwdBlock / 32][2];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5, jw = blockIdx.x * blockDim.x + 32 * wq;
  const unsigned tbytes = (unsigned)(max(min(32, c.N - jw), 0) * sizeof(SplatRec));
  if (lane == 0 && tbytes) {
    mbar_init(&sbar[wq][0], 1);
    mbar_init(&sbar[wq][1], 1);
    fence_mbar_init();
    for (int p = 0; p < min(np, 2); ++p) {
      mbar_expect_tx(&sbar[wq][p], tbytes);
      tma_load_1d(srec[wq][p], rec + (size_t)(i0 + p) * c.N + jw, tbytes, &sbar[wq][p]);
    }
  }
#endif
  __syncthreads();
  if (j >= c.N) return;
  __shared__ float sacc[10][kBwdBlock];   // the chunk's ten running sums (off the registers)
  float *vacc = &sacc[0][threadIdx.x];     // vacc[k * kBwdBlock] = sum k
#pragma unroll
  for (int k = 0; k < 10; ++k) vacc[k * kBwdBlock] = 0.f;
#if GEM_BWD_RPF
  SplatRec rnext;
  rnext.f0 = __ldcs(&rec[(size_t)i0 * c.N + j].f0);
  rnext.f1 = __ldcs(&rec[(size_t)i0 * c.N + j].f1);
#endif
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
  const int i = i0 + p;
#if GEM_BWD_TMA
  mbar_wait(&sbar[wq][p & 1], (p >> 1) & 1);
  const SplatRec rr = srec[wq][p & 1][lane];
  __syncwarp(__activemask());
  if (lane == 0 && p + 2 < np) {
    mbar_expect_tx(&sbar[wq][p & 1], tbytes);
    tma_load_1d(srec[wq][p & 1], rec + (size_t)(i + 2) * c.N + jw, tbytes, &sbar[wq][p & 1]);
  }
#else
#if GEM_BWD_RPF
  // the next particle's record loaded one iteration ahead (registers), evict-first
  const SplatRec rr = rnext;
  if (p + 1 < np) {
    rnext.f0 = __ldcs(&rec[(size_t)(i + 1) * c.N + j].f0);
    rnext.f1 = __ldcs(&rec[(size_t)(i + 1) * c.N + j].f1);
  }
#elif GEM_BWD_CS
  // the records stream through once: evict-first (.cs), so that they do not push dL/dI out of L2
  SplatRec rr;
  rr.f0 = __ldcs(&rec[(size_t)i * c.N + j].f0);
  rr.f1 = __ldcs(&rec[(size_t)i * c.N + j].f1);
#else
  const SplatRec rr = rec[(size_t)i * c.N + j];
#endif
#endif
  const int ub = __float_as_int(rr.f1.z), vb = __float_as_int(rr.f1.w);
  const int ulo = ub & 0xffff, uhi = ub >> 16, vlo = vb & 0xffff, vhi = vb >> 16;
  if (ulo > uhi || vlo > vhi) continue;   // culled: contributes nothing
  const int wd = uhi - ulo + 1, ht = vhi - vlo + 1;
  const float ka = rr.f0.z, kb = rr.f0.w, kc = rr.f1.x, amp = rr.f1.y;
  const float na = nh * ka, nb2 = 2.f * nh * kb, nc = nh * kc;
  const float dx0 = -rr.f0.x, dy0 = -rr.f0.y;   // first pixel relative to the centre
  const float Fx = na * dx0 * dx0, Gx = nb2 * dx0, D0 = na * fmaf(2.f, dx0, 1.f);
  const float dyl = dy0 + (float)(ht - 1);
  const float f0 = fmaf(dy0, fmaf(nc, dy0, Gx), Fx), f1 = fmaf(dyl, fmaf(nc, dyl, Gx), Fx);
  const float r0 = fmaf(nb2, dy0, D0), r1 = fmaf(nb2, dyl, D0);
  const bool slow = !(fminf(f0, f1) >= -100.f && fminf(r0, r1) >= -120.f && nc >= -60.f && fabsf(nb2) <= 120.f);
  // MK: keep a pixel iff e >= ethr (= thr / |amp|, see keep_thr)
  const float ethr = MK ? keep_thr(c, amp, ex2(nh * c.k * c.k)) / fabsf(amp) : 0.f;
  // dL/dI in row-pair interleaved layout (k_dldi_pack): pair m, column u holds (g[2m][u], g[2m+1][u])
  const int Dd = DT ? DT : c.D;
  const float *gi = dldi + (size_t)i * Dd * Dd + ((size_t)(vlo >> 1) * Dd + ulo) * 2;
  // Per row the pixel weights h_k (k = 0 .. wd-1) are summed by three running sums,
  // C += h, Q += C, Z += Q (one packed op each instead of forming h k and h k^2): at the end of
  // the row C = sum h, Q = sum h t, Z = sum h t (t + 1) / 2 with t = wd - k, from which
  // sum h k = wd C - Q and sum h k^2 = wd^2 C - 2 wd Q + 2 Z - Q (linear, so the rows are
  // folded in (C, Q, Z) form and converted once per (i, j)).
  float M0 = 0.f, MQ = 0.f, MZ = 0.f, Y0 = 0.f, YQ = 0.f, YY = 0.f;
  float El = 0.f, V = 0.f, Rl = 0.f, W = 0.f, Kb = 0.f, S = 0.f;
  if (!slow) {
    El = ex2(f0);
    V = ex2(fmaf(nc, fmaf(2.f, dy0, 1.f), Gx));
    Rl = ex2(r0);
    W = ex2(2.f * nc);
    Kb = ex2(nb2);
    S = ex2(2.f * na);
  }
  const float wf = (float)wd;
  const float2 S2 = make_float2(S, S);
  auto fold = [&](float2 C, float2 Q, float2 Z, float dyA, float dyB) {
    M0 += C.x + C.y;
    MQ += Q.x + Q.y;
    MZ += Z.x + Z.y;
    Y0 = fmaf(dyA, C.x, fmaf(dyB, C.y, Y0));
    YQ = fmaf(dyA, Q.x, fmaf(dyB, Q.y, YQ));
    YY = fmaf(dyA * dyA, C.x, fmaf(dyB * dyB, C.y, YY));
  };
  // row pairs at absolute (2m, 2m + 1); r = row of the pair's first row relative to vlo (-1 when
  // vlo is odd: that row is outside the box and carries E = 0)
  const float2 *g0 = reinterpret_cast<const float2 *>(gi);
  if (!slow) {
    // two row pairs per iteration (independent chains: twice the loads in flight); rows outside
    // the box carry E = 0.  The second pair is always read one pair below the first (a constant
    // offset): when it lies wholly below the box it reads the next image's first rows, or the
    // buffer's zeroed one-pair pad after the last image -- finite values times E = 0 (a
    // non-finite dL/dI anywhere already makes the step non-finite, GEM_E_NONFINITE)
    auto adv = [&]() { El *= V; V *= W; Rl *= Kb; };
#pragma unroll 1
    for (int r = -(vlo & 1); r < ht; r += 4) {
      const bool a0 = r >= 0, b0 = r + 1 < ht, a1 = r + 2 < ht, b1 = r + 3 < ht;
      const float2 *gp0 = g0 + (size_t)((r + (vlo & 1)) >> 1) * Dd;
      const float2 *gp1 = gp0 + Dd;
      float2 E0, R0, E1, R1;
      E0.x = a0 ? El : 0.f; R0.x = a0 ? Rl : 0.f; if (a0) adv();
      E0.y = b0 ? El : 0.f; R0.y = b0 ? Rl : 0.f; if (b0) adv();
      E1.x = a1 ? El : 0.f; R1.x = a1 ? Rl : 0.f; if (a1) adv();
      E1.y = b1 ? El : 0.f; R1.y = b1 ? Rl : 0.f; if (b1) adv();
      float2 C0 = make_float2(0.f, 0.f), Q0 = C0, Z0 = C0, C1 = C0, Q1 = C0, Z1 = C0;
      auto step = [&](float2 ga, float2 gb) {
        const float2 Ea = MK ? make_float2(E0.x >= ethr ? E0.x : 0.f, E0.y >= ethr ? E0.y : 0.f) : E0;
        const float2 Eb = MK ? make_float2(E1.x >= ethr ? E1.x : 0.f, E1.y >= ethr ? E1.y : 0.f) : E1;
        C0 = __ffma2_rn(ga, Ea, C0);   // C += h, h = g e
        C1 = __ffma2_rn(gb, Eb, C1);   // Eb = 0 below the box: the read pair is finite (pad zeroed)
        Q0 = __fadd2_rn(Q0, C0);
        Q1 = __fadd2_rn(Q1, C1);
        Z0 = __fadd2_rn(Z0, Q0);
        Z1 = __fadd2_rn(Z1, Q1);
        E0 = __fmul2_rn(E0, R0);
        E1 = __fmul2_rn(E1, R1);
        R0 = __fmul2_rn(R0, S2);
        R1 = __fmul2_rn(R1, S2);
      };
      // column pairs at even absolute columns are read with 128-bit loads (two columns of the
      // row pair), four columns per iteration; an odd first column and the last one to three
      // columns are peeled
      int k = 0;
      if (ulo & 1) {
        step(__ldg(gp0), __ldg(gp1));
        k = 1;
      }
#if GEM_BWD_UNROLL4
#pragma unroll 1
      for (; k + 3 < wd; k += 4) {
        const float4 ga = __ldg(reinterpret_cast<const float4 *>(gp0 + k));
        const float4 gb = __ldg(reinterpret_cast<const float4 *>(gp1 + k));
        const float4 gc = __ldg(reinterpret_cast<const float4 *>(gp0 + k + 2));
        const float4 gd = __ldg(reinterpret_cast<const float4 *>(gp1 + k + 2));
        step(make_float2(ga.x, ga.y), make_float2(gb.x, gb.y));
        step(make_float2(ga.z, ga.w), make_float2(gb.z, gb.w));
        step(make_float2(gc.x, gc.y), make_float2(gd.x, gd.y));
        step(make_float2(gc.z, gc.w), make_float2(gd.z, gd.w));
      }
      if (k + 1 < wd) {
#else
#pragma unroll 1
      for (; k + 1 < wd; k += 2) {
#endif
        const float4 ga = __ldg(reinterpret_cast<const float4 *>(gp0 + k));
        const float4 gb = __ldg(reinterpret_cast<const float4 *>(gp1 + k));
        step(make_float2(ga.x, ga.y), make_float2(gb.x, gb.y));
        step(make_float2(ga.z, ga.w), make_float2(gb.z, gb.w));
#if GEM_BWD_UNROLL4
        k += 2;
#endif
      }
      if (k < wd) step(__ldg(gp0 + k), __ldg(gp1 + k));
      const float dyA = dy0 + (float)r;
      fold(C0, Q0, Z0, dyA, dyA + 1.f);
      fold(C1, Q1, Z1, dyA + 2.f, dyA + 3.f);
    }
  } else {
#pragma unroll 1
    for (int r = -(vlo & 1); r < ht; r += 2) {   // direct evaluation, exp per pixel, (C, Q, Z) form
      const bool vA = r >= 0, vB = r + 1 < ht;
      const float dyA = dy0 + (float)r, dyB = dyA + 1.f;
      const float2 *gp = g0 + (size_t)((r + (vlo & 1)) >> 1) * Dd;
      float2 C = make_float2(0.f, 0.f), Q = C, Z = C;
      const float fA = fmaf(dyA, fmaf(nc, dyA, Gx), Fx), fB = fmaf(dyB, fmaf(nc, dyB, Gx), Fx);
      const float gA = fmaf(nb2, dyA, D0), gB = fmaf(nb2, dyB, D0);
#pragma unroll 1
      for (int k = 0; k < wd; ++k) {
        const float tf = wf - (float)k, kf = (float)k, kq = kf * (kf - 1.f) * na;
        float eA = ex2(fmaf(kf, gA, fA) + kq), eB = ex2(fmaf(kf, gB, fB) + kq);
        if (MK) { eA = eA >= ethr ? eA : 0.f; eB = eB >= ethr ? eB : 0.f; }
        const float2 g2 = __ldg(gp + k);
        const float hA = vA ? g2.x * eA : 0.f;
        const float hB = vB ? g2.y * eB : 0.f;
        const float zt = 0.5f * tf * (tf + 1.f);
        C.x += hA; C.y += hB;
        Q.x = fmaf(hA, tf, Q.x); Q.y = fmaf(hB, tf, Q.y);
        Z.x = fmaf(hA, zt, Z.x); Z.y = fmaf(hB, zt, Z.y);
      }
      fold(C, Q, Z, dyA, dyB);
    }
  }
  // (C, Q, Z) moments -> dx-moments: dx = dx0 + k = dxw - t with dxw = dx0 + wd
  const float dxw = dx0 + wf, Mt2 = fmaf(2.f, MZ, -MQ);   // Mt2 = sum h t^2
  const float A0 = M0, A1 = fmaf(dxw, M0, -MQ), A2 = fmaf(dxw, fmaf(dxw, M0, -2.f * MQ), Mt2);
  const float Ay0 = Y0, Ay1 = fmaf(dxw, Y0, -YQ), Ayy0 = YY;
  const float La = A0;
  const float Lmx = amp * fmaf(ka, A1, kb * Ay0), Lmy = amp * fmaf(kb, A1, kc * Ay0);
  const float Lpa = -0.5f * amp * A2, Lpb = -amp * Ay1, Lpc = -0.5f * amp * Ayy0;
  // G_Sigma_hat (pixel units) = -K Gk K - 1/2 L_amp amp K, Gk = [[Lpa, Lpb/2],[Lpb/2, Lpc]]
  const float g01 = 0.5f * Lpb;
  const float KG00 = ka * Lpa + kb * g01, KG01 = ka * g01 + kb * Lpc;
  const float KG10 = kb * Lpa + kc * g01, KG11 = kb * g01 + kc * Lpc;
  const float hl = 0.5f * La * amp;
  const float inv_px = 1.f / c.px, inv_px2 = inv_px * inv_px;
  const float G00 = (-(KG00 * ka + KG01 * kb) - hl * ka) * inv_px2;
  const float G01 = (-(KG00 * kb + KG01 * kc) - hl * kb) * inv_px2;
  const float G11 = (-(KG10 * kb + KG11 * kc) - hl * kc) * inv_px2;
  // world frame, summed over the chunk in particle order
  const float W0[3] = {sW[p][0], sW[p][1], sW[p][2]}, W1[3] = {sW[p][3], sW[p][4], sW[p][5]};
  const float lmx = Lmx * inv_px, lmy = Lmy * inv_px;
  vacc[0 * kBwdBlock] += La * amp;
  vacc[1 * kBwdBlock] += lmx * W0[0] + lmy * W1[0];
  vacc[2 * kBwdBlock] += lmx * W0[1] + lmy * W1[1];
  vacc[3 * kBwdBlock] += lmx * W0[2] + lmy * W1[2];
  float t0[3], t1[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) { t0[l] = G00 * W0[l] + G01 * W1[l]; t1[l] = G01 * W0[l] + G11 * W1[l]; }
  vacc[4 * kBwdBlock] += W0[0] * t0[0] + W1[0] * t1[0];
  vacc[5 * kBwdBlock] += W0[0] * t0[1] + W1[0] * t1[1];
  vacc[6 * kBwdBlock] += W0[0] * t0[2] + W1[0] * t1[2];
  vacc[7 * kBwdBlock] += W0[1] * t0[1] + W1[1] * t1[1];
  vacc[8 * kBwdBlock] += W0[1] * t0[2] + W1[1] * t1[2];
  vacc[9 * kBwdBlock] += W0[2] * t0[2] + W1[2] * t1[2];
  }
  float *dst = slots + (size_t)chunk * 10 * c.N + j;
#pragma unroll
  for (int k = 0; k < 10; ++k) dst[(size_t)k * c.N] = vacc[k * kBwdBlock];
}

// dL/dI (B images of D x D, row-major, from the C2R) -> row-pair interleaved layout read by
// k_render_bwd: out[i][m][u] = (g[i][2m][u], g[i][2m + 1][u]) (D even)
__global__ void __launch_bounds__(256) k_dldi_pack(int D, int64_t npairs, const float2 *__restrict__ in,
                                                   float4 *__restrict__ out) {
  const int h = D >> 1;   // column pairs per row
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (pair row, column pair)
  if (t >= npairs * h) return;
  const int64_t pr = t / h;
  const int64_t src = 2 * pr * h + (t - pr * h);
  const float2 a = __ldcs(in + src), b = __ldcs(in + src + h);
  out[t] = make_float4(a.x, b.x, a.y, b.y);
}

// Per-Gaussian reduction of the chunk slots in chunk order (deterministic), added to acc:
//   acc = (L_rho, G_mu) | G_Sigma (xx xy xz yy) | (yz zz); L_rho = sum q0 / rho.
__global__ void __launch_bounds__(256) k_bwd_reduce(int nchunk, int N, const float *__restrict__ slots,
                                                    const float4 *__restrict__ mean_rho, float4 *__restrict__ acc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  float v[10] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int ch = 0; ch < nchunk; ++ch) {
    const float *src = slots + (size_t)ch * 10 * N + j;
#pragma unroll
    for (int k = 0; k < 10; ++k) v[k] += __ldg(src + (size_t)k * N);
  }
  const float rho = mean_rho[j].w;
  float4 *dst = acc + 3 * (size_t)j;
  float4 a0 = dst[0], a1 = dst[1], a2 = dst[2];
  a0.x += rho != 0.f ? v[0] / rho : 0.f;
  a0.y += v[1]; a0.z += v[2]; a0.w += v[3];
  a1.x += v[4]; a1.y += v[5]; a1.z += v[6]; a1.w += v[7];
  a2.x += v[8]; a2.y += v[9];
  dst[0] = a0; dst[1] = a1; dst[2] = a2;
}

template <typename K>
int persistent_grid(K kern, int threads, size_t smem) {
  int dev = 0, sms = 0, b = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem);
  return sms * (b > 0 ? b : 1);
}

template <int T, bool MK>
void launch_fwd_t(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids, float *proj,
                  int *ticket, cudaStream_t s) {
  static int grid = 0;
  const size_t smem = sizeof(FwdSmem<T>) * kFwdWarps;
  if (!grid) grid = persistent_grid(k_render_fwd<T, MK>, kFwdWarps * 32, smem);
  k_render_fwd<T, MK><<<grid, kFwdWarps * 32, smem, s>>>(c, B, rec, base, ids, proj, ticket);
}

bool pixel_mask(const CfgDev &c) { return (c.flags & (GEM_FLAG_ELLIPSE | GEM_FLAG_PIXEL_TAU)) != 0; }

}  // namespace

void launch_render_fwd(const CfgDev &c, int B, const SplatRec *rec, const int *base, const int *ids, float *proj,
                       int *ticket, cudaStream_t s, int &launches, bool cleared) {
  const bool mk = pixel_mask(c);
  if (c.T == 8) {
    static int grid[2] = {0, 0};
    int &g = grid[mk ? 1 : 0];
    if (!g) g = mk ? persistent_grid(k_render_fwd_le<true>, kLeWarps * 32, 0)
                   : persistent_grid(k_render_fwd_le<false>, kLeWarps * 32, 0);
    if (mk) k_render_fwd_le<true><<<g, kLeWarps * 32, 0, s>>>(c, B, rec, base, ids, proj, ticket, cleared ? 0 : 1);
    else k_render_fwd_le<false><<<g, kLeWarps * 32, 0, s>>>(c, B, rec, base, ids, proj, ticket, cleared ? 0 : 1);
  } else {   // 16 x 16 tiles: lanes own row pairs, entries binned per pair (k_render_fwd<16>)
    if (mk) launch_fwd_t<16, true>(c, B, rec, base, ids, proj, ticket, s);
    else launch_fwd_t<16, false>(c, B, rec, base, ids, proj, ticket, s);
  }
  ++launches;
}

void launch_dldi_pack(const CfgDev &c, int B, const float *in, float *out, cudaStream_t s, int &launches) {
  const int64_t np = (int64_t)B * c.D / 2, n = np * c.D;
  k_dldi_pack<<<(unsigned)((n / 2 + 255) / 256), 256, 0, s>>>(c.D, np, reinterpret_cast<const float2 *>(in),
                                                              reinterpret_cast<float4 *>(out));
  ++launches;
}

int bwd_chunks(int B) { return (B + kBwdP - 1) / kBwdP; }

void launch_render_bwd(const CfgDev &c, int B, const SplatRec *rec, const float *dldi, const float *rot, float *slots,
                       cudaStream_t s, int &launches) {
  dim3 grid((c.N + kBwdBlock - 1) / kBwdBlock, bwd_chunks(B));
  const bool mk = pixel_mask(c);
  auto go = [&](auto kern) { kern<<<grid, kBwdBlock, 0, s>>>(c, B, rec, dldi, rot, slots); };
  if (c.D == 256) mk ? go(k_render_bwd<true, 256>) : go(k_render_bwd<false, 256>);
  else if (c.D == 128) mk ? go(k_render_bwd<true, 128>) : go(k_render_bwd<false, 128>);
  else mk ? go(k_render_bwd<true, 0>) : go(k_render_bwd<false, 0>);
  ++launches;
}

void launch_bwd_reduce(const CfgDev &c, int B, const float *slots, const float4 *mean_rho, float4 *acc, cudaStream_t s,
                       int &launches) {
  k_bwd_reduce<<<(c.N + 255) / 256, 256, 0, s>>>(bwd_chunks(B), c.N, slots, mean_rho, acc);
  ++launches;
}

}  // namespace gem
