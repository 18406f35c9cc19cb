// f1: z-sorted per-tile lists, GEM_FLAG_ZSORT.
//
// "we sort the selected Gaussians along the z-axis and accumulate them starting
// from the lowest z value (closest to the sensor)".  Each (particle i, tile) list is reordered by
// the key (z_ij, j) ascending, z_ij = camera-frame depth of Gaussian j's centre under pose i,
//   z_ij = ((W20 mu_x + W21 mu_y) + W22 mu_z),   W = P_i^T  (reading L8),
// evaluated in fp64 from the fp32 inputs with round-to-nearest multiplies and adds and no FMA
// contraction (zdepth64), so the key -- and hence the sorted list -- is a bit-exact function of
// the inputs (reading L24 in DESIGN.md; the oracle sorts its own lists with the same definition).
//
// In z-sort mode k_fill writes every entry as an (id, ord32(fp32(z_ij))) pair (zpair) instead of
// an id.  k_zsort_triage (one thread per segment) moves single-entry segments' ids into place and
// queues the longer ones; k_zsort_seg (persistent, one CTA per queued segment) sorts a segment of
// up to kZCap entries with a bucket sort on the fp32 depth followed by an exact in-bucket order:
//   1. the pairs are loaded once into registers; block min / max of the fp32 depth;
//   2. bucket q = min(NB-1, (int)((z - zmin) * (NB-1) / (zmax - zmin))) -- every step is
//      monotone in z, so buckets are ordered by depth -- counted, scanned, and scattered with
//      shared-memory atomics (the order inside a bucket is arbitrary at this point);
//   3. each bucket of >= 2 entries is insertion-sorted by (fp32 depth key, id);
//   4. runs of equal fp32 depth (rare) are re-sorted by the exact (fp64 z, j) key.
// The result is the exact (z, j) order, independent of the atomics' and the queue's order.
// Longer segments (> kZCap entries behind one tile) are sorted in kZCap runs by a shared-memory
// bitonic network on the exact key, then merged pairwise by rank (each element's output slot =
// its rank in its own run + its rank in the sibling run, by binary search) through `tmp`.

#include "gem_internal.cuh"

namespace gem {
namespace {

constexpr int kZThreads = 256;
constexpr int kZCap = 2048;          // entries per shared-memory sort
constexpr int kZPer = kZCap / kZThreads;
constexpr int kZBinsMax = 2 * kZCap;

struct ZKey {
  unsigned long long k;
  int j;
};

__device__ __forceinline__ bool zless(const ZKey &a, const ZKey &b) {
  return a.k < b.k || (a.k == b.k && a.j < b.j);
}

// order-preserving map of an fp64 value to uint64 (-0 < +0 is harmless: the id breaks ties)
__device__ __forceinline__ unsigned long long ord64(double z) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(z);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double depth64(int j, const float4 *__restrict__ mean_rho, double w0, double w1, double w2) {
  return zdepth64(__ldg(mean_rho + j), w0, w1, w2);
}

__device__ __forceinline__ ZKey key_of(int j, const float4 *__restrict__ mean_rho, double w0, double w1, double w2) {
  return ZKey{ord64(depth64(j, mean_rho, w0, w1, w2)), j};
}

__device__ __forceinline__ float unord32(unsigned k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ bool kless(unsigned ka, int ja, unsigned kb, int jb) {
  return ka < kb || (ka == kb && ja < jb);
}

__device__ __forceinline__ void segment(const CfgDev &c, const int *__restrict__ base, int g, int64_t &s, int &n) {
  s = base[g];   // base = lst: list (i, t) = ids[lst[g] .. lst[g + 1]), g = i * NT + t
  int64_t e = base[g + 1];
  if (e > c.cap) e = c.cap;
  n = (int)(e - s);
}

// queue[0] = count; entries (start, length, particle) from int4 slot 1 on
__global__ void __launch_bounds__(256) k_zsort_triage(CfgDev c, int nseg, const int *__restrict__ base,
                                                      const uint2 *__restrict__ zpair, int *__restrict__ ids,
                                                      int *__restrict__ queue) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  int64_t s;
  int n;
  segment(c, base, g, s, n);
  if (n == 1) ids[s] = (int)zpair[s].x;
  else if (n > 1) reinterpret_cast<int4 *>(queue)[1 + atomicAdd(queue, 1)] = make_int4((int)s, n, g / c.NT, 0);
}

// block-wide exclusive scan of one int per thread
__device__ __forceinline__ int block_excl_scan(int v, int *warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  int pre = 0;
  for (int q = 0; q < w; ++q) pre += warp_tot[q];
  __syncthreads();
  return pre + inc - v;
}

struct ZSegSmem {
  unsigned k[kZCap];
  int j[kZCap];
  int cnt[kZBinsMax];
  int warp_tot[kZThreads / 32];
  float red[2][kZThreads / 32];
  int any;
};

__device__ void block_bucket_sort(int *seg, const uint2 *segpair, int n, ZSegSmem &S,
                                  const float4 *__restrict__ mean_rho, double w0, double w1, double w2) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // 1. load once; depth range
  unsigned kr[kZPer];
  int jr[kZPer];
  float zmin = INFINITY, zmax = -INFINITY;
#pragma unroll
  for (int u = 0; u < kZPer; ++u) {
    const int x = tid + u * kZThreads;
    kr[u] = 0u;
    jr[u] = 0;
    if (x < n) {
      const uint2 p = __ldg(segpair + x);
      jr[u] = (int)p.x;
      kr[u] = p.y;
      const float z = unord32(p.y);
      zmin = fminf(zmin, z);
      zmax = fmaxf(zmax, z);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zmin = fminf(zmin, __shfl_xor_sync(0xffffffffu, zmin, o));
    zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  }
  if (lane == 0) { S.red[0][w] = zmin; S.red[1][w] = zmax; }
  int NB = kZThreads;
  while (NB < 2 * n && NB < kZBinsMax) NB <<= 1;
  const int per = NB / kZThreads;   // bins per thread, contiguous
  for (int q = tid; q < NB; q += kZThreads) S.cnt[q] = 0;
  if (tid == 0) S.any = 0;
  __syncthreads();
  zmin = S.red[0][0];
  zmax = S.red[1][0];
  for (int q = 1; q < kZThreads / 32; ++q) { zmin = fminf(zmin, S.red[0][q]); zmax = fmaxf(zmax, S.red[1][q]); }
  const float scale = zmax > zmin ? (float)(NB - 1) / (zmax - zmin) : 0.0f;
  // 2. count, scan, scatter
  int bin[kZPer];
#pragma unroll
  for (int u = 0; u < kZPer; ++u) {
    const int x = tid + u * kZThreads;
    bin[u] = 0;
    if (x < n) {
      bin[u] = min(NB - 1, (int)((unord32(kr[u]) - zmin) * scale));
      atomicAdd(&S.cnt[bin[u]], 1);
    }
  }
  __syncthreads();
  int run = 0;
  for (int q = 0; q < per; ++q) run += S.cnt[tid * per + q];
  int off = block_excl_scan(run, S.warp_tot);
  for (int q = 0; q < per; ++q) {   // cnt[q] := start of bucket q
    const int cq = S.cnt[tid * per + q];
    S.cnt[tid * per + q] = off;
    off += cq;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kZPer; ++u) {
    const int x = tid + u * kZThreads;
    if (x < n) {
      const int pos = atomicAdd(&S.cnt[bin[u]], 1);
      S.k[pos] = kr[u];
      S.j[pos] = jr[u];
    }
  }
  __syncthreads();
  // 3. bucket q now spans [cnt[q-1], cnt[q])
  for (int q = tid * per; q < tid * per + per; ++q) {
    const int e = S.cnt[q], b0 = q == 0 ? 0 : S.cnt[q - 1];
    for (int a = b0 + 1; a < e; ++a) {
      const unsigned ka = S.k[a];
      const int ja = S.j[a];
      int b = a - 1;
      while (b >= b0 && kless(ka, ja, S.k[b], S.j[b])) {
        S.k[b + 1] = S.k[b];
        S.j[b + 1] = S.j[b];
        --b;
      }
      S.k[b + 1] = ka;
      S.j[b + 1] = ja;
    }
  }
  __syncthreads();
  // 4. runs of equal fp32 depth: exact (fp64 z, j) order
  bool tie = false;
  for (int x = tid; x + 1 < n; x += kZThreads) tie |= S.k[x] == S.k[x + 1];
  if (tie) S.any = 1;
  __syncthreads();
  if (S.any) {
    for (int x = tid; x + 1 < n; x += kZThreads) {
      if (S.k[x] != S.k[x + 1] || (x > 0 && S.k[x - 1] == S.k[x])) continue;
      int L = 2;
      while (x + L < n && S.k[x + L] == S.k[x]) ++L;
      for (int a = x + 1; a < x + L; ++a) {
        const int jv = S.j[a];
        const double za = depth64(jv, mean_rho, w0, w1, w2);
        int b = a - 1;
        while (b >= x) {
          const int jw = S.j[b];
          const double zb = depth64(jw, mean_rho, w0, w1, w2);
          if (zb < za || (zb == za && jw < jv)) break;
          S.j[b + 1] = jw;
          --b;
        }
        S.j[b + 1] = jv;
      }
    }
    __syncthreads();
  }
  for (int x = tid; x < n; x += kZThreads) seg[x] = S.j[x];
}

// bitonic sort of P (power of two) exact (key, id) pairs in shared memory
__device__ void smem_bitonic(unsigned long long *sk, int *sj, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int s = k >> 1; s > 0; s >>= 1) {
      for (int x = threadIdx.x; x < P; x += blockDim.x) {
        const int y = x ^ s;
        if (y > x) {
          const bool up = (x & k) == 0;
          const ZKey a{sk[x], sj[x]}, b{sk[y], sj[y]};
          if (zless(b, a) == up) {
            sk[x] = b.k; sj[x] = b.j;
            sk[y] = a.k; sj[y] = a.j;
          }
        }
      }
      __syncthreads();
    }
  }
}

// segments longer than kZCap: exact-key runs + rank merges (rare)
__device__ void block_long_sort(int *seg, const uint2 *segpair, int *segtmp, int n, unsigned long long *sk, int *sj,
                                const float4 *__restrict__ mean_rho, double w0, double w1, double w2) {
  for (int x = threadIdx.x; x < n; x += blockDim.x) seg[x] = (int)segpair[x].x;
  __syncthreads();
  for (int r0 = 0; r0 < n; r0 += kZCap) {
    const int m = min(kZCap, n - r0);
    int P = 2;
    while (P < m) P <<= 1;
    for (int x = threadIdx.x; x < P; x += blockDim.x) {
      if (x < m) {
        const ZKey z = key_of(seg[r0 + x], mean_rho, w0, w1, w2);
        sk[x] = z.k; sj[x] = z.j;
      } else {
        sk[x] = ~0ull; sj[x] = 0x7fffffff;
      }
    }
    __syncthreads();
    smem_bitonic(sk, sj, P);
    for (int x = threadIdx.x; x < m; x += blockDim.x) seg[r0 + x] = sj[x];
    __syncthreads();
  }
  int *src = seg, *dst = segtmp;
  for (int wdt = kZCap; wdt < n; wdt <<= 1) {
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
      const int run = x / wdt, a0 = run * wdt;
      const int p0 = (run ^ 1) * wdt, p1 = min(p0 + wdt, n);
      const int me = src[x];
      int out = x;
      if (p0 < n) {
        const ZKey zx = key_of(me, mean_rho, w0, w1, w2);
        int lo = p0, hi = p1;   // count partner elements < zx
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (zless(key_of(src[mid], mean_rho, w0, w1, w2), zx)) lo = mid + 1; else hi = mid;
        }
        out = min(a0, p0) + (x - a0) + (lo - p0);
      }
      dst[out] = me;
    }
    __syncthreads();
    int *sw = src; src = dst; dst = sw;
  }
  if (src != seg)
    for (int x = threadIdx.x; x < n; x += blockDim.x) seg[x] = src[x];
}

__global__ void __launch_bounds__(kZThreads) k_zsort_seg(CfgDev c, const int *__restrict__ base,
                                                         const float4 *__restrict__ mean_rho,
                                                         const float *__restrict__ rot, const uint2 *__restrict__ zpair,
                                                         int *__restrict__ ids, int *__restrict__ tmp,
                                                         const int *__restrict__ queue) {
  extern __shared__ unsigned long long zsm[];
  ZSegSmem &S = *reinterpret_cast<ZSegSmem *>(zsm);
  const int nq = queue[0];
  const int4 *qe = reinterpret_cast<const int4 *>(queue) + 1;
  int4 nxt = blockIdx.x < nq ? qe[blockIdx.x] : make_int4(0, 0, 0, 0);
  for (int q = blockIdx.x; q < nq; q += gridDim.x) {
    const int4 cur = nxt;
    if (q + (int)gridDim.x < nq) nxt = qe[q + gridDim.x];   // prefetch the next segment's entry
    const int64_t s = cur.x;
    const int n = cur.y, i = cur.z;
    // W = P^T, row 2: (P[2], P[5], P[8])
    const double w0 = (double)rot[9 * i + 2], w1 = (double)rot[9 * i + 5], w2 = (double)rot[9 * i + 8];
    if (n <= kZCap)
      block_bucket_sort(ids + s, zpair + s, n, S, mean_rho, w0, w1, w2);
    else
      block_long_sort(ids + s, zpair + s, tmp + s, n, zsm, reinterpret_cast<int *>(zsm + kZCap), mean_rho, w0, w1, w2);
    __syncthreads();
  }
}

}  // namespace

void launch_zsort(const CfgDev &c, int B, const int *base, const float4 *mean_rho, const float *rot, int *ids,
                  const uint2 *zpair, int *tmp, int *queue, cudaStream_t s, int &launches) {
  static_assert(sizeof(ZSegSmem) >= kZCap * (sizeof(unsigned long long) + sizeof(int)), "long-sort smem");
  const size_t smem = sizeof(ZSegSmem);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_zsort_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_zsort_seg, kZThreads, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = (per_sm > 0 ? per_sm : 1) * sms;
  }
  const int nseg = B * c.NT;
  cudaMemsetAsync(queue, 0, sizeof(int), s);
  k_zsort_triage<<<(nseg + 255) / 256, 256, 0, s>>>(c, nseg, base, zpair, ids, queue);
  k_zsort_seg<<<grid, kZThreads, smem, s>>>(c, base, mean_rho, rot, zpair, ids, tmp, queue);
  launches += 2;
}

}  // namespace gem
