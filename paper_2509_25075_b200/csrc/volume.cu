// volume.cu — a11 density query gem_render_volume (Eq. 5, PAPER.md:192-196,
// :245; Fig. 2b): V(x) = sum_j 1[x in AABB3_j] rho_j exp(-1/2 d^T Sigma_j^-1 d)
// on a Dv^3 grid of voxel centres ((a - Dv/2) vs, ...), x fastest.
//
// Per Gaussian: fp64 Sigma (canonical O3 order, as in a1) -> integer k-sigma
// voxel box and fp32 Sigma^-1; bin into 8^3 bricks (count, scan, fill), then
// persistent CTAs walk every brick: an empty one is written as zeros, a
// non-empty one sorts its list by Gaussian id in shared memory (the fill's
// atomics leave the order open) and accumulates its voxels in fp32 in that
// order, so the volume is bitwise reproducible.  Bound by the HBM write of the
// Dv^3 output (written once: no separate memset).
#include "gem_internal.cuh"

namespace gem {
namespace {

constexpr int kBrick = 8;

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsb(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

struct __align__(16) VolRec {
  float4 a;   // mu, rho
  float4 b;   // inv00, inv01, inv02, inv11
  float4 c;   // inv12, inv22, box x packed, box y packed
  int4 d;     // box z packed, brick rect lo (packed bx|by<<10|bz<<20), rect hi, valid
};

__device__ __forceinline__ int clip_d(double v, int lo, int hi) {
  if (!(v >= (double)lo)) return lo;
  if (v > (double)hi) return hi;
  return (int)v;
}

__global__ void __launch_bounds__(64) k_vol_prep(int N, const float4 *__restrict__ mr, const float4 *__restrict__ ls,
                                                  const float4 *__restrict__ q, int Dv, double vs, double kk,
                                                  VolRec *__restrict__ out, int *__restrict__ cnt, int nb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const float4 qq = q[j], ss = ls[j], m4 = mr[j];
  double w = qq.x, x = qq.y, y = qq.z, z = qq.w;
  const double n = sqrt(da(da(da(dm(w, w), dm(x, x)), dm(y, y)), dm(z, z)));
  VolRec r;
  r.d = make_int4(0, 0, 0, 0);
  bool ok = n > 0.0 && isfinite(n);
  int lo[3] = {1, 1, 1}, hi[3] = {0, 0, 0};
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
    const double e[3] = {exp(dm(2.0, (double)ss.x)), exp(dm(2.0, (double)ss.y)), exp(dm(2.0, (double)ss.z))};
    // sigma^-2 only enters the fp32 Sigma^-1 (not the box): fp32 exp suffices
    const double ie[3] = {(double)expf(-2.f * ss.x), (double)expf(-2.f * ss.y), (double)expf(-2.f * ss.z)};
    double inv[6];
    const int K[6] = {0, 0, 0, 1, 1, 2}, Lx[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const int k = K[t], l = Lx[t];
      inv[t] = da(da(dm(dm(R[3 * k], ie[0]), R[3 * l]), dm(dm(R[3 * k + 1], ie[1]), R[3 * l + 1])),
                  dm(dm(R[3 * k + 2], ie[2]), R[3 * l + 2]));
    }
    const double mu[3] = {m4.x, m4.y, m4.z};
    const double half = (double)(Dv / 2);
    // degenerate as in the step's prep (oracle O1, reading L18): Sigma, |Sigma|, mu, rho finite
    bool fin = isfinite(exp(dm(2.0, da(da((double)ss.x, (double)ss.y), (double)ss.z)))) && isfinite(m4.x) &&
               isfinite(m4.y) && isfinite(m4.z) && isfinite(m4.w);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double saa = da(da(dm(dm(R[3 * ax], e[0]), R[3 * ax]), dm(dm(R[3 * ax + 1], e[1]), R[3 * ax + 1])),
                            dm(dm(R[3 * ax + 2], e[2]), R[3 * ax + 2]));
      fin = fin && isfinite(saa);
      const double rr = dm(kk, sqrt(saa));
      lo[ax] = clip_d(ceil(da(dv(dsb(mu[ax], rr), vs), half)), 0, Dv);
      hi[ax] = clip_d(floor(da(dv(da(mu[ax], rr), vs), half)), -1, Dv - 1);
    }
    ok = fin && isfinite(inv[0]) && isfinite(inv[3]) && isfinite(inv[5]) && lo[0] <= hi[0] && lo[1] <= hi[1] &&
         lo[2] <= hi[2];
    r.a = m4;
    r.b = make_float4((float)inv[0], (float)inv[1], (float)inv[2], (float)inv[3]);
    r.c = make_float4((float)inv[4], (float)inv[5], __int_as_float(lo[0] | (hi[0] << 16)),
                      __int_as_float(lo[1] | (hi[1] << 16)));
  }
  if (ok) {
    const int b0[3] = {lo[0] / kBrick, lo[1] / kBrick, lo[2] / kBrick};
    const int b1[3] = {hi[0] / kBrick, hi[1] / kBrick, hi[2] / kBrick};
    r.d = make_int4(lo[2] | (hi[2] << 16), b0[0] | (b0[1] << 10) | (b0[2] << 20), b1[0] | (b1[1] << 10) | (b1[2] << 20), 1);
    for (int bz = b0[2]; bz <= b1[2]; ++bz)
      for (int by = b0[1]; by <= b1[1]; ++by)
        for (int bx = b0[0]; bx <= b1[0]; ++bx) atomicAdd(&cnt[(bz * nb + by) * nb + bx], 1);
  }
  out[j] = r;
}

__global__ void __launch_bounds__(64) k_vol_fill(int N, const VolRec *__restrict__ rec, const int *__restrict__ off,
                                                  int *__restrict__ cursor, int *__restrict__ ids, int64_t cap, int nb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int4 d = rec[j].d;
  if (!d.w) return;
  const int b0x = d.y & 1023, b0y = (d.y >> 10) & 1023, b0z = d.y >> 20;
  const int b1x = d.z & 1023, b1y = (d.z >> 10) & 1023, b1z = d.z >> 20;
  for (int bz = b0z; bz <= b1z; ++bz)
    for (int by = b0y; by <= b1y; ++by)
      for (int bx = b0x; bx <= b1x; ++bx) {
        const int b = (bz * nb + by) * nb + bx;
        const int slot = off[b] + atomicAdd(&cursor[b], 1);
        if ((int64_t)slot < cap) ids[slot] = j;
      }
}

// Persistent CTAs of 64 threads walk the 8^3 bricks b = blockIdx.x, + gridDim.x, ...; an empty
// brick is written as zeros.  Thread (lx, ly) owns the brick's voxel column (x0 + lx, y0 + ly,
// z0 .. z0 + 7); warp w the rows ly in [4w, 4w + 4).  A brick's list is first put in ascending
// Gaussian id (each id's rank = the number of smaller ids in the segment, counted in shared memory,
// or from global memory into the second id buffer for segments longer than kVolSort), so the fp32
// sums are accumulated in a fixed order.  Its entries are then staged in shared memory 64 at a
// time; per 32 entries each lane tests one against its warp's 8 x 4 x 8 slab, and the warp walks
// the hits (ballot).  Along z the log2-kernel is quadratic, q(dz) = q_xy + (L + F dz) dz, so a
// column is evaluated by the render's multiplicative recurrence, e <- e r, r <- r s (s = 2^{2F}):
// 2 exps and ~3 instructions per voxel instead of an exp per voxel; entries whose start values
// leave the normal range take the direct path.
constexpr int kVolThreads = 64, kVolSort = 1024;

__global__ void __launch_bounds__(kVolThreads) k_vol_render(const VolRec *__restrict__ rec, const int *__restrict__ off,
                                                            const int *__restrict__ ids_in, int *__restrict__ ids2,
                                                            int64_t cap, int Dv, float vs, int nb,
                                                            float *__restrict__ vol, int *ticket,
                                                            const int *__restrict__ nz) {
  __shared__ float4 sa[kVolThreads];   // centre (voxel units, brick-local), rho
  __shared__ float4 sb[kVolThreads];   // A, 2B, 2C, D of q (Sigma^-1 in voxel units, x -1/2 log2 e)
  __shared__ float4 sc[kVolThreads];   // 2E, F, s = 2^{2F}, -
  __shared__ int4 sbox[kVolThreads];   // brick-local x lo|hi<<16, y lo|hi<<16, z lo|hi<<16, -
  __shared__ int sid[2][kVolSort];     // the brick's ids, then the same in ascending order
  const int nbr = nb * nb * nb;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lx = tid & 7, ly = tid >> 3, wy0 = 4 * w;
  const double half = (double)(Dv / 2), ivs = 1.0 / (double)vs;
  const float sc2 = -0.5f * kLog2e * vs * vs;
  const float rx = (float)lx, ry = (float)ly;
  // phase 1: empty bricks are written as zeros (grid-stride, no per-brick latency chain)
  // (thread t writes the brick row y = t % 8 of slice z = t / 8: two 16-byte stores)
  const bool vec = (Dv % kBrick) == 0;
  for (int b = blockIdx.x; b < nbr; b += gridDim.x) {
    if (off[b + 1] > off[b]) continue;
    const int bz = b / (nb * nb), r = b - bz * nb * nb, by = r / nb, bx = r - by * nb;
    if (vec) {
      float4 *row = reinterpret_cast<float4 *>(vol + ((size_t)(bz * kBrick + (tid >> 3)) * Dv + by * kBrick + (tid & 7)) * Dv +
                                               bx * kBrick);
      row[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      row[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const int X = bx * kBrick + lx, Y = by * kBrick + ly, z0 = bz * kBrick;
      if (X < Dv && Y < Dv) {
#pragma unroll
        for (int z = 0; z < kBrick; ++z)
          if (z0 + z < Dv) vol[((size_t)(z0 + z) * Dv + Y) * Dv + X] = 0.f;
      }
    }
  }
  // phase 2: the non-empty bricks (nz[1 ..], nz[0] = their count) from a ticket
  const int nnz = nz[0];
  __shared__ int sbrk;
  for (;;) {
    __syncthreads();
    if (tid == 0) sbrk = atomicAdd(ticket, 1);
    __syncthreads();
    if (sbrk >= nnz) break;
    const int b = nz[1 + sbrk];
    int s = off[b], e = off[b + 1];
    if ((int64_t)e > cap) e = (int)cap;
    if (s > e) s = e;
    const int bx = b % nb, by = (b / nb) % nb, bz = b / (nb * nb);
    const int x0 = bx * kBrick, y0 = by * kBrick, z0 = bz * kBrick;
    float acc[kBrick];
#pragma unroll
    for (int z = 0; z < kBrick; ++z) acc[z] = 0.f;
    // the segment in ascending id (ids are unique within a brick)
    const int n_all = e - s;
    const int *ids = sid[1] - s;   // ids[s + k] = the k-th smallest
    if (n_all > 0 && n_all <= kVolSort) {
      __syncthreads();
      for (int k = tid; k < n_all; k += kVolThreads) sid[0][k] = ids_in[s + k];
      __syncthreads();
      for (int k = tid; k < n_all; k += kVolThreads) {
        const int v = sid[0][k];
        int r = 0;
        for (int m = 0; m < n_all; ++m) r += sid[0][m] < v;
        sid[1][r] = v;
      }
    } else if (n_all > kVolSort) {   // long segment: rank from global memory into ids2
      for (int k = tid; k < n_all; k += kVolThreads) {
        const int v = ids_in[s + k];
        int r = 0;
        for (int m = 0; m < n_all; ++m) r += ids_in[s + m] < v;
        ids2[s + r] = v;
      }
      __threadfence_block();
      ids = ids2;
    }
    for (int cs = s; cs < e; cs += kVolThreads) {
      const int n = min(kVolThreads, e - cs);
      __syncthreads();
      if (tid < n) {
        const VolRec r = rec[ids[cs + tid]];   // (smem or ids2: visible after the loop's barrier)
        // centre in voxel units relative to voxel (x0, y0, z0), rounded once from fp64
        sa[tid] = make_float4((float)fma((double)r.a.x, ivs, half - x0), (float)fma((double)r.a.y, ivs, half - y0),
                              (float)fma((double)r.a.z, ivs, half - z0), r.a.w);
        const float F = sc2 * r.c.y;
        sb[tid] = make_float4(sc2 * r.b.x, 2.f * sc2 * r.b.y, 2.f * sc2 * r.b.z, sc2 * r.b.w);
        float s2;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(s2) : "f"(2.f * F));
        sc[tid] = make_float4(2.f * sc2 * r.c.x, F, s2, 0.f);
        const int px_ = __float_as_int(r.c.z), py_ = __float_as_int(r.c.w), pz_ = r.d.x;
        auto cl = [](int v) { return v < -1 ? -1 : (v > 8 ? 8 : v); };
        const int xl = cl((px_ & 0xffff) - x0), xh = cl((px_ >> 16) - x0);
        const int yl = cl((py_ & 0xffff) - y0), yh = cl((py_ >> 16) - y0);
        const int zl = cl((pz_ & 0xffff) - z0), zh = cl((pz_ >> 16) - z0);
        sbox[tid] = make_int4((xl & 0xffff) | (xh << 16), (yl & 0xffff) | (yh << 16), (zl & 0xffff) | (zh << 16), 0);
      }
      __syncthreads();
      for (int g = 0; g < n; g += 32) {
        const int k = g + lane;
        bool hit = false;
        if (k < n) {
          const int4 bb = sbox[k];
          const int xl = (short)(bb.x & 0xffff), xh = bb.x >> 16, yl = (short)(bb.y & 0xffff), yh = bb.y >> 16;
          const int zl = (short)(bb.z & 0xffff), zh = bb.z >> 16;
          hit = xl <= 7 && xh >= 0 && yl <= wy0 + 3 && yh >= wy0 && zl <= 7 && zh >= 0;
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        while (m) {
          const int kk = g + __ffs(m) - 1;
          m &= m - 1;
          const int4 bb = sbox[kk];
          const int xl = (short)(bb.x & 0xffff), xh = bb.x >> 16, yl = (short)(bb.y & 0xffff), yh = bb.y >> 16;
          if (!(lx >= xl && lx <= xh && ly >= yl && ly <= yh)) continue;
          const int za = max((int)(short)(bb.z & 0xffff), 0), zb = min(bb.z >> 16, 7);
          const float4 A = sa[kk], Bq = sb[kk], Cq = sc[kk];
          const float dx = rx - A.x, dy = ry - A.y, dz0 = (float)za - A.z;
          const float qxy = fmaf(dx, fmaf(Bq.x, dx, Bq.y * dy), Bq.w * dy * dy);
          const float L = fmaf(Bq.z, dx, Cq.x * dy), F = Cq.y;
          const float q0 = fmaf(dz0, fmaf(F, dz0, L), qxy), r0 = fmaf(F, fmaf(2.f, dz0, 1.f), L);
          if (q0 >= -100.f && r0 >= -120.f && F >= -60.f) {
            float ev, rv;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ev) : "f"(q0));
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(rv) : "f"(r0));
            ev *= A.w;
            const unsigned zm = (0xffu << za) & (0xffu >> (7 - zb));   // the covered slices
#pragma unroll
            for (int z = 0; z < kBrick; ++z) {
              if (zm & (1u << z)) {
                acc[z] += ev;
                ev *= rv;
                rv *= Cq.z;
              }
            }
          } else {   // direct evaluation
#pragma unroll
            for (int z = 0; z < kBrick; ++z) {
              if (z >= za && z <= zb) {
                const float dz = (float)z - A.z;
                float ev;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ev) : "f"(fmaf(dz, fmaf(F, dz, L), qxy)));
                acc[z] = fmaf(A.w, ev, acc[z]);
              }
            }
          }
        }
      }
    }
    const int X = x0 + lx, Y = y0 + ly;
    if (X < Dv && Y < Dv) {
#pragma unroll
      for (int z = 0; z < kBrick; ++z)
        if (z0 + z < Dv) vol[((size_t)(z0 + z) * Dv + Y) * Dv + X] = acc[z];
    }
  }
  if (tid == 0) {   // the last CTA out resets the ticket for the next query on this stream
    __threadfence();
    if (atomicAdd(ticket + 1, 1) == (int)gridDim.x - 1) { ticket[0] = 0; ticket[1] = 0; }
  }
}

}  // namespace

// Exclusive scan of the brick counts, one CTA per 1024 bricks and no inter-CTA dependency: CTA k
// first sums the counts (and the non-empty bricks) of the bricks before its range (a redundant
// reduction from L2, cheap for the <= 2^17 bricks of Dv <= 400), then scans its own range, writes
// off[b] and lists its non-empty bricks at nz[1 + their rank] (nz[0] = how many).  out[n] = total.
constexpr int kVsThreads = 1024;
__device__ __forceinline__ int vs_block_scan(int v, int *sw, int &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) sw[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int x = sw[lane];
    int xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    sw[lane] = xi - x;
    if (lane == 31) sw[32] = xi;
  }
  __syncthreads();
  total = sw[32];
  const int r = sw[wid] + incl - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kVsThreads) k_vol_scan(const int *__restrict__ in, int *__restrict__ out, int n,
                                                         int *__restrict__ nz, DevStats *st, int64_t cap) {
  __shared__ int sw[33];
  const int b0 = blockIdx.x * kVsThreads, b = b0 + threadIdx.x;
  int pre = 0, prez = 0;
  for (int k = threadIdx.x; k < b0; k += kVsThreads) {
    const int v = in[k];
    pre += v;
    prez += v > 0;
  }
  int t0, t1;
  pre = vs_block_scan(pre, sw, t0);    // only the totals are used
  prez = vs_block_scan(prez, sw, t1);
  const int v = b < n ? in[b] : 0;
  int tot, totz;
  const int ex = vs_block_scan(v, sw, tot);
  const int exz = vs_block_scan(v > 0 ? 1 : 0, sw, totz);
  if (b < n) {
    out[b] = t0 + ex;
    if (v > 0) nz[1 + t1 + exz] = b;
  }
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) {
    out[n] = t0 + tot;
    nz[0] = t1 + totz;
    st->entries += (unsigned long long)(t0 + tot);
    if ((int64_t)(t0 + tot) > cap) st->overflow = 1;
  }
}

// non-empty brick list for the large-grid path (order irrelevant: bricks are independent)
__global__ void __launch_bounds__(256) k_vol_compact(const int *__restrict__ cnt, int n, int *__restrict__ nz) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n && cnt[b] > 0) nz[1 + atomicAdd(nz, 1)] = b;
}

size_t volume_scratch_bytes(int N, int Dv) {
  const int nb = (Dv + kBrick - 1) / kBrick;
  const size_t nbr = (size_t)nb * nb * nb;
  const size_t nblk = (nbr + 1 + 4095) / 4096;
  size_t s = 0;
  s += align_up(sizeof(VolRec) * (size_t)N, 256);
  s += align_up(sizeof(int) * (nbr + 1), 256) * 3;  // counts, offsets, cursor
  s += align_up(sizeof(int) * (nblk + 1), 256);
  s += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256) * 2;   // brick lists, sorted copies of long ones
  s += align_up(sizeof(int) * (nbr + 1), 256);   // non-empty brick list
  s += sizeof(DevStats) + 256 + 256;   // + the render's ticket
  return s;
}

void launch_scan(const int *in, int *out, int64_t n, int *blk, int64_t nblk, DevStats *st, int64_t cap, cudaStream_t s,
                 int &launches);

// Enqueues the query; *st_out receives the device counters (overflow) for the caller's check.
cudaError_t launch_volume(int N, const float4 *mean_rho, const float4 *log_scale, const float4 *quat, int Dv,
                          float vs, float k, float *vol, char *scratch, size_t scratch_bytes, cudaStream_t s,
                          int &launches, DevStats **st_out) {
  const int nb = (Dv + kBrick - 1) / kBrick;
  const size_t nbr = (size_t)nb * nb * nb;
  const size_t nblk = (nbr + 1 + 4095) / 4096;
  char *p = scratch;
  VolRec *rec = (VolRec *)p; p += align_up(sizeof(VolRec) * (size_t)N, 256);
  int *cnt = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  int *off = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  int *cur = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  int *blk = (int *)p; p += align_up(sizeof(int) * (nblk + 1), 256);
  int *ids = (int *)p; p += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);
  int *ids2 = (int *)p; p += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);
  int *nz = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  DevStats *st = (DevStats *)p;
  int *ticket = (int *)(p + align_up(sizeof(DevStats), 256));
  const int64_t cap = (int64_t)N * 64 + (int64_t)nbr;
  cudaMemsetAsync(cnt, 0, sizeof(int) * (nbr + 1), s);
  cudaMemsetAsync(cur, 0, sizeof(int) * (nbr + 1), s);
  cudaMemsetAsync(st, 0, sizeof(DevStats), s);
  cudaMemsetAsync(ticket, 0, 2 * sizeof(int), s);   // (scratch is the caller's: no state kept)
  k_vol_prep<<<(N + 63) / 64, 64, 0, s>>>(N, mean_rho, log_scale, quat, Dv, (double)vs, (double)k, rec, cnt, nb);
  if (nbr <= (1u << 17)) {
    k_vol_scan<<<(unsigned)((nbr + kVsThreads - 1) / kVsThreads), kVsThreads, 0, s>>>(cnt, off, (int)nbr, nz, st, cap);
    ++launches;
  } else {
    launch_scan(cnt, off, (int64_t)nbr, blk, (int64_t)nblk, st, cap, s, launches);
    cudaMemsetAsync(nz, 0, sizeof(int), s);
    k_vol_compact<<<(unsigned)((nbr + 255) / 256), 256, 0, s>>>(cnt, (int)nbr, nz);
    ++launches;
  }
  k_vol_fill<<<(N + 63) / 64, 64, 0, s>>>(N, rec, off, cur, ids, cap, nb);
  static int rgrid = 0;
  if (!rgrid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vol_render, kVolThreads, 0);
    rgrid = (sms > 0 ? sms : 148) * (per > 0 ? per : 1);
  }
  const unsigned g = (unsigned)(nbr < (size_t)rgrid ? nbr : (size_t)rgrid);
  k_vol_render<<<g, kVolThreads, 0, s>>>(rec, off, ids, ids2, cap, Dv, vs, nb, vol, ticket, nz);   // writes every voxel
  launches += 3;
  *st_out = st;
  return cudaGetLastError();
}

}  // namespace gem
