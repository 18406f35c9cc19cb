// volume.cu — a11 density query gem_render_volume (Eq. 5, PAPER.md:192-196,
// :245; Fig. 2b): V(x) = sum_j 1[x in AABB3_j] rho_j exp(-1/2 d^T Sigma_j^-1 d)
// on a Dv^3 grid of voxel centres ((a - Dv/2) vs, ...), x fastest.
//
// Per Gaussian: fp64 Sigma (canonical O3 order, as in a1) -> integer k-sigma
// voxel box and fp32 Sigma^-1; bin into 8^3 bricks (count, scan, fill), then
// one CTA per brick accumulates its voxels in fp32 over the brick's list with
// the same warp-ballot compaction as the image render.  Bound by the HBM write
// of the Dv^3 output.  Brick lists are filled with atomics (order within a
// brick is not fixed), so voxel sums are reproducible only to fp32 rounding.
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

__global__ void __launch_bounds__(256) k_vol_prep(int N, const float4 *__restrict__ mr, const float4 *__restrict__ ls,
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
    const double ie[3] = {exp(dm(-2.0, (double)ss.x)), exp(dm(-2.0, (double)ss.y)), exp(dm(-2.0, (double)ss.z))};
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

__global__ void __launch_bounds__(256) k_vol_fill(int N, const VolRec *__restrict__ rec, const int *__restrict__ off,
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

// Persistent CTAs of 64 threads, each walking the non-empty 8^3 bricks b = blockIdx.x,
// + gridDim.x, ... (the volume is zeroed by a memset first; most bricks of a Dv^3 grid are
// empty).  Thread (lx, ly) owns the brick's voxel column (x0 + lx, y0 + ly, z0 .. z0 + 7); warp w
// the rows ly in [4w, 4w + 4).  A brick's entries are staged in shared memory 64 at a time; per
// 32 entries each lane tests one against its warp's 8 x 4 x 8 slab, and the warp walks the hits
// (ballot).  Along z the log2-kernel is quadratic, q(dz) = q_xy + (L + F dz) dz, so a column is
// evaluated by the render's multiplicative recurrence, e <- e r, r <- r s (s = 2^{2F}): 2 exps and
// ~3 instructions per voxel instead of an exp per voxel; entries whose start values leave the
// normal range take the direct path.
constexpr int kVolThreads = 64;

__global__ void __launch_bounds__(kVolThreads) k_vol_render(const VolRec *__restrict__ rec, const int *__restrict__ off,
                                                            const int *__restrict__ ids, int64_t cap, int Dv, float vs,
                                                            int nb, float *__restrict__ vol) {
  __shared__ float4 sa[kVolThreads];   // centre (voxel units, brick-local), rho
  __shared__ float4 sb[kVolThreads];   // A, 2B, 2C, D of q (Sigma^-1 in voxel units, x -1/2 log2 e)
  __shared__ float4 sc[kVolThreads];   // 2E, F, s = 2^{2F}, -
  __shared__ int4 sbox[kVolThreads];   // brick-local x lo|hi<<16, y lo|hi<<16, z lo|hi<<16, -
  const int nbr = nb * nb * nb;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lx = tid & 7, ly = tid >> 3, wy0 = 4 * w;
  const double half = (double)(Dv / 2);
  const float sc2 = -0.5f * kLog2e * vs * vs;
  const float rx = (float)lx, ry = (float)ly;
  for (int b = blockIdx.x; b < nbr; b += gridDim.x) {
    int s = off[b], e = off[b + 1];
    if ((int64_t)e > cap) e = (int)cap;
    if (s >= e) continue;   // empty brick: zeros (memset)
    const int bx = b % nb, by = (b / nb) % nb, bz = b / (nb * nb);
    const int x0 = bx * kBrick, y0 = by * kBrick, z0 = bz * kBrick;
    float acc[kBrick];
#pragma unroll
    for (int z = 0; z < kBrick; ++z) acc[z] = 0.f;
    for (int cs = s; cs < e; cs += kVolThreads) {
      const int n = min(kVolThreads, e - cs);
      __syncthreads();
      if (tid < n) {
        const VolRec r = rec[ids[cs + tid]];
        // centre in voxel units relative to voxel (x0, y0, z0), rounded once from fp64
        sa[tid] = make_float4((float)((double)r.a.x / vs + half - x0), (float)((double)r.a.y / vs + half - y0),
                              (float)((double)r.a.z / vs + half - z0), r.a.w);
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
#pragma unroll
            for (int z = 0; z < kBrick; ++z) {
              if (z >= za && z <= zb) {
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
}

}  // namespace

size_t volume_scratch_bytes(int N, int Dv) {
  const int nb = (Dv + kBrick - 1) / kBrick;
  const size_t nbr = (size_t)nb * nb * nb;
  const size_t nblk = (nbr + 1 + 4095) / 4096;
  size_t s = 0;
  s += align_up(sizeof(VolRec) * (size_t)N, 256);
  s += align_up(sizeof(int) * (nbr + 1), 256) * 3;  // counts, offsets, cursor
  s += align_up(sizeof(int) * (nblk + 1), 256);
  s += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);
  s += sizeof(DevStats) + 256;
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
  DevStats *st = (DevStats *)p;
  const int64_t cap = (int64_t)N * 64 + (int64_t)nbr;
  cudaMemsetAsync(cnt, 0, sizeof(int) * (nbr + 1), s);
  cudaMemsetAsync(cur, 0, sizeof(int) * (nbr + 1), s);
  cudaMemsetAsync(st, 0, sizeof(DevStats), s);
  k_vol_prep<<<(N + 255) / 256, 256, 0, s>>>(N, mean_rho, log_scale, quat, Dv, (double)vs, (double)k, rec, cnt, nb);
  launch_scan(cnt, off, (int64_t)nbr, blk, (int64_t)nblk, st, cap, s, launches);
  k_vol_fill<<<(N + 255) / 256, 256, 0, s>>>(N, rec, off, cur, ids, cap, nb);
  static int rgrid = 0;
  if (!rgrid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vol_render, kVolThreads, 0);
    rgrid = (sms > 0 ? sms : 148) * (per > 0 ? per : 1);
  }
  const unsigned g = (unsigned)(nbr < (size_t)rgrid ? nbr : (size_t)rgrid);
  cudaMemsetAsync(vol, 0, sizeof(float) * (size_t)Dv * Dv * Dv, s);
  k_vol_render<<<g, kVolThreads, 0, s>>>(rec, off, ids, cap, Dv, vs, nb, vol);
  launches += 3;
  *st_out = st;
  return cudaGetLastError();
}

}  // namespace gem
