// volume.cu — a11 density query gem_render_volume (Eq. 5, PAPER.md:192-196,
// :245; Fig. 2b): V(x) = sum_j 1[x in AABB3_j] rho_j exp(-1/2 d^T Sigma_j^-1 d)
// on a Dv^3 grid of voxel centres ((a - Dv/2) vs, ...), x fastest.
//
// Per Gaussian: fp64 Sigma (canonical O3 order, as in a1) -> integer k-sigma
// voxel box and fp32 Sigma^-1; bin into 8^3 bricks (count, scan, fill); then
// k_vol_stage zeroes the empty bricks and writes each non-empty brick's list,
// sorted by Gaussian id, as brick-local records, and k_vol_render evaluates
// them: a half-warp per 4^3 sub-brick, one record per lane into 64 private
// fp32 accumulators, lane partials summed in a fixed order, so the volume is
// bitwise reproducible.  Every voxel is written once (no memset).
#include "gem_internal.cuh"

namespace gem {
namespace {

constexpr int kBrick = 8, kVolSlots = 8;   // kVolSlots: bricks per Gaussian whose slot the count pass takes

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
                                                  VolRec *__restrict__ out, int *__restrict__ cnt,
                                                  int *__restrict__ cnt_hi, int *__restrict__ pslot, int ps, int nb) {
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
    // the Gaussian's k-th brick (z, y, x order): for k < ps its slot in the brick is taken here
    // (the fill then needs no atomic); the rest are counted in cnt_hi and placed after them
    int k = 0;
    for (int bz = b0[2]; bz <= b1[2]; ++bz)
      for (int by = b0[1]; by <= b1[1]; ++by)
        for (int bx = b0[0]; bx <= b1[0]; ++bx, ++k) {
          const int b = (bz * nb + by) * nb + bx;
          if (k < ps) pslot[(size_t)j * kVolSlots + k] = atomicAdd(&cnt[b], 1);
          else atomicAdd(&cnt_hi[b], 1);
        }
  }
  out[j] = r;
}

__global__ void __launch_bounds__(64) k_vol_fill(int N, const VolRec *__restrict__ rec, const int *__restrict__ off,
                                                  const int *__restrict__ cnt, const int *__restrict__ pslot, int ps,
                                                  int *__restrict__ cursor, int *__restrict__ ids, int64_t cap, int nb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int4 d = rec[j].d;
  if (!d.w) return;
  const int b0x = d.y & 1023, b0y = (d.y >> 10) & 1023, b0z = d.y >> 20;
  const int b1x = d.z & 1023, b1y = (d.z >> 10) & 1023, b1z = d.z >> 20;
  int k = 0;
  for (int bz = b0z; bz <= b1z; ++bz)
    for (int by = b0y; by <= b1y; ++by)
      for (int bx = b0x; bx <= b1x; ++bx, ++k) {
        const int b = (bz * nb + by) * nb + bx;
        const int slot = off[b] + (k < ps ? pslot[(size_t)j * kVolSlots + k] : cnt[b] + atomicAdd(&cursor[b], 1));
        if ((int64_t)slot < cap) ids[slot] = j;
      }
}

// The query's render runs in two kernels.
// k_vol_stage: warp kb writes brick kb as zeros if it is empty, and, for kb < nz[0], takes the
// non-empty brick nz[1 + kb] (nz[0] = their count): it puts the brick's list in ascending
// Gaussian id -- each id's rank = the number of smaller ids in the segment, counted in shared
// memory (or from global memory for segments longer than kVolSort) -- and writes each entry's
// brick-local record (centre in voxel units rounded once from fp64, the log2-kernel
// coefficients, the clipped box) at its rank: the segment [off[b], off[b + 1]) of `vent` is the
// brick's sorted record list (and of `vbox`, their boxes).
// k_vol_render: persistent warps over the tasks (non-empty brick, pair p of its sub-bricks); the
// half-warp h owns the 4^3 sub-brick 2p + h of the brick: it compacts the records whose box
// meets its sub-brick (ballot over 16 boxes per step, in list order) and deals them to its 16
// lanes round-robin; a lane
// evaluates its record over the whole sub-brick into 64 private fp32 accumulators (the box as
// -inf masks on the log2-exponent, one ex2 per voxel: no recurrence, no range cases).  The 16
// partial sub-bricks are then summed in lane order through shared memory (fixed order: the
// volume is bitwise reproducible) and each lane stores one 4-voxel x-row.  Every voxel is
// written exactly once (zeros by k_vol_stage, the rest here).
constexpr int kVolSort = 512, kStWarps = 8;
constexpr int kVrWarps = 4, kVrThreads = 32 * kVrWarps, kVrStage = 128, kVrPitch = 68;

struct __align__(16) VolEnt {
  float4 c;    // centre relative to the brick origin (voxel units), rho
  float4 q0;   // log2-kernel q(d) = Qxx dx^2 + Qyy dy^2 + Qzz dz^2 + Qxy2 dx dy + Qxz2 dx dz + Qyz2 dy dz
  float2 q1;   // Qxz2, Qyz2
  int box;     // brick-local box bounds + 1 (clipped to [-1, 8]), 4 bits each: xl, xh, yl, yh, zl, zh
  int pad;
};
static_assert(sizeof(VolEnt) == 48, "VolEnt is three 16-byte words");

__global__ void __launch_bounds__(kStWarps * 32) k_vol_stage(const VolRec *__restrict__ rec, const int *__restrict__ off,
                                                             const int *__restrict__ ids_in, int64_t cap, int Dv,
                                                             float vs, int nb, const int *__restrict__ nz,
                                                             VolEnt *__restrict__ vent, int *__restrict__ vbox,
                                                             float *__restrict__ vol) {
  __shared__ int sids[kStWarps][kVolSort];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x * kStWarps + w;
  const int nbr = nb * nb * nb;
  if (kb < nbr && off[kb + 1] == off[kb]) {   // brick kb is empty: zeros (lane l: float4s l, l + 32, ..)
    const int bz = kb / (nb * nb), rr = kb - bz * nb * nb, by = rr / nb, bx = rr - by * nb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int f = lane + 32 * q;   // float4 f: slice f / 16, row (f / 2) % 8, voxels 4 (f % 2) ..
      const int X = bx * kBrick + 4 * (f & 1), Y = by * kBrick + ((f >> 1) & 7), Z = bz * kBrick + (f >> 4);
      if ((Dv % kBrick) == 0) {
        *reinterpret_cast<float4 *>(vol + ((size_t)Z * Dv + Y) * Dv + X) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (Y < Dv && Z < Dv) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (X + u < Dv) vol[((size_t)Z * Dv + Y) * Dv + X + u] = 0.f;
      }
    }
  }
  if (kb >= nz[0]) return;
  const int b = nz[1 + kb];
  int s = off[b], e = off[b + 1];
  if ((int64_t)e > cap) e = (int)cap;
  if (s > e) s = e;
  const int n = e - s;
  const int bz = b / (nb * nb), rr = b - bz * nb * nb, by = rr / nb, bx = rr - by * nb;
  const int x0 = bx * kBrick, y0 = by * kBrick, z0 = bz * kBrick;
  const double half = (double)(Dv / 2), ivs = 1.0 / (double)vs;
  const float sc2 = -0.5f * kLog2e * vs * vs;
  const bool small = n <= kVolSort;
  int *si = sids[w];
  if (small) {
    for (int k = lane; k < n; k += 32) si[k] = ids_in[s + k];
    __syncwarp();
  }
  for (int k = lane; k < n; k += 32) {
    const int v = small ? si[k] : ids_in[s + k];
    int r = 0;   // ids are unique within a brick
    if (small) {
      for (int m = 0; m < n; ++m) r += si[m] < v;
    } else {
      for (int m = 0; m < n; ++m) r += ids_in[s + m] < v;
    }
    const VolRec g = rec[v];
    VolEnt E;
    E.c = make_float4((float)fma((double)g.a.x, ivs, half - x0), (float)fma((double)g.a.y, ivs, half - y0),
                      (float)fma((double)g.a.z, ivs, half - z0), g.a.w);
    E.q0 = make_float4(sc2 * g.b.x, sc2 * g.b.w, sc2 * g.c.y, 2.f * sc2 * g.b.y);
    E.q1 = make_float2(2.f * sc2 * g.b.z, 2.f * sc2 * g.c.x);
    const int px_ = __float_as_int(g.c.z), py_ = __float_as_int(g.c.w), pz_ = g.d.x;
    auto cl = [](int u) { return (u < -1 ? -1 : (u > 8 ? 8 : u)) + 1; };
    E.box = cl((px_ & 0xffff) - x0) | (cl((px_ >> 16) - x0) << 4) | (cl((py_ & 0xffff) - y0) << 8) |
            (cl((py_ >> 16) - y0) << 12) | (cl((pz_ & 0xffff) - z0) << 16) | (cl((pz_ >> 16) - z0) << 20);
    E.pad = 0;
    vent[s + r] = E;
    vbox[s + r] = E.box;
  }
}

__device__ __forceinline__ float vex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Persistent warps over the tasks (non-empty brick kb, sub-brick pair p): task t = 4 kb + p.
__global__ void __launch_bounds__(kVrThreads, 4) k_vol_render(const int *__restrict__ off, const int *__restrict__ nz,
                                                              const VolEnt *__restrict__ vent,
                                                              const int *__restrict__ vbox, int64_t cap, int Dv, int nb,
                                                              float *__restrict__ vol) {
  __shared__ unsigned short wl[2 * kVrWarps][kVrStage];   // per-half-warp hit lists
  __shared__ __align__(16) float red[kVrWarps * 32 * kVrPitch];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane >> 4, hl = lane & 15;
  unsigned short *mylist = wl[2 * w + h];
  float *buf = red + w * 32 * kVrPitch;
  const unsigned lt = ((1u << hl) - 1u) << (16 * h);   // the lower lanes of this half
  const unsigned hm = 0xffffu << (16 * h);
  const bool vec = (Dv % kBrick) == 0;
  const int ntask = 4 * nz[0];
  for (int t = blockIdx.x * kVrWarps + w; t < ntask; t += gridDim.x * kVrWarps) {
    const int b = nz[1 + (t >> 2)], sb_ = 2 * (t & 3) + h;   // half h owns sub-brick sb_
    int s = off[b], e = off[b + 1];
    if ((int64_t)e > cap) e = (int)cap;
    if (s > e) s = e;
    const int bz = b / (nb * nb), rr = b - bz * nb * nb, by = rr / nb, bx = rr - by * nb;
    const int sx = 4 * (sb_ & 1), sy = 4 * ((sb_ >> 1) & 1), sz = 4 * (sb_ >> 2);
    float acc[64];
#pragma unroll
    for (int v = 0; v < 64; ++v) acc[v] = 0.f;
    bool any = false;
    for (int cs = s; cs < e; cs += kVrStage) {
      const int n = min(kVrStage, e - cs);
      // this sub-brick's records, in list order (16 tested per step)
      int nh = 0;
      for (int k0 = 0; k0 < n; k0 += 16) {
        const int k = k0 + hl;
        bool hit = false;
        if (k < n) {
          const int bb = vbox[cs + k];
          const int xl = (bb & 15) - 1, xh = ((bb >> 4) & 15) - 1, yl = ((bb >> 8) & 15) - 1,
                    yh = ((bb >> 12) & 15) - 1, zl = ((bb >> 16) & 15) - 1, zh = ((bb >> 20) & 15) - 1;
          hit = xl <= sx + 3 && xh >= sx && yl <= sy + 3 && yh >= sy && zl <= sz + 3 && zh >= sz;
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) mylist[nh + __popc(m & lt)] = (unsigned short)k;
        nh += __popc(m & hm);
      }
      __syncwarp();
      any = any || nh > 0;
      const int nmax = max(nh, __shfl_xor_sync(0xffffffffu, nh, 16));
      for (int r0 = 0; r0 < nmax; r0 += 16) {
        if (r0 + hl < nh) {
          const VolEnt E = vent[cs + mylist[r0 + hl]];
          const float cx = E.c.x - (float)sx, cy = E.c.y - (float)sy, cz = E.c.z - (float)sz, rho = E.c.w;
          const float Qxx = E.q0.x, Qyy = E.q0.y, Qzz = E.q0.z, Qxy2 = E.q0.w, Qxz2 = E.q1.x, Qyz2 = E.q1.y;
          const int bb = E.box;
          const int xl = (bb & 15) - 1 - sx, xh = ((bb >> 4) & 15) - 1 - sx, yl = ((bb >> 8) & 15) - 1 - sy,
                    yh = ((bb >> 12) & 15) - 1 - sy, zl = ((bb >> 16) & 15) - 1 - sz, zh = ((bb >> 20) & 15) - 1 - sz;
          const float NI = -INFINITY;
          float dx[4], kx[4], dy[4], ky[4], dz[4], kz[4], lz[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            dx[q] = (float)q - cx;
            kx[q] = (q >= xl && q <= xh) ? Qxx * dx[q] * dx[q] : NI;
            dy[q] = (float)q - cy;
            ky[q] = (q >= yl && q <= yh) ? Qyy * dy[q] * dy[q] : NI;
            dz[q] = (float)q - cz;
            kz[q] = (q >= zl && q <= zh) ? Qzz * dz[q] * dz[q] : NI;
            lz[q] = Qxz2 * dz[q];
          }
#pragma unroll
          for (int z = 0; z < 4; ++z)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              const float L = fmaf(Qxy2, dy[y], lz[z]);                   // the x-linear coefficient
              const float K = fmaf(Qyz2 * dy[y], dz[z], ky[y] + kz[z]);   // the x-free part (+ masks)
#pragma unroll
              for (int x = 0; x < 4; ++x)
                acc[16 * z + 4 * y + x] = fmaf(rho, vex2(fmaf(dx[x], L, kx[x] + K)), acc[16 * z + 4 * y + x]);
            }
        }
      }
      __syncwarp();
    }
    // each half's 16 partial sub-bricks, summed in lane order; lane hl keeps the x-row of voxels
    // 4 hl .. 4 hl + 3 (y = hl % 4, z = hl / 4)
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int p = 0; p < 16; ++p)
        *reinterpret_cast<float4 *>(buf + lane * kVrPitch + 4 * p) =
            make_float4(acc[4 * p], acc[4 * p + 1], acc[4 * p + 2], acc[4 * p + 3]);
      __syncwarp();
#pragma unroll 8
      for (int r = 0; r < 16; ++r) {
        const float4 v = *reinterpret_cast<const float4 *>(buf + (16 * h + r) * kVrPitch + 4 * hl);
        sum.x += v.x;
        sum.y += v.y;
        sum.z += v.z;
        sum.w += v.w;
      }
      __syncwarp();
    }
    const int X = bx * kBrick + sx, Y = by * kBrick + sy + (hl & 3), Z = bz * kBrick + sz + (hl >> 2);
    if (vec) {
      *reinterpret_cast<float4 *>(vol + ((size_t)Z * Dv + Y) * Dv + X) = sum;
    } else if (Y < Dv && Z < Dv) {
      const float o4[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (X + u < Dv) vol[((size_t)Z * Dv + Y) * Dv + X + u] = o4[u];
    }
  }
}

}  // namespace

// Exclusive scan of the brick counts (cnt + cnt_hi) for the <= 2^17 bricks of Dv <= 400: CTA c
// owns the kVsThreads x kVsItems bricks from c kVsThreads kVsItems.  It first sums the counts
// (and the non-empty bricks) before its range -- a redundant int4 read from L2, all loads in
// flight, no inter-CTA dependency -- then scans its range: warp w owns 32 kVsItems consecutive
// bricks, lane l the bricks 32 q + l (coalesced loads and stores), scanned in that order with
// warp shuffles, then across the warps.  The non-empty bricks are listed at nz[1 + their rank]
// (nz[0] = how many); out[n] = total.
constexpr int kVsThreads = 1024, kVsItems = 8;
__global__ void __launch_bounds__(kVsThreads) k_vol_scan(const int *__restrict__ in, const int *__restrict__ in2,
                                                         int *__restrict__ out, int n, int *__restrict__ nz,
                                                         DevStats *st, int64_t cap) {
  __shared__ int sw[2][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int base = blockIdx.x * kVsThreads * kVsItems;   // (base and n are multiples of 4 below)
  int carry = 0, carryz = 0;
  {
    const int n4 = base / 4;   // the int4 words before this CTA's range
    int a = 0, az = 0;
#pragma unroll 4
    for (int k = threadIdx.x; k < n4; k += kVsThreads) {
      const int4 x = reinterpret_cast<const int4 *>(in)[k], y = reinterpret_cast<const int4 *>(in2)[k];
      const int c0 = x.x + y.x, c1 = x.y + y.y, c2 = x.z + y.z, c3 = x.w + y.w;
      a += c0 + c1 + c2 + c3;
      az += (c0 > 0) + (c1 > 0) + (c2 > 0) + (c3 > 0);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, d);
      az += __shfl_xor_sync(0xffffffffu, az, d);
    }
    if (lane == 0) { sw[0][w] = a; sw[1][w] = az; }
    __syncthreads();
    if (w == 0) {
      a = sw[0][lane];
      az = sw[1][lane];
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, d);
        az += __shfl_xor_sync(0xffffffffu, az, d);
      }
      if (lane == 0) { sw[0][32] = a; sw[1][32] = az; }
    }
    __syncthreads();
    carry = sw[0][32];
    carryz = sw[1][32];
    __syncthreads();
  }
  {
    const int wb = base + 32 * kVsItems * w + lane;
    int v[kVsItems], ex[kVsItems], ez[kVsItems];
#pragma unroll
    for (int q = 0; q < kVsItems; ++q) v[q] = wb + 32 * q < n ? in[wb + 32 * q] + in2[wb + 32 * q] : 0;
    int run = 0, runz = 0;
#pragma unroll
    for (int q = 0; q < kVsItems; ++q) {
      int incl = v[q];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      ex[q] = run + incl - v[q];
      run += __shfl_sync(0xffffffffu, incl, 31);
      const unsigned m = __ballot_sync(0xffffffffu, v[q] > 0);
      ez[q] = runz + __popc(m & lt);
      runz += __popc(m);
    }
    if (lane == 0) { sw[0][w] = run; sw[1][w] = runz; }
    __syncthreads();
    if (w == 0) {   // exclusive scan of the warp totals
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int x = sw[k][lane];
        int xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, xi, d);
          if (lane >= d) xi += y;
        }
        sw[k][lane] = xi - x;
        if (lane == 31) sw[k][32] = xi;
      }
    }
    __syncthreads();
    const int pre = carry + sw[0][w], prez = carryz + sw[1][w];
#pragma unroll
    for (int q = 0; q < kVsItems; ++q) {
      const int i = wb + 32 * q;
      if (i < n) {
        out[i] = pre + ex[q];
        if (v[q] > 0) nz[1 + prez + ez[q]] = i;
      }
    }
    carry += sw[0][32];
    carryz += sw[1][32];
  }
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) {
    out[n] = carry;
    nz[0] = carryz;
    st->entries += (unsigned long long)carry;
    if ((int64_t)carry > cap) st->overflow = 1;
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
  s += align_up(sizeof(int) * (nbr + 1), 256) * 4;  // counts (two), cursor, offsets
  s += align_up(sizeof(int) * (size_t)N * kVolSlots, 256);   // pre-taken slots
  s += align_up(sizeof(int) * (nblk + 1), 256);
  s += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);   // brick lists
  s += align_up(sizeof(VolEnt) * ((size_t)N * 64 + nbr), 256);   // sorted brick-local records
  s += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);      // their boxes
  s += align_up(sizeof(int) * (nbr + 1), 256);   // non-empty brick list
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
  const size_t ni = align_up(sizeof(int) * (nbr + 1), 256) / sizeof(int);
  int *cnt = (int *)p, *cnt_hi = cnt + ni, *cur = cnt + 2 * ni;   // zeroed together
  p += 3 * ni * sizeof(int);
  int *off = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  int *pslot = (int *)p; p += align_up(sizeof(int) * (size_t)N * kVolSlots, 256);
  int *blk = (int *)p; p += align_up(sizeof(int) * (nblk + 1), 256);
  int *ids = (int *)p; p += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);
  VolEnt *vent = (VolEnt *)p; p += align_up(sizeof(VolEnt) * ((size_t)N * 64 + nbr), 256);
  int *vbox = (int *)p; p += align_up(sizeof(int) * ((size_t)N * 64 + nbr), 256);
  int *nz = (int *)p; p += align_up(sizeof(int) * (nbr + 1), 256);
  DevStats *st = (DevStats *)p;
  const int64_t cap = (int64_t)N * 64 + (int64_t)nbr;
  const bool one = nbr <= (1u << 17);   // k_vol_scan; else the general scan over cnt_hi (ps = 0)
  const int ps = one ? kVolSlots : 0;
  cudaMemsetAsync(cnt, 0, 3 * ni * sizeof(int), s);
  cudaMemsetAsync(st, 0, sizeof(DevStats), s);
  k_vol_prep<<<(N + 63) / 64, 64, 0, s>>>(N, mean_rho, log_scale, quat, Dv, (double)vs, (double)k, rec, cnt, cnt_hi,
                                          pslot, ps, nb);
  if (one) {
    k_vol_scan<<<(unsigned)((nbr + kVsThreads * kVsItems - 1) / (kVsThreads * kVsItems)), kVsThreads, 0, s>>>(
        cnt, cnt_hi, off, (int)nbr, nz, st, cap);
    ++launches;
  } else {
    launch_scan(cnt_hi, off, (int64_t)nbr, blk, (int64_t)nblk, st, cap, s, launches);
    cudaMemsetAsync(nz, 0, sizeof(int), s);
    k_vol_compact<<<(unsigned)((nbr + 255) / 256), 256, 0, s>>>(cnt_hi, (int)nbr, nz);
    ++launches;
  }
  k_vol_fill<<<(N + 63) / 64, 64, 0, s>>>(N, rec, off, cnt, pslot, ps, cur, ids, cap, nb);
  k_vol_stage<<<(unsigned)((nbr + kStWarps - 1) / kStWarps), kStWarps * 32, 0, s>>>(rec, off, ids, cap, Dv, vs, nb, nz,
                                                                                   vent, vbox, vol);
  static int rgrid = 0;
  if (!rgrid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vol_render, kVrThreads, 0);
    rgrid = (sms > 0 ? sms : 148) * (per > 0 ? per : 1);
  }
  k_vol_render<<<(unsigned)rgrid, kVrThreads, 0, s>>>(off, nz, vent, vbox, cap, Dv, nb, vol);   // the non-empty bricks
  launches += 4;   // prep, fill, stage, render
  *st_out = st;
  return cudaGetLastError();
}

}  // namespace gem
