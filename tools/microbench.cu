// microbench.cu — step-0 box facts for the roofline denominators:
// FFMA, MUFU ex2, FP64 DFMA, shared-memory atomics (int, f32 CAS), smem RMW,
// and L2 vector reductions red.global.add.v4.f32 on an L2-resident buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu && ./microbench
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_ffma(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.9999f, d = 0.5f, e = 0.25f, f = 0.125f, g = 0.7f, h = 0.3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a = fmaf(a, b, c); d = fmaf(d, b, c); e = fmaf(e, b, c); f = fmaf(f, b, c);
      g = fmaf(g, b, c); h = fmaf(h, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f + g + h;
}

__global__ void k_ex2(float *out, int iters) {
  float a = threadIdx.x * 1e-6f, b = a + 0.1f, c = a + 0.2f, d = a + 0.3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_dfma(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.9999999, d = 0.5, e = 0.25, f = 0.125;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f;
}

__global__ void k_atoms_int(int *out, int iters) {
  __shared__ int s[1024];
  for (int t = threadIdx.x; t < 1024; t += blockDim.x) s[t] = 0;
  __syncthreads();
  int idx = (threadIdx.x * 33) & 1023;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(&s[(idx + k * 37) & 1023], 1);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x & 1023];
}

__global__ void k_atoms_f32(float *out, int iters) {
  __shared__ float s[1024];
  for (int t = threadIdx.x; t < 1024; t += blockDim.x) s[t] = 0;
  __syncthreads();
  int idx = (threadIdx.x * 33) & 1023;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(&s[(idx + k * 37) & 1023], 1.0f);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x & 1023];
}

// warp-private RMW (what a warp-per-entry splat does): LDS + FADD + STS
__global__ void k_smem_rmw(float *out, int iters) {
  __shared__ float s[8][384];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = lane; t < 384; t += 32) s[w][t] = 0;
  __syncwarp();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int a = ((lane >> 3) + k) % 16 * 24 + (lane & 7) + (k & 7);
      s[w][a] += 1.0f;
      __syncwarp();
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[w][lane];
}

__global__ void k_redv4(float4 *acc, int n, int iters, unsigned seed) {
  unsigned x = seed ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    float4 *p = acc + (x % (unsigned)n);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
  }
}

__global__ void k_red1(float *acc, int n, int iters, unsigned seed) {
  unsigned x = seed ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(acc + (x % (unsigned)n), 1.f);
  }
}


__global__ void k_fmul2(float *out, int iters) {
  float2 a = make_float2(threadIdx.x * 1e-3f, 1.f), b = make_float2(1.0001f, 0.9999f), d = a, e = a, f = a, g = a, h = a;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a = __fmul2_rn(a, b); d = __fmul2_rn(d, b); e = __fmul2_rn(e, b); f = __fmul2_rn(f, b);
      g = __fmul2_rn(g, b); h = __fmul2_rn(h, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + d.x + e.x + f.x + g.x + h.x + a.y + d.y + e.y + f.y + g.y + h.y;
}

__global__ void k_ffma2(float *out, int iters) {
  float2 a = make_float2(threadIdx.x * 1e-3f, 1.f), b = make_float2(1.0001f, 0.9999f), c = make_float2(0.5f, 0.25f);
  float2 d = a, e = a, f = a, g = a, h = a;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a = __ffma2_rn(a, b, c); d = __ffma2_rn(d, b, c); e = __ffma2_rn(e, b, c); f = __ffma2_rn(f, b, c);
      g = __ffma2_rn(g, b, c); h = __ffma2_rn(h, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + d.x + e.x + f.x + g.x + h.x + a.y + d.y + e.y + f.y + g.y + h.y;
}

__global__ void k_fmul(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, d = a + 1, e = a + 2, f = a + 3, g = a + 4, h = a + 5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a *= b; d *= b; e *= b; f *= b; g *= b; h *= b;
      asm volatile("" : "+f"(a), "+f"(d), "+f"(e), "+f"(f), "+f"(g), "+f"(h));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f + g + h;
}

// packed recurrence RMW: per step LDS.64, FADD2, STS.64, FMUL2 x2 (two pixels)
__global__ void k_rec_rmw(float *out, int iters) {
  __shared__ float2 s[8][32 * 9];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = lane; t < 32 * 9; t += 32) s[w][t] = make_float2(0.f, 0.f);
  __syncwarp();
  float2 E = make_float2(1e-3f * lane, 2e-3f), R = make_float2(0.999f, 0.998f), S = make_float2(0.9999f, 0.9999f);
  float2 *row = &s[w][lane * 9];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float2 a = row[k];
      a = __fadd2_rn(a, E);
      row[k] = a;
      E = __fmul2_rn(E, R);
      R = __fmul2_rn(R, S);
    }
  }
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[w][lane].x;
}

// direct evaluation RMW: per pixel 2 FFMA, MUFU.EX2, LDS, FFMA, STS
__global__ void k_ex2_rmw(float *out, int iters) {
  __shared__ float s[8][32 * 17];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = lane; t < 32 * 17; t += 32) s[w][t] = 0.f;
  __syncwarp();
  float na = -0.7f, t1 = 0.01f * lane, t2 = -0.3f, amp = 1.3f;
  float *row = &s[w][lane * 17];
  for (int i = 0; i < iters; ++i) {
    float dx = -4.f + 1e-3f * i;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float arg = fmaf(fmaf(na, dx, t1), dx, t2), e;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(arg));
      row[k] = fmaf(amp, e, row[k]);
      dx += 1.f;
    }
  }
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[w][lane];
}


// smem integer atomics with data-dependent values and scattered addresses (fixed-point accumulation)
__global__ void k_atoms_add32(int *out, int iters) {
  __shared__ int s[4096];
  for (int t = threadIdx.x; t < 4096; t += blockDim.x) s[t] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u;
  int v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x = x * 1664525u + 1013904223u;
      atomicAdd(&s[x >> 20], v);
      v += k;
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}
__global__ void k_atoms_add64(unsigned long long *out, int iters) {
  __shared__ unsigned long long s[2048];
  for (int t = threadIdx.x; t < 2048; t += blockDim.x) s[t] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u;
  unsigned long long v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x = x * 1664525u + 1013904223u;
      atomicAdd(&s[x >> 21], v);
      v += k;
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}
// float -> int32 fixed point via magic-constant add, then ATOMS.ADD
__global__ void k_fix_atoms(int *out, int iters) {
  __shared__ int s[4096];
  for (int t = threadIdx.x; t < 4096; t += blockDim.x) s[t] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u;
  float e = 0.37f + threadIdx.x * 1e-4f, r = 0.999f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x = x * 1664525u + 1013904223u;
      const int q = __float2int_rn(e * 1048576.f);
      atomicAdd(&s[x >> 20], q);
      e *= r;
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1e3);
  float *buf; double *dbuf; int *ibuf;
  const int blocks = sms * 8, threads = 256;
  CK(cudaMalloc(&buf, sizeof(float) * blocks * threads * 4));
  CK(cudaMalloc(&dbuf, sizeof(double) * blocks * threads));
  CK(cudaMalloc(&ibuf, sizeof(int) * blocks * threads));
  const int it = 2000;
  double nthr = (double)blocks * threads;
  float ms = timeit([&] { k_ffma<<<blocks, threads>>>(buf, it); });
  printf("FFMA: %.2f T lane-FMA/s (%.1f TFLOP/s)\n", nthr * it * 16 * 6 / ms / 1e9, 2 * nthr * it * 16 * 6 / ms / 1e9);
  ms = timeit([&] { k_ex2<<<blocks, threads>>>(buf, it); });
  printf("MUFU ex2: %.3f T/s (%.1f per SM per clk at max clock)\n", nthr * it * 64 / ms / 1e9,
         nthr * it * 64 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(dbuf, it / 4); });
  printf("DFMA: %.2f T lane-DFMA/s\n", nthr * (it / 4) * 16 * 4 / ms / 1e9);
  ms = timeit([&] { k_atoms_int<<<blocks, threads>>>(ibuf, it / 4); });
  printf("ATOMS.ADD int (spread): %.3f T lane-ops/s (%.2f lanes/clk/SM)\n", nthr * (it / 4) * 8 / ms / 1e9,
         nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_atoms_f32<<<blocks, threads>>>(buf, it / 4); });
  printf("smem atomicAdd f32 (CAS): %.3f T lane-ops/s (%.2f lanes/clk/SM)\n", nthr * (it / 4) * 8 / ms / 1e9,
         nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_smem_rmw<<<blocks, threads>>>(buf, it / 4); });
  printf("smem RMW warp-private: %.3f T lane-ops/s (%.2f lanes/clk/SM)\n", nthr * (it / 4) * 8 / ms / 1e9,
         nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  float4 *acc;
  const int n = 150000;  // N x 3 float4 at config R (2.4 MB, L2-resident)
  CK(cudaMalloc(&acc, sizeof(float4) * n));
  cudaMemset(acc, 0, sizeof(float4) * n);
  ms = timeit([&] { k_redv4<<<blocks, threads>>>(acc, n, 200, 7); });
  printf("red.global.add.v4.f32 random over %d float4: %.3f G ops/s\n", n, nthr * 200 / ms / 1e6);
  ms = timeit([&] { k_red1<<<blocks, threads>>>((float *)acc, 4 * n, 200, 7); });
  printf("red.global.add.f32 random over %d floats: %.3f G ops/s\n", 4 * n, nthr * 200 / ms / 1e6);
  ms = timeit([&] { k_fmul2<<<blocks, threads>>>(buf, it); });
  printf("FMUL2: %.2f T lane-FMUL/s (x2 packed)\n", 2 * nthr * it * 16 * 6 / ms / 1e9);
  ms = timeit([&] { k_ffma2<<<blocks, threads>>>(buf, it); });
  printf("FFMA2: %.2f T lane-FMA/s (x2 packed)\n", 2 * nthr * it * 16 * 6 / ms / 1e9);
  ms = timeit([&] { k_fmul<<<blocks, threads>>>(buf, it); });
  printf("FMUL: %.2f T lane-FMUL/s\n", nthr * it * 16 * 6 / ms / 1e9);
  ms = timeit([&] { k_rec_rmw<<<blocks, threads>>>(buf, it / 4); });
  printf("recurrence RMW: %.3f T pixel/s (%.2f pixels/clk/SM)\n", 2 * nthr * (it / 4) * 8 / ms / 1e9,
         2 * nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_ex2_rmw<<<blocks, threads>>>(buf, it / 4); });
  printf("ex2 RMW: %.3f T pixel/s (%.2f pixels/clk/SM)\n", nthr * (it / 4) * 16 / ms / 1e9,
         nthr * (it / 4) * 16 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_atoms_add32<<<blocks, threads>>>(ibuf, it / 4); });
  printf("ATOMS.ADD.32 random: %.2f lanes/clk/SM\n", nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_atoms_add64<<<blocks, threads>>>((unsigned long long *)dbuf, it / 4); });
  printf("ATOMS.ADD.64 random: %.2f lanes/clk/SM\n", nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_fix_atoms<<<blocks, threads>>>(ibuf, it / 4); });
  printf("F2I + ATOMS.ADD.32 random: %.2f lanes/clk/SM\n", nthr * (it / 4) * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  printf("done\n");
  return 0;
}
