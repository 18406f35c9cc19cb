// gem_api.cu — the C ABI declared in include/gem.h: validation, workspace
// carving, cuFFT plan management and the launch sequence of one step.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "gem_internal.cuh"

#include <nvtx3/nvToolsExt.h>

using namespace gem;

namespace {

bool resolve(const gem_config *in, gem_config &c, CfgDev &d) {
  if (!in) return false;
  c = *in;
  if (c.D < 2 || (c.D & 1) || c.D > 8192) return false;
  if (!(c.pixel_size > 0.f) || !std::isfinite(c.pixel_size)) return false;
  if (c.n_gauss < 1 || c.n_gauss > (1ll << 30)) return false;
  if (c.max_batch < 1 || c.max_batch > 65535) return false;
  if (c.cull_k == 0.f) c.cull_k = 3.f;
  if (!(c.cull_k > 0.f) || !(c.tau >= 0.f)) return false;
  if (c.tile == 0) c.tile = 8;
  if (c.tile != 8 && c.tile != 16) return false;
  if (c.beta1 == 0.f) c.beta1 = 0.9f;
  if (c.beta2 == 0.f) c.beta2 = 0.999f;
  if (c.eps == 0.f) c.eps = 1e-8f;
  d.D = c.D;
  d.T = c.tile;
  d.tshift = c.tile == 16 ? 4 : 3;
  d.nt = (c.D + c.tile - 1) / c.tile;
  d.NT = d.nt * d.nt;
  d.inv_NT = 1.0f / (float)d.NT;
  d.inv_nt = 1.0f / (float)d.nt;
  d.N = (int)c.n_gauss;
  d.C = (d.N + kChunk - 1) / kChunk;
  d.px = c.pixel_size;
  d.k = c.cull_k;
  d.tau = c.tau;
  d.flags = c.flags;
  if (c.flags & ~(uint32_t)(GEM_FLAG_FUSED | GEM_FLAG_NO_ROTATION | GEM_FLAG_ISOTROPIC | GEM_FLAG_ZSORT |
                             GEM_FLAG_ELLIPSE | GEM_FLAG_PIXEL_TAU | GEM_FLAG_EXACT_TILES)) return false;
  if ((c.flags & GEM_FLAG_EXACT_TILES) && !(c.flags & (GEM_FLAG_ELLIPSE | GEM_FLAG_PIXEL_TAU))) return false;
  if (c.flags & GEM_FLAG_FUSED) {
    if (c.wave <= 0) {   // auto: keep one wave's splat records, lists and images within ~64 MB of L2
      const double per = (double)d.N * (32 + 8 + 4 * (c.tile == 16 ? 2 : 3)) + (double)c.D * c.D * 4 * 3 +
                         (double)c.D * (c.D / 2 + 1) * 8 * 2;
      c.wave = (int32_t)(64.0 * 1024 * 1024 / per);
    }
    if (c.wave < 1) c.wave = 1;
    if (c.wave > c.max_batch) c.wave = c.max_batch;
  } else {
    c.wave = c.max_batch;
  }
  // the splat kernel keeps kFillWarps tile histograms plus a kChunk exact queue in shared memory
  // and the fill kFillWarps cursor arrays: the tile grid must fit (D <= 856 at 8x8 tiles,
  // D <= 1712 at 16x16)
  if ((size_t)(kFillWarps * d.NT + kChunk) * sizeof(int) > 200 * 1024) return false;
  if (c.list_capacity <= 0)   // per wave (= per batch when not fused)
    c.list_capacity = (int64_t)c.wave * ((c.tile == 16 ? 6 : 12) * (int64_t)d.N + d.NT);
  if (c.list_capacity > 0x7fffffffll) c.list_capacity = 0x7fffffffll;
  d.cap = c.list_capacity;
  return true;
}

// 2D plans, or -- on the row-column spectral path (spectral_rows(D), see ctf_loss.cu) -- 1D
// plans over the B*D rows of the batch (R2C: real rows of D -> D/2+1 bins; C2R the reverse)
// il: the inverse of dL/dI for the backward on the row path: a C2C of length D over the B D / 2
// packed row pairs Z_m = A + i B written by k_ctf_colspec; its output (g[2m][u], g[2m + 1][u])
// is the row-pair interleaved layout k_render_bwd reads
bool make_plan(int D, int B, cufftType type, cufftHandle *h, size_t *ws, bool il = false) {
  if (cufftCreate(h) != CUFFT_SUCCESS) return false;
  if (cufftSetAutoAllocation(*h, 0) != CUFFT_SUCCESS) { cufftDestroy(*h); return false; }
  cufftResult r;
  if (il) {
    int n[1] = {D};
    r = cufftMakePlanMany(*h, 1, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_C2C, B * D / 2, ws);
  } else if (spectral_rows(D)) {
    int n[1] = {D};
    const int Hx = D / 2 + 1;
    const bool fwd = type == CUFFT_R2C;
    r = cufftMakePlanMany(*h, 1, n, n, 1, fwd ? D : Hx, n, 1, fwd ? Hx : D, type, B * D, ws);
  } else {
    int n[2] = {D, D};
    r = cufftMakePlanMany(*h, 2, n, nullptr, 1, 0, nullptr, 1, 0, type, B, ws);
  }
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(*h);
    return false;
  }
  return true;
}

Layout layout(const gem_config &c, const CfgDev &d, size_t cufft_bytes) {
  Layout L{};
  const size_t Bm = (size_t)c.max_batch, W = (size_t)c.wave, N = (size_t)d.N, D = (size_t)d.D;
  const size_t H = D * (D / 2 + 1);
  L.n_hist = (int64_t)W * d.NT * d.C;
  L.list_cap = c.list_capacity;
  L.loss_blocks = ctf_loss_blocks(d.D);
  L.cufft_bytes = cufft_bytes;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.prep = take((sizeof(GaussPrep) + sizeof(GaussPrep32)) * N);   // fp64 prep, then fp32 prep
  L.rec = take(sizeof(SplatRec) * W * N);
  L.box = take(sizeof(uint2) * W * N);
  L.hist = take(sizeof(int) * ((size_t)L.n_hist + W));   // [i][t][chunk] counts, then per-particle totals
  L.subcnt = take(sizeof(unsigned short) * (size_t)L.n_hist * kFillWarps);   // per fill-warp sub-chunk tile counts (16 bits)
  L.base = take(sizeof(int) * (size_t)L.n_hist);                  // [i][chunk][t] (the fill's cursors)
  L.lst = take(sizeof(int) * ((size_t)W * d.NT + 1));              // list starts [i][t] + the total
  L.ids = take(sizeof(int) * (size_t)L.list_cap);
  // + one zeroed row pair: the backward reads one pair below a box (render.cu k_render_bwd)
  L.proj = take(sizeof(float) * (W * D * D + 2 * D));
  L.spec_hat = take(sizeof(float2) * W * H);
  L.spec_obs = take(sizeof(float2) * W * H);
  L.spec_pred = take(sizeof(float2) * W * H);
  L.dldi = take(sizeof(float) * (W * D * D + 2 * D));
  L.slots = take(sizeof(float) * 10 * (size_t)bwd_chunks((int)W) * N);   // backward world-frame sums [chunk][10][j]
  L.acc = take(sizeof(float4) * 3 * N);
  L.loss_part = take(sizeof(double) * Bm * (size_t)L.loss_blocks);
  L.ctf_par = take(ctf_par_bytes() * Bm);
  L.stats = take(sizeof(DevStats));
  L.ticket = take(64);   // persistent-kernel work tickets (self-resetting; zeroed at init)
  L.stage_rot = take(sizeof(float) * 2 * 9 * Bm);   // the staging is double-buffered across calls
  L.stage_shift = take(sizeof(float) * 2 * 2 * Bm);
  L.stage_ctf = take(sizeof(float) * 2 * 8 * Bm);
  L.stage_obs = take(sizeof(float) * 2 * Bm * D * D);
  L.stage_loss = take(sizeof(double) * (Bm + 1));
  L.cufft_work = take(cufft_bytes);
  L.cufft_work2 = take(cufft_bytes);
  L.zs_tmp = take((c.flags & GEM_FLAG_ZSORT) ? sizeof(int) * (size_t)L.list_cap : 0);   // z-sort merge scratch
  L.zs_key = take((c.flags & GEM_FLAG_ZSORT) ? sizeof(uint2) * (size_t)L.list_cap : 0);  // (id, fp32 depth key)
  L.zs_queue = take((c.flags & GEM_FLAG_ZSORT) ? sizeof(int4) * (W * d.NT + 1) : 0);     // segment queue
  L.total = o;
  return L;
}

bool cufft_sizes(int D, int B, size_t *bytes) {
  cufftHandle a, b;
  size_t wa = 0, wb = 0;
  if (!make_plan(D, B, CUFFT_R2C, &a, &wa)) return false;
  if (!make_plan(D, B, CUFFT_C2R, &b, &wb)) { cufftDestroy(a); return false; }
  cufftDestroy(a);
  cufftDestroy(b);
  if (spectral_rows(D)) {
    size_t wi = 0;
    if (!make_plan(D, B, CUFFT_C2R, &b, &wi, true)) return false;
    cufftDestroy(b);
    if (wi > wb) wb = wi;
  }
  *bytes = (wa > wb ? wa : wb) + 4096;
  return true;
}

template <typename T>
T *at(gem_ctx *ctx, size_t off) { return reinterpret_cast<T *>(ctx->ws + off); }

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

bool soa_ok(const gem_soa *s) {
  return s && s->mean_rho && s->log_scale && s->quat;
}
bool soa_aligned(const gem_soa *s) {
  return aligned16(s->mean_rho) && aligned16(s->log_scale) && aligned16(s->quat);
}

gem_status plan_for(gem_ctx *ctx, int B, cufftHandle *r2c, cufftHandle *c2r, cufftHandle *r2c_obs,
                    cufftHandle *c2r_il) {
  for (int k = 0; k < ctx->n_plans; ++k)
    if (ctx->plan_B[k] == B) {
      *r2c = ctx->plan_r2c[k];
      *c2r = ctx->plan_c2r[k];
      *r2c_obs = ctx->plan_obs[k];
      *c2r_il = ctx->plan_il[k];
      return GEM_OK;
    }
  int slot = ctx->n_plans < 8 ? ctx->n_plans : 7;
  if (ctx->n_plans >= 8) {  // evict the last slot
    cufftDestroy(ctx->plan_r2c[7]);
    cufftDestroy(ctx->plan_c2r[7]);
    cufftDestroy(ctx->plan_obs[7]);
    if (ctx->plan_il[7]) cufftDestroy(ctx->plan_il[7]);
    ctx->n_plans = 7;
  }
  size_t wa = 0, wb = 0, wc = 0;
  cufftHandle a, b, o;
  if (!make_plan(ctx->dc.D, B, CUFFT_R2C, &a, &wa)) return GEM_E_CUFFT;
  if (!make_plan(ctx->dc.D, B, CUFFT_C2R, &b, &wb)) { cufftDestroy(a); return GEM_E_CUFFT; }
  if (!make_plan(ctx->dc.D, B, CUFFT_R2C, &o, &wc)) { cufftDestroy(a); cufftDestroy(b); return GEM_E_CUFFT; }
  const size_t cap = ctx->L.cufft_bytes;
  void *work = ctx->ws + ctx->L.cufft_work, *work2 = ctx->ws + ctx->L.cufft_work2;
  if (wa > cap || wb > cap || wc > cap || cufftSetWorkArea(a, work) != CUFFT_SUCCESS ||
      cufftSetWorkArea(b, work) != CUFFT_SUCCESS || cufftSetWorkArea(o, work2) != CUFFT_SUCCESS) {
    cufftDestroy(a); cufftDestroy(b); cufftDestroy(o);
    return GEM_E_CUFFT;
  }
  cufftHandle il = 0;
  if (spectral_rows(ctx->dc.D)) {
    size_t wi = 0;
    if (!make_plan(ctx->dc.D, B, CUFFT_C2R, &il, &wi, true) || wi > cap || cufftSetWorkArea(il, work) != CUFFT_SUCCESS) {
      if (il) cufftDestroy(il);
      cufftDestroy(a); cufftDestroy(b); cufftDestroy(o);
      return GEM_E_CUFFT;
    }
  }
  ctx->plan_il[slot] = il;
  ctx->plan_B[slot] = B;
  ctx->plan_r2c[slot] = a;
  ctx->plan_c2r[slot] = b;
  ctx->plan_obs[slot] = o;
  ctx->n_plans = slot + 1;
  *r2c = a;
  *c2r = b;
  *r2c_obs = o;
  *c2r_il = il;
  return GEM_OK;
}

const char *kProfNames[P_COUNT] = {"prep", "splat_count", "scan", "fill", "render_fwd", "fft_r2c",
                                   "ctf_loss", "fft_c2r", "fft_r2c_obs", "render_bwd", "bwd_reduce", "finalize", "adam", "volume", "zsort"};

// Every profiled region is also an NVTX range (host side, the enqueue of its kernels): an nsys
// or ncu --nvtx run sees the step's phases by name; without a tool attached NVTX is a no-op.
struct Prof {
  gem_ctx *ctx;
  cudaStream_t s;
  int rec;
  Prof(gem_ctx *c, cudaStream_t st, int kind) : ctx(c), s(st), rec(-1) {
    nvtxRangePushA(kProfNames[kind]);
    if (!c->prof_on) return;
    if (c->prof_n >= c->prof_cap) {
      int ncap = c->prof_cap ? 2 * c->prof_cap : 256;
      int *nk = (int *)realloc(c->prof_kind, sizeof(int) * ncap);
      cudaEvent_t *ne = (cudaEvent_t *)realloc(c->prof_ev, sizeof(cudaEvent_t) * 2 * ncap);
      if (!nk || !ne) return;
      c->prof_kind = nk;
      c->prof_ev = ne;
      for (int k = 2 * c->prof_cap; k < 2 * ncap; ++k) cudaEventCreate(&c->prof_ev[k]);
      c->prof_cap = ncap;
    }
    rec = c->prof_n++;
    c->prof_kind[rec] = kind;
    cudaEventRecord(c->prof_ev[2 * rec], s);
  }
  ~Prof() {
    if (rec >= 0) cudaEventRecord(ctx->prof_ev[2 * rec + 1], s);
    nvtxRangePop();
  }
};

// one NVTX range per C-ABI call
struct NvtxCall {
  explicit NvtxCall(const char *name) { nvtxRangePushA(name); }
  ~NvtxCall() { nvtxRangePop(); }
};

#define CK(x)                                          \
  do {                                                 \
    if ((x) != cudaSuccess) return GEM_E_CUDA;         \
  } while (0)
#define CKF(x)                                         \
  do {                                                 \
    if ((x) != CUFFT_SUCCESS) return GEM_E_CUFFT;      \
  } while (0)

}  // namespace

extern "C" {

const char *gem_status_string(gem_status s) {
  switch (s) {
    case GEM_OK: return "ok";
    case GEM_E_INVALID: return "invalid argument";
    case GEM_E_SHAPE: return "inconsistent shape";
    case GEM_E_ALIGN: return "misaligned pointer";
    case GEM_E_CUDA: return "CUDA error";
    case GEM_E_CUFFT: return "cuFFT error";
    case GEM_E_CAPACITY: return "list capacity exceeded";
    case GEM_E_STATE: return "backward without a live forward";
    case GEM_E_NONFINITE: return "non-finite loss or gradient";
  }
  return "unknown status";
}

size_t gem_workspace_bytes(const gem_config *cfg) {
  gem_config c;
  CfgDev d;
  if (!resolve(cfg, c, d)) return 0;
  size_t cb = 0;
  if (!cufft_sizes(c.D, c.wave, &cb)) return 0;
  return layout(c, d, cb).total;
}

gem_status gem_init(const gem_config *cfg, void *workspace, size_t bytes, gem_stream_t stream, gem_ctx **out) {
  if (!cfg || !out) return GEM_E_INVALID;
  *out = nullptr;
  gem_config c;
  CfgDev d;
  if (!resolve(cfg, c, d)) return (cfg->D & 1) || cfg->D < 2 ? GEM_E_SHAPE : GEM_E_INVALID;
  if (!workspace) return GEM_E_INVALID;
  if (((uintptr_t)workspace & 255u) != 0) return GEM_E_ALIGN;
  size_t cb = 0;
  if (!cufft_sizes(c.D, c.wave, &cb)) return GEM_E_CUFFT;
  Layout L = layout(c, d, cb);
  if (bytes < L.total) return GEM_E_SHAPE;
  gem_ctx *ctx = new (std::nothrow) gem_ctx();
  if (!ctx) return GEM_E_INVALID;
  ctx->cfg = c;
  ctx->dc = d;
  ctx->L = L;
  ctx->ws = (char *)workspace;
  ctx->ws_bytes = bytes;
  ctx->stream = (cudaStream_t)stream;
  ctx->n_plans = 0;
  ctx->W = c.wave;
  ctx->fused = (c.flags & GEM_FLAG_FUSED) ? 1 : 0;
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_ctf, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_loss, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_small, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_zero, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_obs_free[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_obs_free[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_sfree[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_sfree[1], cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return GEM_E_CUDA;
  }
  cufftHandle a, b, o, il;
  gem_status st = plan_for(ctx, c.wave, &a, &b, &o, &il);
  if (st != GEM_OK) { gem_destroy(ctx); return st; }
  if (cudaMemsetAsync(ctx->ws + L.stats, 0, sizeof(DevStats), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(ctx->ws + L.ticket, 0, 64, ctx->stream) != cudaSuccess ||
      // the backward reads one row pair below a box: the image buffers (and their pad pair) start
      // zeroed, so that read is finite even past the batch's last image
      cudaMemsetAsync(ctx->ws + L.proj, 0, sizeof(float) * ((size_t)c.wave * c.D * c.D + 2 * c.D), ctx->stream) !=
          cudaSuccess ||
      cudaMemsetAsync(ctx->ws + L.dldi, 0, sizeof(float) * ((size_t)c.wave * c.D * c.D + 2 * c.D), ctx->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    gem_destroy(ctx);
    return GEM_E_CUDA;
  }
  *out = ctx;
  return GEM_OK;
}

gem_status gem_destroy(gem_ctx *ctx) {
  if (!ctx) return GEM_E_INVALID;
  cudaStreamSynchronize(ctx->stream);
  for (int k = 0; k < ctx->n_plans; ++k) {
    cufftDestroy(ctx->plan_r2c[k]);
    cufftDestroy(ctx->plan_c2r[k]);
    cufftDestroy(ctx->plan_obs[k]);
    if (ctx->plan_il[k]) cufftDestroy(ctx->plan_il[k]);
  }
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
    cudaEventDestroy(ctx->ev_ctf);
    cudaEventDestroy(ctx->ev_loss);
  }
  if (ctx->copy) {
    cudaStreamSynchronize(ctx->copy);
    cudaStreamDestroy(ctx->copy);
  }
  for (int k = 0; k < ctx->n_ev_obs; ++k) cudaEventDestroy(ctx->ev_obs[k]);
  for (int k = 0; k < 2; ++k) {
    if (ctx->ev_obs_free[k]) cudaEventDestroy(ctx->ev_obs_free[k]);
    if (ctx->ev_sfree[k]) cudaEventDestroy(ctx->ev_sfree[k]);
  }
  if (ctx->ev_small) cudaEventDestroy(ctx->ev_small);
  if (ctx->ev_zero) cudaEventDestroy(ctx->ev_zero);
  free(ctx->ev_obs);
  for (int k = 0; k < 2 * ctx->prof_cap; ++k) cudaEventDestroy(ctx->prof_ev[k]);
  free(ctx->prof_ev);
  free(ctx->prof_kind);
  delete ctx;
  return GEM_OK;
}

int32_t gem_last_launch_count(const gem_ctx *ctx) { return ctx ? ctx->launches : 0; }

gem_status gem_profile_enable(gem_ctx *ctx, int32_t enable) {
  if (!ctx) return GEM_E_INVALID;
  if (enable) ctx->prof_n = 0;
  ctx->prof_on = enable ? 1 : 0;
  return GEM_OK;
}

int32_t gem_profile_read(gem_ctx *ctx, gem_kernel_time_t *out, int32_t cap) {
  if (!ctx || (!out && cap > 0)) return -1;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -1;
  double tot[P_COUNT] = {0};
  int cnt[P_COUNT] = {0};
  for (int r = 0; r < ctx->prof_n; ++r) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->prof_ev[2 * r + 1]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&ms, ctx->prof_ev[2 * r], ctx->prof_ev[2 * r + 1]) != cudaSuccess) return -1;
    tot[ctx->prof_kind[r]] += ms;
    cnt[ctx->prof_kind[r]] += 1;
  }
  int n = 0;
  for (int k = 0; k < P_COUNT; ++k) {
    if (!cnt[k]) continue;
    if (n < cap) {
      memset(&out[n], 0, sizeof(out[n]));
      strncpy(out[n].name, kProfNames[k], sizeof(out[n].name) - 1);
      out[n].launches = cnt[k];
      out[n].total_ms = tot[k];
    }
    ++n;
  }
  return n;
}

gem_status gem_forward(gem_ctx *ctx, const gem_soa *params, const gem_batch *batch, double *loss, float *proj_out,
                       float *pred_out, gem_stream_t stream) {
  NvtxCall nvtx_("gem_forward");
  if (!ctx || !soa_ok(params) || !batch || !loss) return GEM_E_INVALID;
  if (!batch->rot || !batch->shift || !batch->ctf || !batch->observed) return GEM_E_INVALID;
  const int B = batch->B;
  if (B < 1 || B > ctx->cfg.max_batch) return GEM_E_SHAPE;
  if (!soa_aligned(params)) return GEM_E_ALIGN;
  if (batch->memory != GEM_MEM_DEVICE && batch->memory != GEM_MEM_HOST) return GEM_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  ctx->stream = s;
  ctx->launches = 0;
  ctx->fwd_live = 0;
  const CfgDev &c = ctx->dc;
  const Layout &L = ctx->L;
  const size_t D = (size_t)c.D;
  const float *shift = batch->shift, *ctf = batch->ctf, *obs = batch->observed;
  const bool host = batch->memory == GEM_MEM_HOST;
  // The staging (rotations, kept for gem_backward; in host mode also the shifts, CTFs and
  // images) is double-buffered across calls: this call uses half h.  Half 1 - h was the
  // previous call's: the compute stream reaching this point means its backward has run.
  const int h = ctx->obs_half;
  ctx->obs_half ^= 1;
  const size_t Bm = (size_t)ctx->cfg.max_batch;
  float *rot = at<float>(ctx, L.stage_rot) + (size_t)h * 9 * Bm;
  ctx->rot_cur = rot;
  CK(cudaEventRecord(ctx->ev_sfree[1 - h], s));
  if (!host) {
    CK(cudaMemcpyAsync(rot, batch->rot, sizeof(float) * 9 * B, cudaMemcpyDeviceToDevice, s));
  } else {
    // Every host->device copy runs on the internal copy stream (none on the compute stream,
    // where a small copy could queue behind the images of the next call), after the last
    // readers of half h: the compute stream two calls back (ev_sfree) and that call's image
    // R2Cs on the side stream (ev_obs_free).  Poses and CTFs first (the compute stream waits
    // for them), then the images wave by wave (4 D^2 bytes per particle, the bulk of the
    // input), one event per wave: their R2C on the side stream waits for its wave only.  A
    // caller that enqueues its steps back to back gets call k + 1's inputs copied while call k
    // computes.
    const int nw = (B + ctx->W - 1) / ctx->W;
    if (ctx->n_ev_obs < nw) {
      cudaEvent_t *ne = (cudaEvent_t *)realloc(ctx->ev_obs, sizeof(cudaEvent_t) * nw);
      if (!ne) return GEM_E_CUDA;
      ctx->ev_obs = ne;
      for (; ctx->n_ev_obs < nw; ++ctx->n_ev_obs)
        CK(cudaEventCreateWithFlags(&ctx->ev_obs[ctx->n_ev_obs], cudaEventDisableTiming));
    }
    float *sshift = at<float>(ctx, L.stage_shift) + (size_t)h * 2 * Bm;
    float *sctf = at<float>(ctx, L.stage_ctf) + (size_t)h * 8 * Bm;
    float *sobs = at<float>(ctx, L.stage_obs) + (size_t)h * Bm * D * D;
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_sfree[h], 0));
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_obs_free[h], 0));
    CK(cudaMemcpyAsync(rot, batch->rot, sizeof(float) * 9 * B, cudaMemcpyHostToDevice, ctx->copy));
    CK(cudaMemcpyAsync(sshift, shift, sizeof(float) * 2 * B, cudaMemcpyHostToDevice, ctx->copy));
    CK(cudaMemcpyAsync(sctf, ctf, sizeof(float) * 8 * B, cudaMemcpyHostToDevice, ctx->copy));
    CK(cudaEventRecord(ctx->ev_small, ctx->copy));
    for (int w = 0; w < nw; ++w) {
      const int q0 = w * ctx->W, qn = B - q0 < ctx->W ? B - q0 : ctx->W;
      CK(cudaMemcpyAsync(sobs + q0 * D * D, obs + q0 * D * D, sizeof(float) * qn * D * D, cudaMemcpyHostToDevice,
                         ctx->copy));
      CK(cudaEventRecord(ctx->ev_obs[w], ctx->copy));
    }
    CK(cudaStreamWaitEvent(s, ctx->ev_small, 0));
    shift = sshift;
    ctf = sctf;
    obs = sobs;
  }
  DevStats *st = at<DevStats>(ctx, L.stats);
  CK(cudaMemsetAsync(st, 0, sizeof(DevStats), s));
  GaussPrep *prep = at<GaussPrep>(ctx, L.prep);
  SplatRec *rec = at<SplatRec>(ctx, L.rec);
  uint2 *box = at<uint2>(ctx, L.box);
  int *hist = at<int>(ctx, L.hist), *base = at<int>(ctx, L.base), *ids = at<int>(ctx, L.ids);
  float2 *sh = at<float2>(ctx, L.spec_hat), *so = at<float2>(ctx, L.spec_obs), *sp = at<float2>(ctx, L.spec_pred);
  float *dldi = at<float>(ctx, L.dldi);
  float4 *acc = at<float4>(ctx, L.acc);
  double *lpart = at<double>(ctx, L.loss_part);
  if (ctx->fused) CK(cudaMemsetAsync(acc, 0, sizeof(float4) * 3 * (size_t)c.N, s));
  { Prof p(ctx, s, P_PREP); launch_prep(c, (const float4 *)params->mean_rho, (const float4 *)params->log_scale, (const float4 *)params->quat, prep, st, s, ctx->launches); CK(cudaGetLastError()); }
  const size_t DD = D * D;
  int p0 = 0, nb = 0;
  for (p0 = 0; p0 < B; p0 += ctx->W) {   // one wave (all of B when not fused)
    nb = B - p0 < ctx->W ? B - p0 : ctx->W;
    cufftHandle r2c, c2r, r2c_obs, c2r_il;
    gem_status ps = plan_for(ctx, nb, &r2c, &c2r, &r2c_obs, &c2r_il);
    if (ps != GEM_OK) return ps;
    // fork: the observed images' R2C and the per-particle CTF constants run on the internal side
    // stream, overlapped with the render of this wave; joined before the CTF/loss kernel.  (Forked
    // at the wave's start instead, the R2C overlaps the splat, scan and fill and slows them: the
    // same device-resident step, but 2.5 % less end to end with host inputs.)
    auto fork_side = [&]() -> gem_status {
      CK(cudaEventRecord(ctx->ev_fork, s));
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
      CKF(cufftSetStream(r2c_obs, ctx->side));
      if (host) CK(cudaStreamWaitEvent(ctx->side, ctx->ev_obs[p0 / ctx->W], 0));
      {
        Prof p(ctx, ctx->side, P_FFT_OBS);
        CKF(cufftExecR2C(r2c_obs, (cufftReal *)(obs + p0 * DD), (cufftComplex *)so));
      }
      { Prof p(ctx, ctx->side, P_CTF_LOSS); launch_ctf_params(c, nb, ctf + 8 * (size_t)p0, ctx->ws + L.ctf_par, ctx->side, ctx->launches); CK(cudaGetLastError()); }
      CK(cudaEventRecord(ctx->ev_join, ctx->side));
      return GEM_OK;
    };
    const float *rw = rot + 9 * (size_t)p0;
    // device-resident inputs: the projections of this wave are cleared on the side stream while
    // the splat and binning run, and the 8x8 render skips the empty tiles (~2/3 at R) instead of
    // writing their zeros.  (With host inputs the extra HBM writes during the DMA of the next
    // images cost more end to end than they save: the render writes the zeros itself.)
    const bool cleared = !host && c.T == 8;
    if (cleared) {
      float *projz = proj_out ? proj_out + p0 * DD : at<float>(ctx, L.proj);
      CK(cudaEventRecord(ctx->ev_fork, s));
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
      CK(cudaMemsetAsync(projz, 0, sizeof(float) * nb * DD, ctx->side));
      CK(cudaEventRecord(ctx->ev_zero, ctx->side));
    }
    const int64_t nh = (int64_t)nb * c.NT * c.C;
    int *ptot = hist + nh;   // per-particle entry totals (the splat adds, the scan reads)
    unsigned short *hist16 = reinterpret_cast<unsigned short *>(hist);   // 16-bit counts (<= kChunk)
    CK(cudaMemsetAsync(ptot, 0, sizeof(int) * nb, s));
    { Prof p(ctx, s, P_SPLAT); launch_splat_count(c, nb, prep, (const float4 *)params->mean_rho, rw, shift + 2 * (size_t)p0, rec, box, hist16, at<unsigned short>(ctx, L.subcnt), ptot, st, s,
                         ctx->launches); CK(cudaGetLastError()); }
    {
      Prof p(ctx, s, P_SCAN);
      launch_scan_pp(c, nb, hist16, base, at<int>(ctx, L.lst), ptot, st, at<int>(ctx, L.ticket) + 8, s, ctx->launches);
      CK(cudaGetLastError());
    }
    uint2 *zpair = (c.flags & GEM_FLAG_ZSORT) ? at<uint2>(ctx, L.zs_key) : nullptr;
    { Prof p(ctx, s, P_FILL); launch_fill(c, nb, box, base, at<unsigned short>(ctx, L.subcnt), ids, (const float4 *)params->mean_rho, rw, zpair, rec, s, ctx->launches); CK(cudaGetLastError()); }
    if (zpair) {
      Prof p(ctx, s, P_ZSORT);
      launch_zsort(c, nb, at<int>(ctx, L.lst), (const float4 *)params->mean_rho, rw, ids, zpair, at<int>(ctx, L.zs_tmp),
                   at<int>(ctx, L.zs_queue), s, ctx->launches);
      CK(cudaGetLastError());
    }
    {   // the side stream's work starts with the render (see fork_side)
      const gem_status fs = fork_side();
      if (fs != GEM_OK) return fs;
    }
    float *proj = proj_out ? proj_out + p0 * DD : at<float>(ctx, L.proj);
    if (cleared) CK(cudaStreamWaitEvent(s, ctx->ev_zero, 0));
    { Prof p(ctx, s, P_RENDER_FWD); launch_render_fwd(c, nb, rec, at<int>(ctx, L.lst), ids, proj, at<int>(ctx, L.ticket), s, ctx->launches, cleared); CK(cudaGetLastError()); }
    CKF(cufftSetStream(r2c, s));
    CKF(cufftSetStream(c2r, s));
    {
      Prof p(ctx, s, P_FFT_R2C);
      CKF(cufftExecR2C(r2c, (cufftReal *)proj, (cufftComplex *)sh));
    }
    CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    {
      Prof p(ctx, s, P_CTF_LOSS);
      launch_ctf_loss(c, nb, ctx->ws + L.ctf_par, sh, so, pred_out ? sp : nullptr,
                      c2r_il ? at<float2>(ctx, L.proj) : nullptr, lpart + (size_t)p0 * L.loss_blocks,
                      L.loss_blocks, s, ctx->launches);
      CK(cudaGetLastError());
    }
    CK(cudaEventRecord(ctx->ev_ctf, s));
    {
      Prof p(ctx, s, P_FFT_C2R);
      if (pred_out) CKF(cufftExecC2R(c2r, (cufftComplex *)sp, (cufftReal *)(pred_out + p0 * DD)));
      // dL/dI in the backward's row-pair interleaved layout: on the row path the column kernel
      // wrote the packed row pairs Z into the proj region (dead after the R2C; unused when the
      // caller takes the projections) and one C2C inverts them; otherwise the 2D C2R writes
      // row-major into the proj region and k_dldi_pack interleaves
      if (c2r_il) {
        CKF(cufftSetStream(c2r_il, s));
        CKF(cufftExecC2C(c2r_il, at<cufftComplex>(ctx, L.proj), (cufftComplex *)dldi, CUFFT_INVERSE));
      } else {
        float *raw = at<float>(ctx, L.proj);
        CKF(cufftExecC2R(c2r, (cufftComplex *)sh, (cufftReal *)raw));
        launch_dldi_pack(c, nb, raw, dldi, s, ctx->launches);
        CK(cudaGetLastError());
      }
    }
    if (ctx->fused) {
      {
        Prof p(ctx, s, P_RENDER_BWD);
        launch_render_bwd(c, nb, rec, dldi, rw, at<float>(ctx, L.slots), s, ctx->launches);
        CK(cudaGetLastError());
      }
      Prof p(ctx, s, P_BWD_REDUCE);
      launch_bwd_reduce(c, nb, at<float>(ctx, L.slots), (const float4 *)params->mean_rho, acc, s, ctx->launches);
      CK(cudaGetLastError());
    }
  }
  if (host) CK(cudaEventRecord(ctx->ev_obs_free[h], ctx->side));   // its images' R2Cs are enqueued above
  ctx->last_p0 = p0 - ctx->W;
  ctx->last_nb = nb;
  // the per-particle loss reduction (and the host copy of the loss) runs on the side stream,
  // overlapped with the last C2R; the caller's stream joins it before anything that follows
  double *lossd = host ? at<double>(ctx, L.stage_loss) : loss;
  CK(cudaStreamWaitEvent(ctx->side, ctx->ev_ctf, 0));
  { Prof p(ctx, ctx->side, P_CTF_LOSS); launch_loss_reduce(B, lpart, L.loss_blocks, lossd, st, at<int>(ctx, L.ticket) + 4, ctx->side, ctx->launches); CK(cudaGetLastError()); }
  if (host) CK(cudaMemcpyAsync(loss, lossd, sizeof(double) * (B + 1), cudaMemcpyDeviceToHost, ctx->side));
  CK(cudaEventRecord(ctx->ev_loss, ctx->side));
  CK(cudaStreamWaitEvent(s, ctx->ev_loss, 0));
  CK(cudaGetLastError());
  ctx->fwd_live = 1;
  ctx->last_B = B;
  return GEM_OK;
}

gem_status gem_backward(gem_ctx *ctx, const gem_soa *params, gem_soa *grad, gem_stream_t stream) {
  NvtxCall nvtx_("gem_backward");
  if (!ctx || !soa_ok(params) || !soa_ok(grad)) return GEM_E_INVALID;
  if (!soa_aligned(params) || !soa_aligned(grad)) return GEM_E_ALIGN;
  if (!ctx->fwd_live) return GEM_E_STATE;
  cudaStream_t s = (cudaStream_t)stream;
  ctx->stream = s;
  ctx->launches = 0;
  const CfgDev &c = ctx->dc;
  const Layout &L = ctx->L;
  float4 *acc = at<float4>(ctx, L.acc);
  if (!ctx->fused) {   // one batch: backward, then chunk sums reduced and finalized in one kernel
    {
      Prof p(ctx, s, P_RENDER_BWD);
      launch_render_bwd(c, ctx->last_B, at<SplatRec>(ctx, L.rec), at<float>(ctx, L.dldi), ctx->rot_cur,
                        at<float>(ctx, L.slots), s, ctx->launches);
      CK(cudaGetLastError());
    }
    Prof p(ctx, s, P_BWD_REDUCE);
    launch_reduce_finalize(c, ctx->last_B, at<float>(ctx, L.slots), at<GaussPrep>(ctx, L.prep), (const float4 *)params->mean_rho,
                           (const float4 *)params->log_scale, (const float4 *)params->quat, (float4 *)grad->mean_rho,
                           (float4 *)grad->log_scale, (float4 *)grad->quat, at<DevStats>(ctx, L.stats), s,
                           ctx->launches);
    CK(cudaGetLastError());
  } else {   // fused mode: the forward already reduced every wave into acc
    Prof pf(ctx, s, P_FINALIZE);
    launch_finalize(c, acc, at<GaussPrep>(ctx, L.prep), (const float4 *)params->mean_rho, (const float4 *)params->log_scale,
                    (const float4 *)params->quat, (float4 *)grad->mean_rho, (float4 *)grad->log_scale,
                    (float4 *)grad->quat, at<DevStats>(ctx, L.stats), s, ctx->launches);
    CK(cudaGetLastError());
  }
  CK(cudaGetLastError());
  return GEM_OK;
}

gem_status gem_step(gem_ctx *ctx, gem_soa *params, const gem_soa *grad, gem_soa *m, gem_soa *v, int64_t t,
                    gem_stream_t stream) {
  NvtxCall nvtx_("gem_step");
  if (!ctx || !soa_ok(params) || !soa_ok(grad) || !soa_ok(m) || !soa_ok(v) || t < 1) return GEM_E_INVALID;
  if (!soa_aligned(params) || !soa_aligned(grad) || !soa_aligned(m) || !soa_aligned(v)) return GEM_E_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  ctx->stream = s;
  ctx->launches = 0;
  const gem_config &c = ctx->cfg;
  const double bc1 = 1.0 - std::pow((double)c.beta1, (double)t), bc2 = 1.0 - std::pow((double)c.beta2, (double)t);
  Prof pa(ctx, s, P_ADAM);
  launch_adam(ctx->dc.N, (float4 *)params->mean_rho, (float4 *)params->log_scale, (float4 *)params->quat,
              (const float4 *)grad->mean_rho, (const float4 *)grad->log_scale, (const float4 *)grad->quat,
              (float4 *)m->mean_rho, (float4 *)m->log_scale, (float4 *)m->quat, (float4 *)v->mean_rho,
              (float4 *)v->log_scale, (float4 *)v->quat, c.lr_mean, c.lr_log_scale, c.lr_quat, c.lr_density, c.beta1,
              c.beta2, c.eps, (float)bc1, (float)bc2, (int)c.flags, s, ctx->launches);
  CK(cudaGetLastError());
  return GEM_OK;
}

size_t gem_volume_scratch_bytes(const gem_ctx *ctx, int32_t Dv, float voxel_size) {
  (void)voxel_size;
  if (!ctx || Dv < 2) return 0;
  return volume_scratch_bytes(ctx->dc.N, Dv);
}

gem_status gem_render_volume(gem_ctx *ctx, const gem_soa *params, int32_t Dv, float voxel_size, float *vol_out,
                             void *scratch, size_t scratch_bytes, gem_stream_t stream) {
  NvtxCall nvtx_("gem_render_volume");
  if (!ctx || !soa_ok(params) || !vol_out || Dv < 2 || Dv > 4096 || !(voxel_size > 0.f)) return GEM_E_INVALID;
  if (!soa_aligned(params)) return GEM_E_ALIGN;
  const size_t need = volume_scratch_bytes(ctx->dc.N, Dv);
  char *sc = (char *)scratch;
  if (!sc) {
    sc = ctx->ws;
    scratch_bytes = ctx->ws_bytes;
    ctx->fwd_live = 0;  // the step workspace is reused
  }
  if (scratch_bytes < need) return GEM_E_SHAPE;
  if (((uintptr_t)sc & 255u) != 0) return GEM_E_ALIGN;
  cudaStream_t s = (cudaStream_t)stream;
  ctx->stream = s;
  ctx->launches = 0;
  DevStats *dst = nullptr;
  cudaError_t e;
  {
    Prof pv(ctx, s, P_VOLUME);   // device time of the query (the overflow check below syncs)
    e = launch_volume(ctx->dc.N, (const float4 *)params->mean_rho, (const float4 *)params->log_scale,
                      (const float4 *)params->quat, Dv, voxel_size, ctx->cfg.cull_k, vol_out, sc, scratch_bytes, s,
                      ctx->launches, &dst);
  }
  if (e != cudaSuccess) return GEM_E_CUDA;
  DevStats h;
  if (cudaMemcpyAsync(&h, dst, sizeof(DevStats), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return GEM_E_CUDA;
  if (h.overflow) return GEM_E_CAPACITY;
  return GEM_OK;
}

gem_status gem_export_lists(gem_ctx *ctx, int32_t particle, int32_t *tile_off, int32_t *ids, int64_t ids_cap,
                            int32_t *aabb) {
  if (!ctx) return GEM_E_INVALID;
  if (!ctx->fwd_live) return GEM_E_STATE;
  if (particle < 0 || particle >= ctx->last_B) return GEM_E_SHAPE;
  if (particle < ctx->last_p0 || particle >= ctx->last_p0 + ctx->last_nb) return GEM_E_STATE;  // not resident
  particle -= ctx->last_p0;
  CK(cudaStreamSynchronize(ctx->stream));
  const CfgDev &c = ctx->dc;
  const Layout &L = ctx->L;
  // list (particle, t) = ids[lst[particle NT + t] .. lst[particle NT + t + 1])
  int *hb = (int *)malloc(sizeof(int) * (c.NT + 1));
  if (!hb) return GEM_E_INVALID;
  if (cudaMemcpy(hb, at<int>(ctx, L.lst) + (size_t)particle * c.NT, sizeof(int) * (c.NT + 1), cudaMemcpyDeviceToHost) !=
      cudaSuccess) {
    free(hb);
    return GEM_E_CUDA;
  }
  const int start = hb[0];
  if (tile_off)
    for (int t = 0; t <= c.NT; ++t) tile_off[t] = hb[t] - start;
  const int64_t end = hb[c.NT];
  free(hb);
  if (ids) {
    int64_t n = end - start;
    if (n > ids_cap) n = ids_cap;
    if ((int64_t)start + n > c.cap) n = c.cap - start;
    if (n > 0)
      CK(cudaMemcpy(ids, at<int>(ctx, L.ids) + start, sizeof(int) * n, cudaMemcpyDeviceToHost));
  }
  if (aabb) {
    uint2 *hbx = (uint2 *)malloc(sizeof(uint2) * c.N);
    if (!hbx) return GEM_E_INVALID;
    if (cudaMemcpy(hbx, at<uint2>(ctx, L.box) + (size_t)particle * c.N, sizeof(uint2) * c.N, cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
      free(hbx);
      return GEM_E_CUDA;
    }
    for (int j = 0; j < c.N; ++j) {
      aabb[4 * j] = (int)(hbx[j].x & 0xffff);
      aabb[4 * j + 1] = (int)(short)(hbx[j].x >> 16);
      aabb[4 * j + 2] = (int)(hbx[j].y & 0xffff);
      aabb[4 * j + 3] = (int)(short)(hbx[j].y >> 16);
    }
    free(hbx);
  }
  return GEM_OK;
}

gem_status gem_stats(gem_ctx *ctx, gem_stats_t *out) {
  if (!ctx || !out) return GEM_E_INVALID;
  CK(cudaStreamSynchronize(ctx->stream));
  DevStats h;
  CK(cudaMemcpy(&h, ctx->ws + ctx->L.stats, sizeof(DevStats), cudaMemcpyDeviceToHost));
  // sticky overflow word (ticket[12], set by the scan of any forward since the last call)
  int sticky = 0;
  CK(cudaMemcpy(&sticky, ctx->ws + ctx->L.ticket + 12 * sizeof(int), sizeof(int), cudaMemcpyDeviceToHost));
  if (sticky) CK(cudaMemset(ctx->ws + ctx->L.ticket + 12 * sizeof(int), 0, sizeof(int)));
  h.overflow |= sticky;
  out->entries = (int64_t)h.entries;
  out->capacity = ctx->dc.cap;
  out->degenerate = h.degenerate;
  out->overflow = h.overflow;
  out->nonfinite = h.nonfinite;
  out->batch = ctx->last_B;
  out->workspace_bytes = (int64_t)ctx->ws_bytes;
  out->pairs = (int64_t)h.pairs;
  out->wave = ctx->W;
  out->fused = ctx->fused;
  if (h.overflow) return GEM_E_CAPACITY;
  if (h.nonfinite) return GEM_E_NONFINITE;
  return GEM_OK;
}

}  // extern "C"
