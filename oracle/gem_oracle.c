/*
 * gem_oracle.c — plain, slow fp64 CPU oracle for one GEM training step.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may link, load or call
 * this file: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg use it.  It shares no code, header, table or constant
 * generator with the CUDA library (paper_2509_25075_b200/csrc).
 *
 * Citations: "P:L" = PAPER.md line L (arXiv 2509.25075, GEM), "S:L" = SPEC.md
 * line L; "O<n>"/"L<n>" = the oracle steps / ledger readings of SURVEY.md §8(c),
 * restated in DESIGN.md §3.
 *
 * Every routine is a direct transcription of a definition: no tiling, no
 * culling lists used for arithmetic, no reordering.  All arithmetic is double.
 * Compile with -ffp-contract=off (no FMA contraction) so that the O3 bound
 * expressions evaluate exactly left-to-right as written.
 *
 * Layouts (inputs are the fp32 bytes the GPU receives, promoted to double):
 *   mean_rho [N][4] = (mu_x, mu_y, mu_z, rho)        mu in Angstrom
 *   log_scale[N][4] = (s0, s1, s2, pad)               sigma_k = exp(s_k), Angstrom
 *   quat     [N][4] = (w, x, y, z)
 *   rot      [B][9] = particle rotation P_i row-major; world->camera W = P_i^T (L8)
 *   shift    [B][2] = in-plane translation t_i, Angstrom
 *   ctf      [B][8] = du, dv (A), astig angle (rad), kV, Cs (mm), amp contrast,
 *                     phase shift (rad), B-factor (A^2)
 *   images   [B][D][D] row-major [v][u]; pixel (u,v) centre at
 *                     x = (u - D/2) px, y = (v - D/2) px          (L7)
 *   grad     [N][12] = (dmu_x, dmu_y, dmu_z, drho, ds0, ds1, ds2, 0, dqw, dqx, dqy, dqz)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_SQRT_2PI 2.5066282746310002 /* sqrt(2*pi) to double precision */
#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ O1 ---
 * Per Gaussian (Eq. 4): q_hat = q/|q|, R = R(q_hat),
 * sigma_k^2 = exp(2 s_k), Sigma = R diag(sigma^2) R^T, |Sigma| = exp(2(s0+s1+s2)).
 * Returns 0 if degenerate (|q| = 0 or non-finite; L18).  Op order = O3 rule. */
int orc_gauss(const double q[4], const double s[3], double R[9], double Sig[6],
              double *detS, double *qnorm, double qhat[4]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double n = sqrt(((w * w + x * x) + y * y) + z * z);
  *qnorm = n;
  if (!(n > 0.0) || !isfinite(n)) return 0;
  w = w / n; x = x / n; y = y / n; z = z / n;
  qhat[0] = w; qhat[1] = x; qhat[2] = y; qhat[3] = z;
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
  double s2[3];
  for (int k = 0; k < 3; ++k) s2[k] = exp(2.0 * s[k]);
  /* Sigma_kl = ((R_k0 s2_0) R_l0 + (R_k1 s2_1) R_l1) + (R_k2 s2_2) R_l2 ;
   * unique entries stored as (00, 01, 02, 11, 12, 22). */
  static const int KL[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  for (int e = 0; e < 6; ++e) {
    int k = KL[e][0], l = KL[e][1];
    Sig[e] = ((R[3 * k + 0] * s2[0]) * R[3 * l + 0] + (R[3 * k + 1] * s2[1]) * R[3 * l + 1]) +
             (R[3 * k + 2] * s2[2]) * R[3 * l + 2];
  }
  *detS = exp(2.0 * ((s[0] + s[1]) + s[2]));
  return isfinite(*detS) && isfinite(Sig[0]) && isfinite(Sig[3]) && isfinite(Sig[5]);
}

static double sig_at(const double Sig[6], int k, int l) {
  static const int IDX[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return Sig[IDX[k][l]];
}

/* ---------------------------------------------------------------- O2/O3 ---
 * Per (particle i, Gaussian j): pose, marginalise along camera z (App. A.2,
 * P:486-503, J = I for parallel rays P:498), exact marginal amplitude
 * amp = rho sqrt(2 pi) sqrt(|Sigma| / det2) (reading L1), conic
 * K = Sigma_hat^{-1}, and the integer AABB of the k-sigma ellipse in pixel
 * index space (reading L6; O3 canonical op order, no contraction). */
typedef struct {
  double mx, my, mz;     /* posed centre, Angstrom (camera frame)          */
  double A, B, C;        /* Sigma_hat = [[A,B],[B,C]], Angstrom^2            */
  double det2;           /* |Sigma_hat|                                      */
  double a, b, c;        /* conic K = Sigma_hat^{-1}, Angstrom^-2            */
  double amp;            /* exact marginal amplitude                         */
  double ampfac;         /* sqrt(2 pi) sqrt(|Sigma|/det2) = d amp / d rho    */
  int ulo, uhi, vlo, vhi;/* clipped integer AABB (inclusive)                 */
  int visible;
} orc_splat_t;

static int clip_int(double v, int lo, int hi) { /* v already an integer value or +-inf */
  if (!(v >= (double)lo)) return lo; /* also catches NaN */
  if (v > (double)hi) return hi;
  return (int)v;
}

void orc_splat(const double P[9], const double t[2], const double mu[3], const double Sig[6],
               double detS, double rho, int gauss_ok, double px, int D, double k, double tau,
               orc_splat_t *o) {
  memset(o, 0, sizeof(*o));
  /* W = P^T : W_rk = P_kr */
  double W[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) W[3 * r + c] = P[3 * c + r];
  o->mx = ((W[0] * mu[0] + W[1] * mu[1]) + W[2] * mu[2]) + t[0];
  o->my = ((W[3] * mu[0] + W[4] * mu[1]) + W[5] * mu[2]) + t[1];
  o->mz = (W[6] * mu[0] + W[7] * mu[1]) + W[8] * mu[2];
  double v0[3], v1[3];
  for (int kk = 0; kk < 3; ++kk) {
    v0[kk] = (sig_at(Sig, kk, 0) * W[0] + sig_at(Sig, kk, 1) * W[1]) + sig_at(Sig, kk, 2) * W[2];
    v1[kk] = (sig_at(Sig, kk, 0) * W[3] + sig_at(Sig, kk, 1) * W[4]) + sig_at(Sig, kk, 2) * W[5];
  }
  o->A = (W[0] * v0[0] + W[1] * v0[1]) + W[2] * v0[2];
  o->B = (W[0] * v1[0] + W[1] * v1[1]) + W[2] * v1[2];
  o->C = (W[3] * v1[0] + W[4] * v1[1]) + W[5] * v1[2];
  o->det2 = o->A * o->C - o->B * o->B;
  o->ampfac = ORC_SQRT_2PI * sqrt(detS / o->det2);
  o->amp = rho * o->ampfac;
  o->a = o->C / o->det2;
  o->b = -o->B / o->det2;
  o->c = o->A / o->det2;
  int ok = gauss_ok && isfinite(o->mx) && isfinite(o->my) && isfinite(o->A) && isfinite(o->C) &&
           isfinite(o->det2) && o->det2 > 0.0 && isfinite(o->amp);
  if (!ok) { o->visible = 0; o->ulo = 1; o->uhi = 0; o->vlo = 1; o->vhi = 0; return; }
  double rx = k * sqrt(o->A), ry = k * sqrt(o->C);
  double half = (double)(D / 2);
  double ulo = ceil((o->mx - rx) / px + half), uhi = floor((o->mx + rx) / px + half);
  double vlo = ceil((o->my - ry) / px + half), vhi = floor((o->my + ry) / px + half);
  o->ulo = clip_int(ulo, 0, D - 1 + 1);  /* clip to [0, D-1]; values outside -> empty */
  o->uhi = clip_int(uhi, -1, D - 1);
  o->vlo = clip_int(vlo, 0, D - 1 + 1);
  o->vhi = clip_int(vhi, -1, D - 1);
  o->visible = (fabs(o->amp) > tau) && (o->ulo <= o->uhi) && (o->vlo <= o->vhi);
}

/* Helper shared by the batch routines below: O1 for every Gaussian. */
typedef struct {
  double R[9], Sig[6], detS, qn, qhat[4];
  int ok;
} orc_gauss_t;

/* O1 for all Gaussians.  Reading L18: a Gaussian is degenerate (skipped in every pair, zero
 * gradient row, counted) if |q| = 0 or anything it is made of is non-finite: q, Sigma, |Sigma|
 * (orc_gauss) and also its centre mu and density rho, which reach every pair through m and amp. */
static orc_gauss_t *prep_all(int N, const double *mean_rho, const double *quat, const double *log_scale) {
  orc_gauss_t *g = (orc_gauss_t *)calloc((size_t)N, sizeof(orc_gauss_t));
  for (int j = 0; j < N; ++j) {
    g[j].ok = orc_gauss(quat + 4 * j, log_scale + 4 * j, g[j].R, g[j].Sig, &g[j].detS, &g[j].qn,
                        g[j].qhat);
    const double *m = mean_rho + 4 * j;
    if (!(isfinite(m[0]) && isfinite(m[1]) && isfinite(m[2]) && isfinite(m[3]))) g[j].ok = 0;
  }
  return g;
}

/* O2/O3 for all (i, j).  aabb [B][N][4] = (ulo, uhi, vlo, vhi), visible [B][N],
 * splat [B][N][10] = (mx, my, mz, a, b, c, amp, det2, A, C) — any output may be NULL. */
void orc_splats(int N, int B, const double *mean_rho, const double *log_scale, const double *quat,
                const double *rot, const double *shift, int D, double px, double k, double tau,
                int32_t *aabb, int32_t *visible, double *splat) {
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
#pragma omp parallel for collapse(2) schedule(static)
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < N; ++j) {
      orc_splat_t s;
      orc_splat(rot + 9 * i, shift + 2 * i, mean_rho + 4 * j, g[j].Sig, g[j].detS, mean_rho[4 * j + 3],
                g[j].ok, px, D, k, tau, &s);
      size_t ij = (size_t)i * N + j;
      if (aabb) { aabb[4 * ij] = s.ulo; aabb[4 * ij + 1] = s.uhi; aabb[4 * ij + 2] = s.vlo; aabb[4 * ij + 3] = s.vhi; }
      if (visible) visible[ij] = s.visible;
      if (splat) {
        double *o = splat + 10 * ij;
        o[0] = s.mx; o[1] = s.my; o[2] = s.mz; o[3] = s.a; o[4] = s.b; o[5] = s.c;
        o[6] = s.amp; o[7] = s.det2; o[8] = s.A; o[9] = s.C;
      }
    }
  free(g);
}

/* ------------------------------------------------------------------ O4 ---
 * Tile lists (Eq. 8 selection as the AABB contract):
 * tiles T x T, row-major tile index tv*(ceil(D/T)) + tu;
 * list(i,t) = { j visible : floor(ulo/T) <= tu <= floor(uhi/T) and same for v },
 * ascending j.  Naive scan over every (tile, j).  tile_off [B][NT+1] is the
 * per-particle exclusive prefix of list lengths; ids is concatenated per
 * particle (particle i's lists start at ids + ids_base[i]).  Returns the total
 * number of entries, or -1 if it would exceed cap. */
long long orc_lists(int N, int B, int D, int T, const int32_t *aabb, const int32_t *visible,
                    int32_t *tile_off, int64_t *ids_base, int32_t *ids, long long cap) {
  int nt = (D + T - 1) / T, NT = nt * nt;
  long long total = 0;
  for (int i = 0; i < B; ++i) {
    ids_base[i] = total;
    int32_t cnt = 0;
    for (int t = 0; t < NT; ++t) {
      int tu = t % nt, tv = t / nt;
      tile_off[(size_t)i * (NT + 1) + t] = cnt;
      for (int j = 0; j < N; ++j) {
        size_t ij = (size_t)i * N + j;
        if (!visible[ij]) continue;
        const int32_t *bx = aabb + 4 * ij;
        if (bx[0] / T <= tu && tu <= bx[1] / T && bx[2] / T <= tv && tv <= bx[3] / T) {
          if (total + cnt >= cap) return -1;
          ids[total + cnt] = j;
          ++cnt;
        }
      }
    }
    tile_off[(size_t)i * (NT + 1) + NT] = cnt;
    total += cnt;
  }
  return total;
}

/* ----------------------------------------------------------------- O4m ---
 * Tile lists for the per-pixel selection variants ("exact ellipse-tile
 * intersection instead of the AABB"; reading L26): list(i,t) = { j visible : some pixel of
 * tile t inside AABB_ij is kept by pix_keep (Q <= k^2 and/or |amp| exp(-Q/2) >= tau) },
 * ascending j.  Brute force over the pixels of every tile x AABB intersection.  Same layout as
 * orc_lists.  Defined after pix_keep below (forward declaration). */
static int pix_keep(const orc_splat_t *s, double Q, int pixmask, double k, double tau);
long long orc_lists_pixmask(int N, int B, const double *mean_rho, const double *log_scale, const double *quat,
                            const double *rot, const double *shift, int D, double px, double k, double tau, int T,
                            int pixmask, int32_t *tile_off, int64_t *ids_base, int32_t *ids, long long cap) {
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
  orc_splat_t *sp = (orc_splat_t *)malloc((size_t)B * N * sizeof(orc_splat_t));
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < N; ++j)
      orc_splat(rot + 9 * i, shift + 2 * i, mean_rho + 4 * j, g[j].Sig, g[j].detS, mean_rho[4 * j + 3], g[j].ok, px,
                D, k, tau, &sp[(size_t)i * N + j]);
  int nt = (D + T - 1) / T, NT = nt * nt;
  double half = (double)(D / 2);
  long long total = 0;
  for (int i = 0; i < B; ++i) {
    ids_base[i] = total;
    int32_t cnt = 0;
    for (int t = 0; t < NT; ++t) {
      int tu = t % nt, tv = t / nt;
      tile_off[(size_t)i * (NT + 1) + t] = cnt;
      for (int j = 0; j < N; ++j) {
        const orc_splat_t *s = &sp[(size_t)i * N + j];
        if (!s->visible) continue;
        int u0 = s->ulo > tu * T ? s->ulo : tu * T, u1 = s->uhi < tu * T + T - 1 ? s->uhi : tu * T + T - 1;
        int v0 = s->vlo > tv * T ? s->vlo : tv * T, v1 = s->vhi < tv * T + T - 1 ? s->vhi : tv * T + T - 1;
        int keep = 0;
        for (int v = v0; v <= v1 && !keep; ++v)
          for (int u = u0; u <= u1 && !keep; ++u) {
            double dx = ((double)u - half) * px - s->mx, dy = ((double)v - half) * px - s->my;
            keep = pix_keep(s, s->a * dx * dx + 2.0 * s->b * dx * dy + s->c * dy * dy, pixmask, k, tau);
          }
        if (keep) {
          if (total + cnt >= cap) { free(sp); free(g); return -1; }
          ids[total + cnt] = j;
          ++cnt;
        }
      }
    }
    tile_off[(size_t)i * (NT + 1) + NT] = cnt;
    total += cnt;
  }
  free(sp);
  free(g);
  return total;
}

/* ------------------------------------------------------------------ O5 ---
 * Projection, Eq. 6 with the Eq. 8 selection as contracted:
 *   masked:   I(u,v) = sum_{j visible, (u,v) in AABB_ij} amp exp(-Q/2)
 *   unmasked: I(u,v) = sum_{j non-degenerate} amp exp(-Q/2)  (mask == 1)
 * Q = a dx^2 + 2 b dx dy + c dy^2, dx = x - m_x, dy = y - m_y (Angstrom),
 * every Gaussian at every pixel.  img [B][D][D].
 * Per-pixel selection variants (reading L26), bits of `masked` / `pixmask`:
 *   2  exact ellipse: the pixel also needs Q <= k^2 (inside the k-sigma ellipse, not only its box);
 *   4  per-pixel tau (Eq. 8 "G_j > tau" at the pixel): |amp| exp(-Q/2) >= tau. */
static int pix_keep(const orc_splat_t *s, double Q, int pixmask, double k, double tau) {
  if ((pixmask & 2) && !(Q <= k * k)) return 0;
  if ((pixmask & 4) && !(fabs(s->amp) * exp(-0.5 * Q) >= tau)) return 0;
  return 1;
}

void orc_project(int N, int B, const double *mean_rho, const double *log_scale, const double *quat,
                 const double *rot, const double *shift, int D, double px, double k, double tau,
                 int masked, double *img) {
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
  orc_splat_t *sp = (orc_splat_t *)malloc((size_t)B * N * sizeof(orc_splat_t));
#pragma omp parallel for collapse(2) schedule(static)
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < N; ++j)
      orc_splat(rot + 9 * i, shift + 2 * i, mean_rho + 4 * j, g[j].Sig, g[j].detS, mean_rho[4 * j + 3],
                g[j].ok, px, D, k, tau, &sp[(size_t)i * N + j]);
  double half = (double)(D / 2);
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int i = 0; i < B; ++i)
    for (int v = 0; v < D; ++v)
      for (int u = 0; u < D; ++u) {
        double x = ((double)u - half) * px, y = ((double)v - half) * px;
        double acc = 0.0;
        for (int j = 0; j < N; ++j) {
          const orc_splat_t *s = &sp[(size_t)i * N + j];
          int use;
          if (masked) use = s->visible && u >= s->ulo && u <= s->uhi && v >= s->vlo && v <= s->vhi;
          else use = g[j].ok && isfinite(s->amp) && s->det2 > 0.0;
          if (!use) continue;
          double dx = x - s->mx, dy = y - s->my;
          double Q = s->a * dx * dx + 2.0 * s->b * dx * dy + s->c * dy * dy;
          if (masked && !pix_keep(s, Q, masked, k, tau)) continue;
          acc += s->amp * exp(-0.5 * Q);
        }
        img[((size_t)i * D + v) * D + u] = acc;
      }
  free(sp);
  free(g);
}

/* Sampled pixels of particle 0 of the given pose (used for full-size sampled
 * parity): pix[n][2] = (u, v) -> out[n]; masked as in orc_project. */
void orc_project_pixels(int N, const double *mean_rho, const double *log_scale, const double *quat,
                        const double *rot, const double *shift, int D, double px, double k, double tau,
                        int masked, int npix, const int32_t *pix, double *out) {
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
  orc_splat_t *sp = (orc_splat_t *)malloc((size_t)N * sizeof(orc_splat_t));
#pragma omp parallel for schedule(static)
  for (int j = 0; j < N; ++j)
    orc_splat(rot, shift, mean_rho + 4 * j, g[j].Sig, g[j].detS, mean_rho[4 * j + 3], g[j].ok, px, D, k,
              tau, &sp[j]);
  double half = (double)(D / 2);
#pragma omp parallel for schedule(static)
  for (int n = 0; n < npix; ++n) {
    int u = pix[2 * n], v = pix[2 * n + 1];
    double x = ((double)u - half) * px, y = ((double)v - half) * px, acc = 0.0;
    for (int j = 0; j < N; ++j) {
      const orc_splat_t *s = &sp[j];
      int use;
      if (masked) use = s->visible && u >= s->ulo && u <= s->uhi && v >= s->vlo && v <= s->vhi;
      else use = g[j].ok && isfinite(s->amp) && s->det2 > 0.0;
      if (!use) continue;
      double dx = x - s->mx, dy = y - s->my;
      double Q = s->a * dx * dx + 2.0 * s->b * dx * dy + s->c * dy * dy;
      if (masked && !pix_keep(s, Q, masked, k, tau)) continue;
      acc += s->amp * exp(-0.5 * Q);
    }
    out[n] = acc;
  }
  free(sp);
  free(g);
}

/* ------------------------------------------------------------------ O6 ---
 * CTF on the unshifted D x D DFT grid (formula: reading L10, CTFFIND form;
 * Eq. 1 / Eq. 7 apply it in Fourier space, reading L11).
 * Electron wavelength: lambda = h / sqrt(2 m0 e V (1 + eV/(2 m0 c^2))).
 * Hermitian fix (reading L12): C(k) = mean of C_raw over the alias set of k, a
 * Nyquist component (k = D/2) taking both +-1/(2 px). */
double orc_wavelength_A(double kV) {
  const double h = 6.62607015e-34, m0 = 9.1093837015e-31, e = 1.602176634e-19, c = 299792458.0;
  double V = kV * 1000.0;
  return h / sqrt(2.0 * m0 * e * V * (1.0 + e * V / (2.0 * m0 * c * c))) * 1e10;
}

double orc_ctf_raw(const double p[8], double fx, double fy) {
  double du = p[0], dv = p[1], th = p[2], lam = orc_wavelength_A(p[3]), Cs = p[4] * 1e7;
  double alpha = p[5], phi = p[6], bfac = p[7];
  double s2 = fx * fx + fy * fy;
  double df = 0.5 * (du + dv);
  if (s2 > 0.0)
    df += 0.5 * (du - dv) * ((fx * fx - fy * fy) * cos(2.0 * th) + 2.0 * fx * fy * sin(2.0 * th)) / s2;
  double chi = ORC_PI * lam * df * s2 - 0.5 * ORC_PI * Cs * lam * lam * lam * s2 * s2 + phi;
  return -exp(-bfac * s2 / 4.0) * (sqrt(1.0 - alpha * alpha) * sin(chi) + alpha * cos(chi));
}

static int alias_set(int kidx, int D, double px, double f[2]) {
  if (2 * kidx == D) { f[0] = 1.0 / (2.0 * px); f[1] = -1.0 / (2.0 * px); return 2; }
  if (2 * kidx < D) f[0] = (double)kidx / ((double)D * px);
  else f[0] = (double)(kidx - D) / ((double)D * px);
  return 1;
}

void orc_ctf(const double p[8], int D, double px, double *Cgrid /* [D][D], [ky][kx] */) {
  for (int ky = 0; ky < D; ++ky)
    for (int kx = 0; kx < D; ++kx) {
      double fxs[2], fys[2];
      int nx = alias_set(kx, D, px, fxs), ny = alias_set(ky, D, px, fys);
      double acc = 0.0;
      for (int a = 0; a < nx; ++a)
        for (int b = 0; b < ny; ++b) acc += orc_ctf_raw(p, fxs[a], fys[b]);
      Cgrid[(size_t)ky * D + kx] = acc / (double)(nx * ny);
    }
}

/* ------------------------------------------------------------------ O7 ---
 * Separable O(D^3) 2D DFT, unnormalised forward F[ky][kx] = sum I[v][u]
 * exp(-2 pi i (ky v + kx u)/D); inverse has +i and 1/D^2.  Twiddles use the
 * exact index reduction (n k) mod D. */
void orc_dft2(int D, const double *re, const double *im, double *ore, double *oim, int inverse) {
  double *twc = (double *)malloc(sizeof(double) * D), *tws = (double *)malloc(sizeof(double) * D);
  double sgn = inverse ? 1.0 : -1.0;
  for (int m = 0; m < D; ++m) {
    twc[m] = cos(2.0 * ORC_PI * (double)m / (double)D);
    tws[m] = sgn * sin(2.0 * ORC_PI * (double)m / (double)D);
  }
  size_t DD = (size_t)D * D;
  double *tr = (double *)calloc(DD, sizeof(double)), *ti = (double *)calloc(DD, sizeof(double));
  /* along u (rows) */
  for (int v = 0; v < D; ++v)
    for (int kx = 0; kx < D; ++kx) {
      double sr = 0.0, si = 0.0;
      for (int u = 0; u < D; ++u) {
        int m = (int)(((long long)u * kx) % D);
        double xr = re[(size_t)v * D + u], xi = im ? im[(size_t)v * D + u] : 0.0;
        sr += xr * twc[m] - xi * tws[m];
        si += xr * tws[m] + xi * twc[m];
      }
      tr[(size_t)v * D + kx] = sr; ti[(size_t)v * D + kx] = si;
    }
  /* along v (columns) */
  double scale = inverse ? 1.0 / (double)DD : 1.0;
  for (int ky = 0; ky < D; ++ky)
    for (int kx = 0; kx < D; ++kx) {
      double sr = 0.0, si = 0.0;
      for (int v = 0; v < D; ++v) {
        int m = (int)(((long long)v * ky) % D);
        double xr = tr[(size_t)v * D + kx], xi = ti[(size_t)v * D + kx];
        sr += xr * twc[m] - xi * tws[m];
        si += xr * tws[m] + xi * twc[m];
      }
      ore[(size_t)ky * D + kx] = sr * scale; oim[(size_t)ky * D + kx] = si * scale;
    }
  free(tr); free(ti); free(twc); free(tws);
}

/* I_pred = IDFT(C . DFT(img)) (Eq. 7).  Returns max |Im| / max |Re|. */
double orc_apply_ctf(int D, const double *Cgrid, const double *img, double *out) {
  size_t DD = (size_t)D * D;
  double *fr = (double *)malloc(DD * sizeof(double)), *fi = (double *)malloc(DD * sizeof(double));
  double *orr = (double *)malloc(DD * sizeof(double)), *oi = (double *)malloc(DD * sizeof(double));
  orc_dft2(D, img, NULL, fr, fi, 0);
  for (size_t n = 0; n < DD; ++n) { fr[n] *= Cgrid[n]; fi[n] *= Cgrid[n]; }
  orc_dft2(D, fr, fi, orr, oi, 1);
  double mr = 0.0, mi = 0.0;
  for (size_t n = 0; n < DD; ++n) {
    out[n] = orr[n];
    if (fabs(orr[n]) > mr) mr = fabs(orr[n]);
    if (fabs(oi[n]) > mi) mi = fabs(oi[n]);
  }
  free(fr); free(fi); free(orr); free(oi);
  return mr > 0.0 ? mi / mr : mi;
}

/* -------------------------------------------------------------- O7-O10 ---
 * One forward + backward over a batch.
 *   proj   = masked projection (O5)                       [B][D][D]
 *   pred   = IDFT(C . DFT(proj))                           (Eq. 7)
 *   loss_i = sum_{u,v} (pred - obs)^2   (sum, reading L14)
 *   g_i    = dL/dproj = 2 IDFT(C . DFT(pred - obs))       (O8; C real & even)
 *   per (i,j) over masked pixels (O9), then pose-independent finalize (O10).
 * If frozen_aabb/frozen_vis are non-NULL the masks are taken from them instead
 * of recomputed ("differentiate what you compute" with masks frozen).
 * Outputs (any may be NULL except loss): loss[B], proj, pred, gimg [B][D][D],
 * grad [N][12], acc [N][10] (world accumulators L_rho, G_mu(3), G_Sigma(6)).
 * Returns total loss. */
double orc_loss_grad(int N, int B, const double *mean_rho, const double *log_scale, const double *quat,
                     const double *rot, const double *shift, const double *ctf, const double *obs, int D,
                     double px, double k, double tau, int pixmask, const int32_t *frozen_aabb,
                     const int32_t *frozen_vis, double *loss, double *proj_out, double *pred_out,
                     double *gimg_out, double *grad, double *acc_out) {
  size_t DD = (size_t)D * D;
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
  orc_splat_t *sp = (orc_splat_t *)malloc((size_t)B * N * sizeof(orc_splat_t));
#pragma omp parallel for collapse(2) schedule(static)
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < N; ++j) {
      size_t ij = (size_t)i * N + j;
      orc_splat(rot + 9 * i, shift + 2 * i, mean_rho + 4 * j, g[j].Sig, g[j].detS, mean_rho[4 * j + 3],
                g[j].ok, px, D, k, tau, &sp[ij]);
      if (frozen_aabb) {
        sp[ij].ulo = frozen_aabb[4 * ij]; sp[ij].uhi = frozen_aabb[4 * ij + 1];
        sp[ij].vlo = frozen_aabb[4 * ij + 2]; sp[ij].vhi = frozen_aabb[4 * ij + 3];
        sp[ij].visible = frozen_vis[ij];
      }
    }
  double half = (double)(D / 2);
  double *proj = (double *)calloc((size_t)B * DD, sizeof(double));
  /* O5 masked projection */
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int i = 0; i < B; ++i)
    for (int v = 0; v < D; ++v)
      for (int u = 0; u < D; ++u) {
        double x = ((double)u - half) * px, y = ((double)v - half) * px, a = 0.0;
        for (int j = 0; j < N; ++j) {
          const orc_splat_t *s = &sp[(size_t)i * N + j];
          if (!(s->visible && u >= s->ulo && u <= s->uhi && v >= s->vlo && v <= s->vhi)) continue;
          double dx = x - s->mx, dy = y - s->my;
          double Q = s->a * dx * dx + 2.0 * s->b * dx * dy + s->c * dy * dy;
          if (pixmask && !pix_keep(s, Q, pixmask, k, tau)) continue;
          a += s->amp * exp(-0.5 * Q);
        }
        proj[((size_t)i * D + v) * D + u] = a;
      }
  double *gim = (double *)calloc((size_t)B * DD, sizeof(double));
  double total = 0.0;
  /* O6-O8 per particle */
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
  for (int i = 0; i < B; ++i) {
    double *C = (double *)malloc(DD * sizeof(double)), *pred = (double *)malloc(DD * sizeof(double));
    double *res = (double *)malloc(DD * sizeof(double)), *tmp = (double *)malloc(DD * sizeof(double));
    orc_ctf(ctf + 8 * i, D, px, C);
    orc_apply_ctf(D, C, proj + (size_t)i * DD, pred);
    double L = 0.0;
    for (size_t n = 0; n < DD; ++n) {
      res[n] = pred[n] - obs[(size_t)i * DD + n];
      L += res[n] * res[n];
    }
    loss[i] = L;
    total += L;
    orc_apply_ctf(D, C, res, tmp);
    for (size_t n = 0; n < DD; ++n) gim[(size_t)i * DD + n] = 2.0 * tmp[n];
    if (pred_out) memcpy(pred_out + (size_t)i * DD, pred, DD * sizeof(double));
    free(C); free(pred); free(res); free(tmp);
  }
  /* O9: per (i,j) backward over masked pixels; world-frame accumulators */
  double *acc = (double *)calloc((size_t)N * 10, sizeof(double));
#pragma omp parallel for schedule(dynamic, 8)
  for (int j = 0; j < N; ++j) {
    double *aj = acc + 10 * (size_t)j;
    for (int i = 0; i < B; ++i) {
      const orc_splat_t *s = &sp[(size_t)i * N + j];
      if (!s->visible) continue;
      double La = 0, Lmx = 0, Lmy = 0, Lpa = 0, Lpb = 0, Lpc = 0;
      for (int v = 0; v < D; ++v)
        for (int u = 0; u < D; ++u) {
          if (!(u >= s->ulo && u <= s->uhi && v >= s->vlo && v <= s->vhi)) continue;
          double x = ((double)u - half) * px, y = ((double)v - half) * px;
          double dx = x - s->mx, dy = y - s->my;
          double Q = s->a * dx * dx + 2.0 * s->b * dx * dy + s->c * dy * dy;
          if (pixmask && !pix_keep(s, Q, pixmask, k, tau)) continue;
          double e = exp(-0.5 * Q);
          double gg = gim[((size_t)i * D + v) * D + u];
          double h = gg * s->amp * e;
          La += gg * e;
          Lmx += h * (s->a * dx + s->b * dy);
          Lmy += h * (s->b * dx + s->c * dy);
          Lpa += -0.5 * h * dx * dx;
          Lpb += -h * dx * dy;
          Lpc += -0.5 * h * dy * dy;
        }
      /* G_Sigma_hat = -K Gk K - 1/2 L_amp amp K,  Gk = [[La, Lb/2],[Lb/2, Lc]] */
      double K[2][2] = {{s->a, s->b}, {s->b, s->c}};
      double Gk[2][2] = {{Lpa, 0.5 * Lpb}, {0.5 * Lpb, Lpc}};
      double KG[2][2], Gh[2][2];
      for (int r = 0; r < 2; ++r)
        for (int c2 = 0; c2 < 2; ++c2) KG[r][c2] = K[r][0] * Gk[0][c2] + K[r][1] * Gk[1][c2];
      for (int r = 0; r < 2; ++r)
        for (int c2 = 0; c2 < 2; ++c2)
          Gh[r][c2] = -(KG[r][0] * K[0][c2] + KG[r][1] * K[1][c2]) - 0.5 * La * s->amp * K[r][c2];
      const double *P = rot + 9 * i;
      double W[9];
      for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) W[3 * r + c2] = P[3 * c2 + r];
      aj[0] += La * s->ampfac;                      /* L_rho */
      for (int c2 = 0; c2 < 3; ++c2) aj[1 + c2] += Lmx * W[c2] + Lmy * W[3 + c2]; /* W^T (Lmx, Lmy, 0) */
      static const int KL[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
      for (int e6 = 0; e6 < 6; ++e6) {           /* G_Sigma += W^T [[Gh,0],[0,0]] W */
        int kk = KL[e6][0], ll = KL[e6][1];
        double sum = 0.0;
        for (int a2 = 0; a2 < 2; ++a2)
          for (int b2 = 0; b2 < 2; ++b2) sum += W[3 * a2 + kk] * Gh[a2][b2] * W[3 * b2 + ll];
        aj[4 + e6] += sum;
      }
    }
  }
  /* O10 finalize (pose independent) */
  if (grad) {
    memset(grad, 0, sizeof(double) * 12 * (size_t)N);
    for (int j = 0; j < N; ++j) {
      double *gr = grad + 12 * (size_t)j;
      const double *aj = acc + 10 * (size_t)j;
      if (!g[j].ok) continue;
      double GS[3][3];
      static const int IDX[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
      for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) GS[r][c2] = aj[4 + IDX[r][c2]];
      const double *R = g[j].R;
      double s2[3];
      for (int kk = 0; kk < 3; ++kk) s2[kk] = exp(2.0 * log_scale[4 * j + kk]);
      gr[0] = aj[1]; gr[1] = aj[2]; gr[2] = aj[3];
      gr[3] = aj[0];
      double rho = mean_rho[4 * j + 3];
      for (int kk = 0; kk < 3; ++kk) { /* ds_k = 2 sigma_k^2 (R^T G R)_kk + rho L_rho */
        double q = 0.0;
        for (int a2 = 0; a2 < 3; ++a2)
          for (int b2 = 0; b2 < 3; ++b2) q += R[3 * a2 + kk] * GS[a2][b2] * R[3 * b2 + kk];
        gr[4 + kk] = 2.0 * s2[kk] * q + rho * aj[0];
      }
      /* dL/dR = 2 G R diag(sigma^2) */
      double dR[9];
      for (int m = 0; m < 3; ++m)
        for (int n = 0; n < 3; ++n) {
          double q = 0.0;
          for (int a2 = 0; a2 < 3; ++a2) q += GS[m][a2] * R[3 * a2 + n];
          dR[3 * m + n] = 2.0 * q * s2[n];
        }
      double w = g[j].qhat[0], x = g[j].qhat[1], y = g[j].qhat[2], z = g[j].qhat[3];
      const double dRw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
      const double dRx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
      const double dRy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
      const double dRz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
      double dqh[4] = {0, 0, 0, 0};
      for (int e9 = 0; e9 < 9; ++e9) {
        dqh[0] += dR[e9] * 2.0 * dRw[e9];
        dqh[1] += dR[e9] * 2.0 * dRx[e9];
        dqh[2] += dR[e9] * 2.0 * dRy[e9];
        dqh[3] += dR[e9] * 2.0 * dRz[e9];
      }
      /* dL/dq = (I - qh qh^T) dL/dqh / |q| */
      double dot = dqh[0] * w + dqh[1] * x + dqh[2] * y + dqh[3] * z;
      const double qh[4] = {w, x, y, z};
      for (int c2 = 0; c2 < 4; ++c2) gr[8 + c2] = (dqh[c2] - dot * qh[c2]) / g[j].qn;
    }
  }
  if (acc_out) memcpy(acc_out, acc, sizeof(double) * 10 * (size_t)N);
  if (proj_out) memcpy(proj_out, proj, sizeof(double) * (size_t)B * DD);
  if (gimg_out) memcpy(gimg_out, gim, sizeof(double) * (size_t)B * DD);
  free(acc); free(gim); free(proj); free(sp); free(g);
  return total;
}

/* ----------------------------------------------------------------- O11 ---
 * Adam (reading L15: PyTorch bias-corrected form), per scalar with its
 * class learning rate lr[4] = (mean, log_scale, quat, density); then
 * q <- q/|q| when |q| > 0.  Pad lane (log_scale.w) never updated.
 * params/grad/m/v: [3][N][4] = (mean_rho, log_scale, quat). */
void orc_adam(int N, double *params, const double *grad, double *m, double *v, long long t,
              const double lr[4], double b1, double b2, double eps) {
  double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  for (int arr = 0; arr < 3; ++arr)
    for (int j = 0; j < N; ++j)
      for (int c = 0; c < 4; ++c) {
        double l;
        if (arr == 0) l = (c < 3) ? lr[0] : lr[3];
        else if (arr == 1) { if (c == 3) continue; l = lr[1]; }
        else l = lr[2];
        size_t n = ((size_t)arr * N + j) * 4 + c;
        m[n] = b1 * m[n] + (1.0 - b1) * grad[n];
        v[n] = b2 * v[n] + (1.0 - b2) * grad[n] * grad[n];
        double mh = m[n] / bc1, vh = v[n] / bc2;
        params[n] = params[n] - l * mh / (sqrt(vh) + eps);
      }
  for (int j = 0; j < N; ++j) {
    double *q = params + ((size_t)2 * N + j) * 4;
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (n > 0.0) for (int c = 0; c < 4; ++c) q[c] /= n;
  }
}

/* ----------------------------------------------------------------- O12 ---
 * Density query on a Dv^3 grid (Eq. 5): voxel (a,b,c) centre
 * ((a - Dv/2) vs, (b - Dv/2) vs, (c - Dv/2) vs); V(x) = sum_j 1[x in AABB3_j]
 * rho_j exp(-1/2 d^T Sigma_j^{-1} d), AABB3 half-widths k sqrt(Sigma_xx) etc.
 * (O3 rules, integer voxel-index box).  masked = 0 gives the un-culled V.
 * vol [Dv][Dv][Dv] with x fastest: vol[(c*Dv + b)*Dv + a]. */
void orc_volume(int N, const double *mean_rho, const double *log_scale, const double *quat, int Dv,
                double vs, double k, int masked, double *vol) {
  orc_gauss_t *g = prep_all(N, mean_rho, quat, log_scale);
  double *inv = (double *)malloc(sizeof(double) * 9 * (size_t)N);
  int *box = (int *)malloc(sizeof(int) * 6 * (size_t)N);
  double half = (double)(Dv / 2);
  for (int j = 0; j < N; ++j) {
    double s2inv[3];
    for (int kk = 0; kk < 3; ++kk) s2inv[kk] = exp(-2.0 * log_scale[4 * j + kk]);
    const double *R = g[j].R;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        inv[9 * (size_t)j + 3 * r + c] =
            ((R[3 * r + 0] * s2inv[0]) * R[3 * c + 0] + (R[3 * r + 1] * s2inv[1]) * R[3 * c + 1]) +
            (R[3 * r + 2] * s2inv[2]) * R[3 * c + 2];
    for (int ax = 0; ax < 3; ++ax) {
      double r = k * sqrt(sig_at(g[j].Sig, ax, ax));
      double lo = ceil((mean_rho[4 * j + ax] - r) / vs + half), hi = floor((mean_rho[4 * j + ax] + r) / vs + half);
      box[6 * j + 2 * ax] = clip_int(lo, 0, Dv);
      box[6 * j + 2 * ax + 1] = clip_int(hi, -1, Dv - 1);
    }
  }
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
  for (int c = 0; c < Dv; ++c)
    for (int b = 0; b < Dv; ++b)
      for (int a = 0; a < Dv; ++a) {
        double x[3] = {((double)a - half) * vs, ((double)b - half) * vs, ((double)c - half) * vs};
        int idx[3] = {a, b, c};
        double accv = 0.0;
        for (int j = 0; j < N; ++j) {
          if (!g[j].ok) continue;
          if (masked) {
            int in = 1;
            for (int ax = 0; ax < 3; ++ax)
              if (idx[ax] < box[6 * j + 2 * ax] || idx[ax] > box[6 * j + 2 * ax + 1]) in = 0;
            if (!in) continue;
          }
          double d[3] = {x[0] - mean_rho[4 * j], x[1] - mean_rho[4 * j + 1], x[2] - mean_rho[4 * j + 2]};
          double Q = 0.0;
          for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) Q += d[r] * inv[9 * (size_t)j + 3 * r + cc] * d[cc];
          accv += mean_rho[4 * j + 3] * exp(-0.5 * Q);
        }
        vol[((size_t)c * Dv + b) * Dv + a] = accv;
      }
  free(box); free(inv); free(g);
}
