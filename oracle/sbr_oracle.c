/*
 * sbr_oracle.c -- CPU restatement of the emtrace SBR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * Pinning: every routine is checked against golden vectors produced by the
 * real reference (tests/golden/make_golden.py imports emtrace from
 * /root/reference in the build container) -- see tests/test_oracle_golden.py.
 *
 * The restatement is scalar per ray (the reference is numpy-vectorised per
 * segment) but keeps the reference's float64 operation order, including the
 * OpenBLAS FMA order of its `@` products, so results agree to the last bit
 * in the common case.  Compile WITHOUT -ffast-math and with
 * -ffp-contract=off.
 *
 * Reference anchors (all under /root/reference/pkg/src/emtrace/):
 *   philox stream    sampling.py:42-78        fibonacci   sampling.py:81-95
 *   SAH BVH build    geometry.py:244-349      traversal   _core.pyx:26-253
 *   slab Fresnel     materials.py:163-245     patterns    materials.py:354-397
 *   incidence frame  radiomap.py:291-300      map loop    radiomap.py:347-563
 *   direct term      radiomap.py:566-583      antenna     em.py:258-308,
 *                                                         radiomap.py:253-277
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/sbr.h"

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* Philox4x64-10 counter stream == numpy Philox + Generator.random           */
/* ------------------------------------------------------------------------- */

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

/* RngStream(seed, sample, depth, tag).generator().random(n)[i]
 * key = (seed, sample); counter = (i//4 + 1, 0, depth, tag_hash)
 * (sampling.py:74-78: counter = depth<<128 | tag<<192, Philox advances the
 * counter once before producing the first block). */
ORC_EXPORT double orc_philox_uniform(uint64_t seed, uint64_t sample, uint64_t depth,
                                     uint64_t tag, uint64_t i) {
  uint64_t blk = i / 4 + 1;
  uint64_t c0 = blk, c1 = 0, c2 = depth, c3 = tag;
  uint64_t k0 = seed, k1 = sample;
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  uint64_t w;
  switch (i & 3) {
    case 0: w = c0; break;
    case 1: w = c1; break;
    case 2: w = c2; break;
    default: w = c3; break;
  }
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

ORC_EXPORT uint64_t orc_tag_hash(const char* s) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (; *s; ++s) h = (h ^ (uint8_t)*s) * 0x100000001B3ULL;
  return h;
}

/* tag hashes (sampling.py:42-46 applied to the map purposes) */
#define TAG_MAP_INTERACTION 0xb89bb7c3608d55f4ULL
#define TAG_MAP_RESPAWN 0x123e3e11a6151f88ULL
#define TAG_MAP_PHASE 0xec7920a818db590bULL
#define TAG_MAP_ROULETTE 0xba18862d049a6e7cULL

/* ------------------------------------------------------------------------- */
/* Fibonacci lattice (sampling.py:81-95)                                     */
/* ------------------------------------------------------------------------- */
static const double GOLDEN = 1.618033988749895; /* (1+sqrt(5))/2 in f64 */
static const double TWO_PI = 6.283185307179586;
static const double FOUR_PI = 12.566370614359172;
static const double PI_ = 3.141592653589793;

ORC_EXPORT void orc_fibonacci(uint64_t N, uint64_t g, double out[3]) {
  double n = (double)((int64_t)g - (int64_t)(N / 2));
  double cos_t = 2.0 * n / (double)N;
  double x = 1.0 - cos_t * cos_t;
  double sin_t = sqrt(x > 0.0 ? x : 0.0);
  double phi = TWO_PI * n / GOLDEN;
  out[0] = sin_t * cos(phi);
  out[1] = sin_t * sin(phi);
  out[2] = cos_t;
}

/* ------------------------------------------------------------------------- */
/* Small vector helpers with numpy's evaluation order                        */
/* ------------------------------------------------------------------------- */
/* np.sum(a*b, axis=1) over 3 columns: sequential */
static inline double dot_seq(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
/* (n,3) @ (3,) through OpenBLAS dgemv (measured order) */
static inline double dot_gemv(const double* a, const double* b) {
  return fma(a[2], b[2], fma(a[0], b[0], a[1] * b[1]));
}
/* 1-D v @ w through ddot */
static inline double dot_ddot(const double* a, const double* b) {
  return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}
static inline void cross3(const double* a, const double* b, double* c) {
  double c0 = a[1] * b[2] - a[2] * b[1];
  double c1 = a[2] * b[0] - a[0] * b[2];
  double c2 = a[0] * b[1] - a[1] * b[0];
  c[0] = c0; c[1] = c1; c[2] = c2;
}
static inline double norm_seq(const double* a) {
  return sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
}

/* ------------------------------------------------------------------------- */
/* complex128 with numpy's algorithms                                        */
/* ------------------------------------------------------------------------- */
typedef struct { double re, im; } cpx;
static inline cpx C(double r, double i) { cpx z = {r, i}; return z; }
static inline cpx cadd(cpx a, cpx b) { return C(a.re + b.re, a.im + b.im); }
static inline cpx csub(cpx a, cpx b) { return C(a.re - b.re, a.im - b.im); }
static inline cpx cmul(cpx a, cpx b) {
  return C(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
static inline cpx cscale(double s, cpx a) { return C(s * a.re, s * a.im); }
/* numpy CDOUBLE_divide (Smith with reciprocal) */
static inline cpx cdiv(cpx a, cpx b) {
  double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return C(a.re / br, a.im / br);
    double rat = b.im / b.re;
    double scl = 1.0 / (b.re + b.im * rat);
    return C((a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl);
  }
  double rat = b.re / b.im;
  double scl = 1.0 / (b.im + b.re * rat);
  return C((a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl);
}
/* np.abs(complex128): numpy 2.x SIMD loop computes max*sqrt(fma(r,r,1)),
 * r = min/max (measured bit-exact against numpy 2.3 on 2e5 samples). */
static inline double cabs_(cpx a) {
  double x = fabs(a.re), y = fabs(a.im);
  double m = x > y ? x : y, k = x > y ? y : x;
  if (m == 0.0 || isinf(m)) return m + k;
  double r = k / m;
  return m * sqrt(fma(r, r, 1.0));
}
static inline double cabs2(cpx a) { double m = cabs_(a); return m * m; }
static inline cpx cexp_(cpx a) {
  double e = exp(a.re);
  return C(e * cos(a.im), e * sin(a.im));
}
/* principal square root, glibc csqrt's finite-argument branch (np.sqrt on
 * complex128 calls libm csqrt) */
static cpx csqrt_(cpx z) {
  double x = z.re, y = z.im;
  if (y == 0.0) {
    if (x < 0.0) return C(0.0, copysign(sqrt(-x), y));
    return C(fabs(sqrt(x)), copysign(0.0, y));
  }
  if (x == 0.0) {
    double r = sqrt(0.5 * fabs(y));
    return C(r, copysign(r, y));
  }
  double d = hypot(x, y), r, s;
  if (x > 0.0) {
    r = sqrt(0.5 * (d + x));
    s = 0.5 * (y / r);
  } else {
    s = sqrt(0.5 * (d - x));
    r = fabs(0.5 * (y / s));
  }
  return C(r, copysign(s, y));
}
/* _sqrt_lossy: branch with Im <= 0 (materials.py:163-170) */
static inline cpx csqrt_lossy(cpx z) {
  cpx s = csqrt_(z);
  if (s.im > 0.0) return C(-s.re, -s.im);
  return s;
}

/* ------------------------------------------------------------------------- */
/* Slab reflection / transmission (materials.py:173-245)                      */
/* ------------------------------------------------------------------------- */
typedef struct { cpx rp, rl, tp, tl; } Fresnel4;

static Fresnel4 slab_fresnel(const SbrMaterial* m, double c0) {
  Fresnel4 f;
  cpx eta = C(m->eta_re, m->eta_im);
  double sin2 = 1.0 - c0 * c0;
  cpx root = csqrt_lossy(C(eta.re - sin2, eta.im));
  cpx c_plus = C(c0 + root.re, root.im);
  cpx ec = C(eta.re * c0, eta.im * c0);
  cpx ec_plus = cadd(ec, root);
  cpx r_perp = cdiv(C(c0 - root.re, -root.im), c_plus);
  cpx r_par = cdiv(csub(ec, root), ec_plus);
  int total = (eta.im == 0.0) && (sin2 >= cabs_(eta));
  if (total) { r_perp = C(1.0, 0.0); r_par = C(1.0, 0.0); }
  if (m->thickness == 0.0) {
    f.rp = C(0.0, 0.0); f.rl = C(0.0, 0.0);
    f.tp = C(1.0, 0.0); f.tl = C(1.0, 0.0);
    return f;
  }
  cpx q = cscale(m->kd, root);
  /* -2j*q and -1j*q */
  cpx phase2 = cexp_(C(2.0 * q.im, -2.0 * q.re));
  cpx phase1 = cexp_(C(q.im, -q.re));
  cpx one_m_p2 = C(1.0 - phase2.re, -phase2.im);
  cpx r1s[2] = {r_perp, r_par};
  cpx rr[2], tt[2];
  for (int p = 0; p < 2; ++p) {
    cpx r1 = r1s[p];
    cpx r1sq = cmul(r1, r1);
    cpx z = cmul(r1sq, phase2);
    cpx denom = C(1.0 - z.re, -z.im);
    rr[p] = cdiv(cmul(r1, one_m_p2), denom);
    tt[p] = cdiv(cmul(C(1.0 - r1sq.re, -r1sq.im), phase1), denom);
  }
  f.rp = rr[0]; f.rl = rr[1]; f.tp = tt[0]; f.tl = tt[1];
  return f;
}

ORC_EXPORT void orc_slab_fresnel(const SbrMaterial* m, const double* cos_theta, int64_t n,
                                 double* out /* (n, 8) */) {
  for (int64_t i = 0; i < n; ++i) {
    Fresnel4 f = slab_fresnel(m, cos_theta[i]);
    double* o = out + 8 * i;
    o[0] = f.rp.re; o[1] = f.rp.im; o[2] = f.rl.re; o[3] = f.rl.im;
    o[4] = f.tp.re; o[5] = f.tp.im; o[6] = f.tl.re; o[7] = f.tl.im;
  }
}

/* scattering_pattern_eval (materials.py:354-397) */
static double binom(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
  return floor(r + 0.5);
}
static double lobe_norm(int alpha, double cos_ti) {
  double sin2 = 1.0 - cos_ti * cos_ti;
  if (sin2 < 0.0) sin2 = 0.0;
  double total = 0.0;
  for (int k = 0; k <= alpha; ++k) {
    double ik;
    if (k % 2 == 0) {
      ik = TWO_PI / (double)(k + 1);
    } else {
      double inner = 0.0;
      for (int w = 0; w <= (k - 1) / 2; ++w)
        inner = inner + binom(2 * w, w) * pow(sin2 / 4.0, (double)w);
      ik = TWO_PI / (double)(k + 1) * cos_ti * inner;
    }
    total = total + binom(alpha, k) * ik;
  }
  return total / pow(2.0, (double)alpha);
}
static double pattern_density(const SbrMaterial* m, const double* ki, const double* ks,
                              const double* n) {
  if (m->pattern_kind == SBR_SCAT_LAMBERTIAN) {
    double c = dot_seq(ks, n);
    c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
    return c / PI_;
  }
  double ci = -dot_seq(ki, n);
  ci = ci < -1.0 ? -1.0 : (ci > 1.0 ? 1.0 : ci);
  double kn = dot_seq(ki, n);
  double kr[3] = {ki[0] - 2.0 * kn * n[0], ki[1] - 2.0 * kn * n[1], ki[2] - 2.0 * kn * n[2]};
  double lobe_r = pow((1.0 + dot_seq(kr, ks)) / 2.0, (double)m->alpha_r);
  if (m->pattern_kind == SBR_SCAT_DIRECTIVE) return lobe_r / lobe_norm(m->alpha_r, ci);
  double lobe_i = pow((1.0 - dot_seq(ki, ks)) / 2.0, (double)m->alpha_i);
  double lam = m->lambda_mix;
  double nrm = lam * lobe_norm(m->alpha_r, ci) + (1.0 - lam) * lobe_norm(m->alpha_i, ci);
  return (lam * lobe_r + (1.0 - lam) * lobe_i) / nrm;
}

/* ------------------------------------------------------------------------- */
/* Antenna pattern -> world field (radiomap.py:266-277, em.py:263-288)       */
/* ------------------------------------------------------------------------- */
static void transverse(const double* d, double th[3], double ph[3]) {
  double z = d[2] < -1.0 ? -1.0 : (d[2] > 1.0 ? 1.0 : d[2]);
  double theta = acos(z), phi = atan2(d[1], d[0]);
  double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
  th[0] = ct * cp; th[1] = ct * sp; th[2] = -st;
  ph[0] = -sp; ph[1] = cp; ph[2] = 0.0;
}

static double tr38901_amp(double scale, double theta, double phi) {
  double theta_deg = theta * (180.0 / PI_);
  double phi_deg = atan2(sin(phi), cos(phi)) * (180.0 / PI_);
  double a = (theta_deg - 90.0) / 65.0;
  double av = 12.0 * (a * a);
  av = -(av < 30.0 ? av : 30.0);
  double b = phi_deg / 65.0;
  double ah = 12.0 * (b * b);
  ah = -(ah < 30.0 ? ah : 30.0);
  double s = -(av + ah);
  double g = -(s < 30.0 ? s : 30.0) + 8.0;
  return scale * pow(10.0, g / 20.0);
}

/* rows @ R (dgemm, we use the dgemv order) */
static void mat_t_vec(const double* R, const double* d, double* out) {
  /* out_k = sum_j d_j R[j][k] */
  for (int k = 0; k < 3; ++k) {
    double col[3] = {R[0 * 3 + k], R[1 * 3 + k], R[2 * 3 + k]};
    out[k] = dot_gemv(d, col);
  }
}
static void mat_vec(const double* R, const double* v, double* out) {
  /* (v @ R.T)_k = sum_j v_j R[k][j] */
  for (int k = 0; k < 3; ++k) out[k] = dot_gemv(v, R + 3 * k);
}

static void pattern_field(const SbrAntenna* a, const double* d, cpx E[3]) {
  double local[3];
  if (a->identity) { local[0] = d[0]; local[1] = d[1]; local[2] = d[2]; }
  else mat_t_vec(a->rot, d, local);
  double z = local[2] < -1.0 ? -1.0 : (local[2] > 1.0 ? 1.0 : local[2]);
  double theta = acos(z), phi = atan2(local[1], local[0]);
  double cth = 1.0;
  if (a->kind == SBR_PATTERN_TR38901) cth = tr38901_amp(a->scale, theta, phi);
  double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
  double th_l[3] = {ct * cp, ct * sp, -st}, ph_l[3] = {-sp, cp, 0.0};
  double th[3], ph[3];
  if (a->identity) { memcpy(th, th_l, sizeof th); memcpy(ph, ph_l, sizeof ph); }
  else { mat_vec(a->rot, th_l, th); mat_vec(a->rot, ph_l, ph); }
  (void)ph;
  for (int k = 0; k < 3; ++k) E[k] = C(cth * th[k], 0.0);
}

static double alpha_sq(const SbrMapParams* p, const double* offs, const double* prec,
                       const double* d) {
  if (p->n_elements <= 0) return 1.0;
  double k = TWO_PI / p->wavelength;
  cpx acc = C(0.0, 0.0);
  for (int m = 0; m < p->n_elements; ++m) {
    double ph = k * dot_gemv(d, offs + 3 * m);
    cpx e = C(cos(ph), sin(ph));
    acc = cadd(acc, cmul(e, C(prec[2 * m], prec[2 * m + 1])));
  }
  return cabs2(acc);
}

/* ------------------------------------------------------------------------- */
/* BVH: binned SAH restated from geometry.py:244-349                         */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t ntri;
  const double *v0, *v1, *v2;     /* input order */
  double *lo, *hi, *cen;          /* (ntri,3) */
  double *bmin, *bmax;            /* (2*ntri,3) nodes */
  int32_t *right, *start, *count;
  int64_t *perm;
  int64_t nnodes, out_pos;
  int64_t *tmp;
} Builder;

static int64_t new_node(Builder* B, const double* lo, const double* hi) {
  int64_t me = B->nnodes++;
  for (int k = 0; k < 3; ++k) {
    B->bmin[3 * me + k] = lo[k] - 1e-12 * (1.0 + fabs(lo[k]));
    B->bmax[3 * me + k] = hi[k] + 1e-12 * (1.0 + fabs(hi[k]));
  }
  B->right[me] = -1; B->start[me] = -1; B->count[me] = 0;
  return me;
}

static double half_area(const double* lo, const double* hi) {
  double e[3];
  for (int k = 0; k < 3; ++k) { e[k] = hi[k] - lo[k]; if (e[k] < 0.0) e[k] = 0.0; }
  return e[0] * e[1] + e[1] * e[2] + e[2] * e[0];
}

typedef struct { double k; int64_t pos; int64_t id; } KP;
static int cmp_kp(const void* x, const void* y) {
  const KP* a = (const KP*)x;
  const KP* b = (const KP*)y;
  if (a->k < b->k) return -1;
  if (a->k > b->k) return 1;
  return (a->pos > b->pos) - (a->pos < b->pos);
}

#define NB 16
static int64_t build_rec(Builder* B, int64_t* idx, int64_t n) {
  double blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      double l = B->lo[3 * idx[i] + k], h = B->hi[3 * idx[i] + k];
      if (l < blo[k]) blo[k] = l;
      if (h > bhi[k]) bhi[k] = h;
    }
  int64_t me = new_node(B, blo, bhi);
  if (n <= 4) {
    B->start[me] = (int32_t)B->out_pos;
    B->count[me] = (int32_t)n;
    for (int64_t i = 0; i < n; ++i) B->perm[B->out_pos++] = idx[i];
    return me;
  }
  double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      double c = B->cen[3 * idx[i] + k];
      if (c < clo[k]) clo[k] = c;
      if (c > chi[k]) chi[k] = c;
    }
  int axis = 0;
  double ext0 = chi[0] - clo[0];
  for (int k = 1; k < 3; ++k) if (chi[k] - clo[k] > ext0) { ext0 = chi[k] - clo[k]; axis = k; }
  double extent = chi[axis] - clo[axis];
  int64_t nleft = -1;
  int64_t* tmp = B->tmp;
  if (extent > 0.0) {
    int64_t counts[NB] = {0};
    double plo[NB][3], phi[NB][3], slo[NB][3], shi[NB][3];
    for (int b = 0; b < NB; ++b)
      for (int k = 0; k < 3; ++k) { plo[b][k] = INFINITY; phi[b][k] = -INFINITY; }
    unsigned char* bins = (unsigned char*)malloc((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      double c = B->cen[3 * idx[i] + axis];
      int64_t b = (int64_t)(NB * (c - clo[axis]) / extent);
      if (b > NB - 1) b = NB - 1;
      bins[i] = (unsigned char)b;
      counts[b]++;
      for (int k = 0; k < 3; ++k) {
        double l = B->lo[3 * idx[i] + k], h = B->hi[3 * idx[i] + k];
        if (l < plo[b][k]) plo[b][k] = l;
        if (h > phi[b][k]) phi[b][k] = h;
      }
    }
    for (int k = 0; k < 3; ++k) { slo[NB - 1][k] = plo[NB - 1][k]; shi[NB - 1][k] = phi[NB - 1][k]; }
    for (int b = NB - 2; b >= 0; --b)
      for (int k = 0; k < 3; ++k) {
        slo[b][k] = fmin(plo[b][k], slo[b + 1][k]);
        shi[b][k] = fmax(phi[b][k], shi[b + 1][k]);
      }
    double rlo[3] = {INFINITY, INFINITY, INFINITY}, rhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int64_t nl = 0;
    double best = INFINITY;
    int plane = -1;
    for (int b = 0; b < NB - 1; ++b) {
      for (int k = 0; k < 3; ++k) { rlo[k] = fmin(rlo[k], plo[b][k]); rhi[k] = fmax(rhi[k], phi[b][k]); }
      nl += counts[b];
      int64_t nr = n - nl;
      if (nl == 0 || nr == 0) continue;
      double cost = (double)nl * half_area(rlo, rhi) + (double)nr * half_area(slo[b + 1], shi[b + 1]);
      if (cost < best) { best = cost; plane = b; }
    }
    if (plane >= 0) {
      int64_t a = 0, r = 0;
      int64_t* right_buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
      for (int64_t i = 0; i < n; ++i) {
        if (bins[i] <= plane) tmp[a++] = idx[i];
        else right_buf[r++] = idx[i];
      }
      memcpy(idx, tmp, sizeof(int64_t) * (size_t)a);
      memcpy(idx + a, right_buf, sizeof(int64_t) * (size_t)r);
      free(right_buf);
      nleft = a;
    }
    free(bins);
  }
  if (nleft < 0) {
    /* median split on a stable sort of the centroid coordinate:
     * qsort on (key, position) pairs is stable by construction */
    KP* kp = (KP*)malloc(sizeof(KP) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) { kp[i].k = B->cen[3 * idx[i] + axis]; kp[i].pos = i; kp[i].id = idx[i]; }
    qsort(kp, (size_t)n, sizeof(KP), cmp_kp);
    for (int64_t i = 0; i < n; ++i) idx[i] = kp[i].id;
    free(kp);
    nleft = n / 2;
  }
  build_rec(B, idx, nleft);
  int64_t r = build_rec(B, idx + nleft, n - nleft);
  B->right[me] = (int32_t)r;
  return me;
}

/* Returns the node count; node arrays must hold 2*ntri entries. */
ORC_EXPORT int64_t orc_build_bvh(int64_t ntri, const double* v0, const double* v1,
                                 const double* v2, double* bmin, double* bmax,
                                 int32_t* right, int32_t* start, int32_t* count,
                                 int64_t* perm) {
  Builder B;
  memset(&B, 0, sizeof B);
  B.ntri = ntri; B.v0 = v0; B.v1 = v1; B.v2 = v2;
  B.lo = (double*)malloc(sizeof(double) * 3 * (size_t)ntri);
  B.hi = (double*)malloc(sizeof(double) * 3 * (size_t)ntri);
  B.cen = (double*)malloc(sizeof(double) * 3 * (size_t)ntri);
  B.tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)ntri);
  for (int64_t i = 0; i < ntri; ++i)
    for (int k = 0; k < 3; ++k) {
      double a = v0[3 * i + k], b = v1[3 * i + k], c = v2[3 * i + k];
      double lo = fmin(fmin(a, b), c), hi = fmax(fmax(a, b), c);
      B.lo[3 * i + k] = lo; B.hi[3 * i + k] = hi;
      B.cen[3 * i + k] = (lo + hi) * 0.5;
    }
  B.bmin = bmin; B.bmax = bmax; B.right = right; B.start = start; B.count = count;
  B.perm = perm;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)ntri);
  for (int64_t i = 0; i < ntri; ++i) idx[i] = i;
  build_rec(&B, idx, ntri);
  free(idx); free(B.lo); free(B.hi); free(B.cen); free(B.tmp);
  return B.nnodes;
}

/* ------------------------------------------------------------------------- */
/* Traversal restated from _core.pyx:26-253                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t ntri, nnodes;
  const double *bmin, *bmax;
  const int32_t *right, *start, *count;
  const double *v0, *v1, *v2;     /* slot order */
  const int64_t *obj, *prim;      /* slot order */
  const double* normal;           /* slot order (T,3) */
  const int32_t* matrow;          /* slot order */
  const SbrMaterial* mats;
  int32_t nmat;
} OrcScene;

typedef struct {
  double ox, oy, oz, inv0, inv1, inv2;
  int kx, ky, kz;
  double sx, sy, sz;
} RayCtx;

static inline void ray_setup(const double* o, const double* d, RayCtx* c) {
  c->ox = o[0]; c->oy = o[1]; c->oz = o[2];
  c->inv0 = fabs(d[0]) > 1e-300 ? 1.0 / d[0] : copysign(1e300, d[0]);
  c->inv1 = fabs(d[1]) > 1e-300 ? 1.0 / d[1] : copysign(1e300, d[1]);
  c->inv2 = fabs(d[2]) > 1e-300 ? 1.0 / d[2] : copysign(1e300, d[2]);
  int kz = 0;
  if (fabs(d[1]) > fabs(d[0])) kz = 1;
  if (fabs(d[2]) > fabs(d[kz])) kz = 2;
  int kx = (kz + 1) % 3, ky = (kx + 1) % 3;
  if (d[kz] < 0.0) { int t = kx; kx = ky; ky = t; }
  c->kx = kx; c->ky = ky; c->kz = kz;
  c->sx = d[kx] / d[kz];
  c->sy = d[ky] / d[kz];
  c->sz = 1.0 / d[kz];
}

static inline double box_enter(const double* bmin, const double* bmax, const RayCtx* c,
                               double t_min, double bound) {
  double t0, t1, lo, hi, tn, tf;
  t0 = (bmin[0] - c->ox) * c->inv0; t1 = (bmax[0] - c->ox) * c->inv0;
  tn = t0 < t1 ? t0 : t1; tf = t0 > t1 ? t0 : t1;
  t0 = (bmin[1] - c->oy) * c->inv1; t1 = (bmax[1] - c->oy) * c->inv1;
  lo = t0 < t1 ? t0 : t1; hi = t0 > t1 ? t0 : t1;
  if (lo > tn) tn = lo;
  if (hi < tf) tf = hi;
  t0 = (bmin[2] - c->oz) * c->inv2; t1 = (bmax[2] - c->oz) * c->inv2;
  lo = t0 < t1 ? t0 : t1; hi = t0 > t1 ? t0 : t1;
  if (lo > tn) tn = lo;
  if (hi < tf) tf = hi;
  if (tn <= tf && tf > t_min && tn <= bound) return tn;
  return INFINITY;
}

static inline int tri_hit(const double* p0, const double* p1, const double* p2,
                          const RayCtx* c, double t_min, double* t_out, double* u_out,
                          double* v_out) {
  double o[3] = {c->ox, c->oy, c->oz};
  double av[3] = {p0[0] - o[0], p0[1] - o[1], p0[2] - o[2]};
  double bv[3] = {p1[0] - o[0], p1[1] - o[1], p1[2] - o[2]};
  double cv[3] = {p2[0] - o[0], p2[1] - o[1], p2[2] - o[2]};
  double az = av[c->kz], bz = bv[c->kz], cz = cv[c->kz];
  double ax = av[c->kx] - c->sx * az, ay = av[c->ky] - c->sy * az;
  double bx = bv[c->kx] - c->sx * bz, by = bv[c->ky] - c->sy * bz;
  double cx = cv[c->kx] - c->sx * cz, cy = cv[c->ky] - c->sy * cz;
  double u = cx * by - cy * bx;
  double v = ax * cy - ay * cx;
  double w = bx * ay - by * ax;
  if ((u < 0.0 || v < 0.0 || w < 0.0) && (u > 0.0 || v > 0.0 || w > 0.0)) return 0;
  double det = u + v + w;
  if (det == 0.0) return 0;
  double t_num = u * (c->sz * az) + v * (c->sz * bz) + w * (c->sz * cz);
  *t_out = t_num / det;
  if (!(*t_out > t_min)) return 0;
  *u_out = v / det;
  *v_out = w / det;
  return 1;
}

#define STACK_CAP 256

/* returns 0 ok, 1 overflow */
static int closest1(const OrcScene* S, const double* o, const double* d, double t_min,
                    double t_max, double* t_res, int64_t* tri_res, double* u_res,
                    double* v_res) {
  RayCtx c;
  ray_setup(o, d, &c);
  double best_t = t_max;
  int64_t best = -1;
  double bu = 0.0, bv = 0.0;
  int32_t stack[STACK_CAP];
  int sp = 0;
  if (box_enter(S->bmin, S->bmax, &c, t_min, best_t) < INFINITY) stack[sp++] = 0;
  while (sp > 0) {
    int32_t node = stack[--sp];
    if (S->count[node] > 0) {
      int32_t s = S->start[node];
      for (int32_t j = s; j < s + S->count[node]; ++j) {
        double t, u, v;
        if (tri_hit(S->v0 + 3 * j, S->v1 + 3 * j, S->v2 + 3 * j, &c, t_min, &t, &u, &v)) {
          if (t < best_t || (t == best_t && best >= 0 &&
                             (S->obj[j] < S->obj[best] ||
                              (S->obj[j] == S->obj[best] && S->prim[j] < S->prim[best])))) {
            best_t = t; best = j; bu = u; bv = v;
          }
        }
      }
      continue;
    }
    int32_t l = node + 1, r = S->right[node];
    double el = box_enter(S->bmin + 3 * l, S->bmax + 3 * l, &c, t_min, best_t);
    double er = box_enter(S->bmin + 3 * r, S->bmax + 3 * r, &c, t_min, best_t);
    if (el < INFINITY && er < INFINITY) {
      if (sp + 2 > STACK_CAP) return 1;
      if (el <= er) { stack[sp] = r; stack[sp + 1] = l; }
      else { stack[sp] = l; stack[sp + 1] = r; }
      sp += 2;
    } else if (el < INFINITY) {
      stack[sp++] = l;
    } else if (er < INFINITY) {
      stack[sp++] = r;
    }
  }
  if (best >= 0) { *t_res = best_t; *tri_res = best; *u_res = bu; *v_res = bv; }
  else { *t_res = INFINITY; *tri_res = -1; *u_res = 0.0; *v_res = 0.0; }
  return 0;
}

static int any1(const OrcScene* S, const double* o, const double* d, double t_min,
                double limit, int* found_out) {
  RayCtx c;
  ray_setup(o, d, &c);
  int32_t stack[STACK_CAP];
  int sp = 0, found = 0;
  if (box_enter(S->bmin, S->bmax, &c, t_min, limit) < INFINITY) stack[sp++] = 0;
  while (sp > 0 && !found) {
    int32_t node = stack[--sp];
    if (S->count[node] > 0) {
      int32_t s = S->start[node];
      for (int32_t j = s; j < s + S->count[node]; ++j) {
        double t, u, v;
        if (tri_hit(S->v0 + 3 * j, S->v1 + 3 * j, S->v2 + 3 * j, &c, t_min, &t, &u, &v)) {
          if (t < limit) { found = 1; break; }
        }
      }
      continue;
    }
    int32_t l = node + 1, r = S->right[node];
    if (sp + 2 > STACK_CAP) return 1;
    if (box_enter(S->bmin + 3 * l, S->bmax + 3 * l, &c, t_min, limit) < INFINITY) stack[sp++] = l;
    if (box_enter(S->bmin + 3 * r, S->bmax + 3 * r, &c, t_min, limit) < INFINITY) stack[sp++] = r;
  }
  *found_out = found;
  return 0;
}

ORC_EXPORT int orc_trace_closest(const OrcScene* S, const double* origins, const double* dirs,
                                 double t_min, const double* t_max, int64_t n, double* t,
                                 int64_t* tri, double* u, double* v) {
  for (int64_t i = 0; i < n; ++i)
    if (closest1(S, origins + 3 * i, dirs + 3 * i, t_min, t_max[i], t + i, tri + i, u + i, v + i))
      return SBR_ERR_STACK;
  return 0;
}

ORC_EXPORT int orc_trace_any(const OrcScene* S, const double* origins, const double* dirs,
                             double t_min, const double* t_max, int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    int f;
    if (any1(S, origins + 3 * i, dirs + 3 * i, t_min, t_max[i], &f)) return SBR_ERR_STACK;
    out[i] = (uint8_t)f;
  }
  return 0;
}

/* occluded_batch (geometry.py:187-201) for one segment */
static int occluded1(const OrcScene* S, const double* a, const double* b, double eps,
                     int* occ) {
  double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double len = norm_seq(d);
  *occ = 0;
  if (!(len > 2.0 * eps)) return 0;
  double dn[3] = {d[0] / len, d[1] / len, d[2] / len};
  double o[3] = {a[0] + eps * dn[0], a[1] + eps * dn[1], a[2] + eps * dn[2]};
  return any1(S, o, dn, 0.0, len - 2.0 * eps, occ);
}

ORC_EXPORT int orc_occluded(const OrcScene* S, const double* a, const double* b, double eps,
                            int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    int o;
    if (occluded1(S, a + 3 * i, b + 3 * i, eps, &o)) return SBR_ERR_STACK;
    out[i] = (uint8_t)o;
  }
  return 0;
}

ORC_EXPORT int64_t orc_scene_struct_size(void) { return (int64_t)sizeof(OrcScene); }

/* ------------------------------------------------------------------------- */
/* Radio map: one ray through radiomap.py:_map_chunk (347-563)                */
/* ------------------------------------------------------------------------- */
static void incidence_frame(const double* k, const double* n, double* e_perp, double* e_par) {
  double cr[3];
  cross3(k, n, cr);
  double nrm = norm_seq(cr);
  if (nrm < 1e-9) {
    /* deterministic_perpendicular (em.py:96-107), 1-D numpy ops */
    double axes[2][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}};
    for (int a = 0; a < 2; ++a) {
      double av = dot_ddot(axes[a], k);
      double u[3] = {axes[a][0] - av * k[0], axes[a][1] - av * k[1], axes[a][2] - av * k[2]};
      double un = sqrt(dot_ddot(u, u));
      if (un > 1e-9) { cr[0] = u[0] / un; cr[1] = u[1] / un; cr[2] = u[2] / un; break; }
    }
    nrm = 1.0;
  }
  e_perp[0] = cr[0] / nrm; e_perp[1] = cr[1] / nrm; e_perp[2] = cr[2] / nrm;
  cross3(e_perp, k, e_par);
}

/* _perpendicular_batch (sampling.py:179-190) */
static void perp_batch(const double* v, double* out) {
  double c[3] = {1.0 - v[0] * v[0], 0.0 - v[0] * v[1], 0.0 - v[0] * v[2]};
  double nrm = norm_seq(c);
  if (nrm <= 1e-9) {
    c[0] = 0.0 - v[1] * v[0]; c[1] = 1.0 - v[1] * v[1]; c[2] = 0.0 - v[1] * v[2];
    nrm = norm_seq(c);
  }
  out[0] = c[0] / nrm; out[1] = c[1] / nrm; out[2] = c[2] / nrm;
}

static inline cpx cdot_real(const cpx* f, const double* e) {
  cpx a = C(f[0].re * e[0], f[0].im * e[0]);
  cpx b = C(f[1].re * e[1], f[1].im * e[1]);
  cpx c = C(f[2].re * e[2], f[2].im * e[2]);
  return C((a.re + b.re) + c.re, (a.im + b.im) + c.im);
}

static inline double field_energy(const cpx* f) {
  return (cabs2(f[0]) + cabs2(f[1])) + cabs2(f[2]);
}

typedef struct {
  uint64_t c[SBR_MC_COUNT];
} MapCounters;

static int map_ray(const OrcScene* S, const SbrMapParams* P, const double* offs,
                   const double* prec, uint64_t g, double* grid, MapCounters* K) {
  const uint64_t chunk = g >> SBR_CHUNK_LOG2;
  const uint64_t slot = g & ((1ULL << SBR_CHUNK_LOG2) - 1);
  double dir[3], org[3] = {P->source[0], P->source[1], P->source[2]};
  orc_fibonacci(P->num_samples, g, dir);
  cpx E[3];
  pattern_field(&P->pattern, dir, E);
  double r_dist = 0.0, omega = P->omega0;
  double weight = alpha_sq(P, offs, prec, dir);
  for (int seg = 0; seg <= P->max_depth; ++seg) {
    double t_hit, u_, v_;
    int64_t tri;
    K->c[SBR_MC_RAY_BOUNCES]++;
    if (closest1(S, org, dir, 1e-4, INFINITY, &t_hit, &tri, &u_, &v_)) {
      K->c[SBR_MC_STACK_OVERFLOW]++;
      return 1;
    }
    if (seg >= 1) {
      double denom = dot_gemv(dir, P->normal);
      double s = -1.0;
      if (fabs(denom) > 1e-12) s = (P->plane_off - dot_gemv(org, P->normal)) / denom;
      if (s > 1e-4 && s < t_hit) {
        double pt[3] = {org[0] + s * dir[0], org[1] + s * dir[1], org[2] + s * dir[2]};
        double rel[3] = {pt[0] - P->corner[0], pt[1] - P->corner[1], pt[2] - P->corner[2]};
        double fu = floor(dot_gemv(rel, P->u_hat) / P->cell_w);
        double fv = floor(dot_gemv(rel, P->v_hat) / P->cell_h);
        if (fu >= 0.0 && fu < (double)P->nx && fv >= 0.0 && fv < (double)P->ny) {
          int64_t iu = (int64_t)fu, iv = (int64_t)fv;
          double val = P->scale * field_energy(E) * omega / fabs(denom) * weight;
          grid[iv * P->nx + iu] += val;
          K->c[SBR_MC_DEPOSITS]++;
        }
      }
    }
    if (tri < 0) { K->c[SBR_MC_ESCAPED]++; return 0; }
    if (seg == P->max_depth) return 0;
    double r_hit = r_dist + t_hit;
    if (seg >= P->cull_from && (P->gain_threshold > 0.0 || P->rr_depth >= 0)) {
      double e_sq = field_energy(E);
      int keep = 1;
      if (P->gain_threshold > 0.0) {
        keep = e_sq >= P->gain_threshold * (r_hit * r_hit);
        if (!keep) K->c[SBR_MC_THRESHOLD_KILLED]++;
      }
      if (P->rr_depth >= 0 && seg >= P->rr_depth) {
        double surv = e_sq < P->rr_max ? e_sq : P->rr_max;
        double u_rr = orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_ROULETTE, slot);
        if (keep && u_rr >= surv) K->c[SBR_MC_ROULETTE_KILLED]++;
        keep = keep && (u_rr < surv);
        if (keep) weight /= surv;
      }
      if (!keep) return 0;
    }
    double pt[3] = {org[0] + t_hit * dir[0], org[1] + t_hit * dir[1], org[2] + t_hit * dir[2]};
    const double* nr = S->normal + 3 * tri;
    double n[3] = {nr[0], nr[1], nr[2]};
    if (dot_seq(dir, n) > 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
    double cos_i = fabs(dot_seq(dir, n));
    const SbrMaterial* m = S->mats + S->matrow[tri];
    Fresnel4 F = slab_fresnel(m, cos_i);
    double r_sq = cabs2(F.rp) + cabs2(F.rl);
    double t_sq = cabs2(F.tp) + cabs2(F.tl);
    /* _interaction_rows (paths.py:572-595) with q_D = 0 */
    double q[4] = {0.0, 0.0, 0.0, 0.0};
    double den = r_sq + t_sq;
    if (den > 0.0) {
      double s_sq = m->scattering * m->scattering;
      q[0] = 1.0 * (1.0 - s_sq) * r_sq / den;
      q[1] = 1.0 * s_sq * r_sq / den;
      q[2] = 1.0 * t_sq / den;
    }
    for (int k = 0; k < 3; ++k) if (!(P->allow_mask >> k & 1)) q[k] = 0.0;
    q[3] = 0.0;
    double total = ((q[0] + q[1]) + q[2]) + q[3];
    if (!(total > 0.0)) { K->c[SBR_MC_TERMINATED]++; return 0; }
    for (int k = 0; k < 4; ++k) q[k] /= total;
    double u = orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_INTERACTION, slot);
    double cum = 0.0;
    int code = 0;
    for (int k = 0; k < 4; ++k) { cum = k ? cum + q[k] : q[k]; code += (u >= cum); }
    if (code > 3) code = 3;
    weight /= q[code];
    double e_perp[3], e_par[3];
    incidence_frame(dir, n, e_perp, e_par);
    cpx c_perp = cdot_real(E, e_perp), c_par = cdot_real(E, e_par);
    double ndir[3] = {dir[0], dir[1], dir[2]};
    if (code == 0) {
      double dn = dot_seq(dir, n);
      double kr[3] = {dir[0] - 2.0 * dn * n[0], dir[1] - 2.0 * dn * n[1], dir[2] - 2.0 * dn * n[2]};
      double e_par_r[3];
      cross3(e_perp, kr, e_par_r);
      cpx a = cmul(F.rp, c_perp), b = cmul(F.rl, c_par);
      for (int k = 0; k < 3; ++k) {
        cpx v = cadd(cscale(e_perp[k], a), cscale(e_par_r[k], b));
        E[k] = cscale(m->spec_amp, v);
      }
      memcpy(ndir, kr, sizeof kr);
    } else if (code == 2) {
      cpx a = cmul(F.tp, c_perp), b = cmul(F.tl, c_par);
      for (int k = 0; k < 3; ++k) E[k] = cadd(cscale(e_perp[k], a), cscale(e_par[k], b));
    }
    r_dist = r_hit;
    if (code == 1) {
      double u0 = orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot);
      double u1 = orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot + 1);
      double cos_t = u0, azim = TWO_PI * u1;
      double x = 1.0 - cos_t * cos_t;
      double sin_t = sqrt(x > 0.0 ? x : 0.0);
      double t1[3], t2[3];
      perp_batch(n, t1);
      cross3(n, t1, t2);
      double a = sin_t * cos(azim), b = sin_t * sin(azim);
      double ks[3];
      for (int k = 0; k < 3; ++k) ks[k] = (a * t1[k] + b * t2[k]) + cos_t * n[k];
      cpx rpc = cmul(F.rp, c_perp), rlc = cmul(F.rl, c_par);
      double g_num = sqrt(cabs2(rpc) + cabs2(rlc));
      double g_den = sqrt(cabs2(c_perp) + cabs2(c_par));
      double gamma = g_den > 0.0 ? g_num / g_den : 0.0;
      double f_s = pattern_density(m, dir, ks, n);
      double cos_s = cos_i;
      double patch = omega * (r_hit * r_hit) / (cos_s > 1e-12 ? cos_s : 1e-12);
      double amp = m->scattering * gamma * sqrt(f_s * cos_s * patch);
      double th_i[3], ph_i[3];
      transverse(dir, th_i, ph_i);
      cpx ci0 = cdot_real(E, th_i), ci1 = cdot_real(E, ph_i);
      double kx = m->xpd_kx;
      double chi1 = 0.0, chi2 = 0.0;
      if (P->any_random_phase && m->random_phases) {
        chi1 = TWO_PI * orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot);
        chi2 = TWO_PI * orc_philox_uniform(P->seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot + 1);
      }
      double sq = sqrt(1.0 - kx), sk = sqrt(kx);
      cpx e1 = cscale(amp, C(cos(chi1), sin(chi1)));
      cpx e2 = cscale(amp, C(cos(chi2), sin(chi2)));
      cpx co0 = cmul(e1, csub(cscale(sq, ci0), cscale(sk, ci1)));
      cpx co1 = cmul(e2, cadd(cscale(sk, ci0), cscale(sq, ci1)));
      double th_s[3], ph_s[3];
      transverse(ks, th_s, ph_s);
      for (int k = 0; k < 3; ++k) {
        cpx v = cadd(cscale(th_s[k], co0), cscale(ph_s[k], co1));
        E[k] = cdiv(v, C(r_hit, 0.0));
      }
      memcpy(ndir, ks, sizeof ks);
      r_dist = 0.0;
      omega = TWO_PI;
      K->c[SBR_MC_RESPAWNS]++;
    }
    memcpy(org, pt, sizeof pt);
    memcpy(dir, ndir, sizeof ndir);
  }
  return 0;
}

/* Bounce loop over global sample ids [begin, end).  grid (ny,nx) is
 * accumulated into; counters (SBR_MC_COUNT) likewise. */
ORC_EXPORT int orc_radiomap_bounce(const OrcScene* S, const SbrMapParams* P,
                                   const double* offs, const double* prec, uint64_t begin,
                                   uint64_t end, double* grid, uint64_t* counters) {
  MapCounters K;
  memset(&K, 0, sizeof K);
  int rc = 0;
  for (uint64_t g = begin; g < end; ++g)
    if (map_ray(S, P, offs, prec, g, grid, &K)) { rc = SBR_ERR_STACK; break; }
  for (int k = 0; k < SBR_MC_COUNT; ++k) counters[k] += K.c[k];
  return rc;
}

/* _direct_cells (radiomap.py:566-583) */
ORC_EXPORT int orc_radiomap_direct(const OrcScene* S, const SbrMapParams* P, const double* offs,
                                   const double* prec, double* out, uint64_t* counters) {
  for (int j = 0; j < P->ny; ++j)
    for (int i = 0; i < P->nx; ++i) {
      double uu = ((double)i + 0.5) * P->cell_w, vv = ((double)j + 0.5) * P->cell_h;
      double c[3];
      for (int k = 0; k < 3; ++k) c[k] = (P->corner[k] + uu * P->u_hat[k]) + vv * P->v_hat[k];
      double diff[3] = {c[0] - P->source[0], c[1] - P->source[1], c[2] - P->source[2]};
      double dist = norm_seq(diff);
      double val = 0.0;
      if (dist > 1e-9) {
        double d[3] = {diff[0] / dist, diff[1] / dist, diff[2] / dist};
        cpx E[3];
        pattern_field(&P->pattern, d, E);
        double e_sq = field_energy(E);
        double a_sq = alpha_sq(P, offs, prec, d);
        double x = P->wavelength / (FOUR_PI * dist);
        double gain = x * x * e_sq * a_sq;
        int occ;
        if (occluded1(S, P->source, c, 1e-4, &occ)) return SBR_ERR_STACK;
        val = occ ? 0.0 : gain;
      }
      out[j * P->nx + i] = val;
      if (val > 0.0) counters[SBR_MC_DIRECT_VISIBLE]++;
    }
  return 0;
}
