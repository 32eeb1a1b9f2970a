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
#include <pthread.h>
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
  const uint64_t *hash_r, *hash_f; /* slot order plane hashes (paths.py:449-450) */
  /* diffraction wedges (geometry.py:356-494; paths.py:452-475 tables) */
  int64_t nw;
  const double *w_origin, *w_ehat, *w_t0, *w_n0, *w_nn; /* (nw,3) */
  const double *w_len, *w_nopen;                         /* (nw) */
  const uint64_t *w_hr, *w_hf;                           /* hash_edge */
  const int32_t *w_mat0, *w_matn;                        /* face material rows */
  const int32_t *slot_woff, *slot_wids;                  /* CSR: slot -> owned wedges */
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

/* node / triangle visit statistics of closest1 (BVH-quality diagnostics) */
static __thread uint64_t g_orc_nodes = 0, g_orc_tris = 0;  /* per thread */
ORC_EXPORT void orc_visit_stats(uint64_t* nodes, uint64_t* tris, int reset) {
  *nodes = g_orc_nodes;
  *tris = g_orc_tris;
  if (reset) g_orc_nodes = g_orc_tris = 0;
}

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
      g_orc_tris += (uint64_t)S->count[node];
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
    g_orc_nodes++;
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

/* ========================================================================= */
/* Path solver (CIR): generate_candidates / refine_candidate /               */
/* compute_path_fields / frequency_response, restated from paths.py          */
/* ========================================================================= */
/* Sequential restatement at workers=1: one chunk holding every sample, the
 * depth loop of _sweep_chunk (paths.py:704-828) over all live samples, rows
 * emitted in (depth, sample, target) order (_emit_records 903-987) with the
 * in-chunk "seen pairs" dedup and per-depth truncation, then the ordered
 * DedupTable / PathBuffer registration of generate_candidates (1019-1103).
 * Diffraction is out of scope (no wedges): D is never allowed. */

#define TAG_INTERACTION 0x5c798e00ad8012ebULL
#define TAG_RESPAWN 0x742c480a24ff9b7fULL
#define TAG_CONE 0x0bc9fb91195d708aULL
#define FNV_OFFSET 0xCBF29CE484222325ULL
#define FNV_PRIME 0x100000001B3ULL

typedef struct {
  double source[3];
  const double* targets;   /* (nt, 3) */
  int32_t nt;
  int32_t max_depth;
  int32_t allow;           /* R=1 S=2 T=4 */
  int32_t pad_;
  double q_d;
  uint64_t num_samples, seed;
  uint64_t n_hash;
  int64_t n_buffer;
} OrcCirParams;

/* records, caller-allocated with capacity n_buffer (step arrays stride L) */
typedef struct {
  int32_t* target;
  int64_t* sample;
  int32_t* depth;
  int32_t* suffix_start;
  uint8_t* diffuse;
  uint64_t* chain_hash;
  double* prefix_prob;
  double* anchor;          /* (n,3) */
  int8_t* kind;            /* (n,L) */
  int32_t* tri;            /* (n,L) slot */
  double* vertex;          /* (n,L,3) */
  double* normal;          /* (n,L,3) */
  int32_t L;
  int32_t pad_;
  int32_t* wedge;          /* (n,L) wedge index, -1 */
} OrcRecords;

enum { OC_ESCAPED = 0, OC_TERMINATED, OC_RB, OC_VIS, OC_ROWS, OC_DUP, OC_TRUNC, OC_OVERFLOW,
       OC_CAND, OC_REG, OC_SLOTS, OC_COUNT };

static uint64_t fnv1a_u64(uint64_t v, uint64_t h) {
  for (int s = 0; s < 64; s += 8) h = (h ^ ((v >> s) & 0xFFULL)) * FNV_PRIME;
  return h;
}

/* per (sample, depth) state after the interaction at that depth */
typedef struct {
  double vertex[3], normal[3];
  double run_prob;
  uint64_t hr, hf;
  int32_t tri;
  int32_t wedge;
  int8_t code;             /* -1: no interaction at this depth (dead) */
  int8_t suffix_start;
} Hist;

/* open-addressing set of (pr, pf) pairs */
typedef struct { uint64_t* k; uint8_t* used; uint64_t cap, n; } PairSet;
static int pairset_insert(PairSet* s, uint64_t a, uint64_t b) {
  if (2 * (s->n + 1) > s->cap) {
    uint64_t nc = s->cap ? 2 * s->cap : 1024;
    uint64_t* nk = (uint64_t*)calloc(2 * nc, sizeof(uint64_t));
    uint8_t* nu = (uint8_t*)calloc(nc, 1);
    for (uint64_t i = 0; i < s->cap; ++i)
      if (s->used[i]) {
        uint64_t h = (s->k[2 * i] * 0x9E3779B97F4A7C15ULL ^ s->k[2 * i + 1]) % nc;
        while (nu[h]) h = (h + 1) % nc;
        nu[h] = 1; nk[2 * h] = s->k[2 * i]; nk[2 * h + 1] = s->k[2 * i + 1];
      }
    free(s->k); free(s->used);
    s->k = nk; s->used = nu; s->cap = nc;
  }
  uint64_t h = (a * 0x9E3779B97F4A7C15ULL ^ b) % s->cap;
  while (s->used[h]) {
    if (s->k[2 * h] == a && s->k[2 * h + 1] == b) return 0;
    h = (h + 1) % s->cap;
  }
  s->used[h] = 1; s->k[2 * h] = a; s->k[2 * h + 1] = b; s->n++;
  return 1;
}

typedef struct { int64_t g; int32_t depth, k; uint8_t chain, diffuse; uint64_t pr, pf; } Row;

/* interaction probabilities (_interaction_rows paths.py:572-595) */
/* allow: bit0 R, bit1 S, bit2 T, bit3 D (already masked by has_s / has_d / wedges) */
static int interaction_q(const SbrMaterial* m, double cos_i, double q_d, int allow, double q[4]) {
  Fresnel4 F = slab_fresnel(m, cos_i);
  double r_sq = cabs2(F.rp) + cabs2(F.rl);
  double t_sq = cabs2(F.tp) + cabs2(F.tl);
  double den = r_sq + t_sq;
  q[0] = q[1] = q[2] = 0.0;
  q[3] = q_d;
  if (den > 0.0) {
    double keep = 1.0 - q_d, s_sq = m->scattering * m->scattering;
    q[0] = keep * (1.0 - s_sq) * r_sq / den;
    q[1] = keep * s_sq * r_sq / den;
    q[2] = keep * t_sq / den;
  }
  for (int k = 0; k < 4; ++k) if (!(allow >> k & 1)) q[k] = 0.0;
  double total = ((q[0] + q[1]) + q[2]) + q[3];
  if (!(total > 0.0)) return 0;
  for (int k = 0; k < 4; ++k) q[k] /= total;
  return 1;
}

/* allowed kinds at a hit (paths.py:743-748) */
static int allowed_kinds(const OrcScene* S, int allow, int64_t tri, int has_s, int has_d) {
  int a = allow & 15;
  if (has_d) a &= ~2;
  if (has_d || has_s) a &= ~8;
  if (!(S->nw > 0 && S->slot_woff[tri + 1] > S->slot_woff[tri])) a &= ~8;
  return a;
}

/* _project_diffractions (paths.py:831-852): nearest owned wedge, clamped foot */
static int32_t project_wedge(const OrcScene* S, int64_t tri, const double* p, double* foot) {
  double best = INFINITY;
  int32_t bw = -1;
  for (int32_t k = S->slot_woff[tri]; k < S->slot_woff[tri + 1]; ++k) {
    const int32_t w = S->slot_wids[k];
    const double* o = S->w_origin + 3 * w;
    const double* e = S->w_ehat + 3 * w;
    double rel[3] = {p[0] - o[0], p[1] - o[1], p[2] - o[2]};
    double x = dot_seq(rel, e);
    x = x < 0.0 ? 0.0 : (x > S->w_len[w] ? S->w_len[w] : x);
    double f[3] = {o[0] + x * e[0], o[1] + x * e[1], o[2] + x * e[2]};
    double df[3] = {p[0] - f[0], p[1] - f[1], p[2] - f[2]};
    double dist = norm_seq(df);
    if (dist < best) { best = dist; bw = w; memcpy(foot, f, sizeof f); }
  }
  return bw;
}

/* Per-sample sweep of global ids [lo, hi) into H (indexed g - lo). */
static int sweep_one(const OrcScene* S, const OrcCirParams* P, uint64_t lo, uint64_t g, Hist* H,
                     uint64_t* counters) {
  const int L = P->max_depth;
  const uint64_t N = P->num_samples;
  {
    double o[3] = {P->source[0], P->source[1], P->source[2]}, d[3];
    orc_fibonacci(N, g, d);
    uint64_t hr = 0, hf = 0;
    double run_prob = 1.0;
    int suffix = 0, has_s = 0, has_d = 0;
    for (int depth = 1; depth <= L; ++depth) {
      double t, u_, v_;
      int64_t tri;
      counters[OC_RB]++;
      if (closest1(S, o, d, 1e-4, INFINITY, &t, &tri, &u_, &v_)) return SBR_ERR_STACK;
      if (tri < 0) { counters[OC_ESCAPED]++; break; }
      double pt[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
      const double* nr = S->normal + 3 * tri;
      double n[3] = {nr[0], nr[1], nr[2]};
      if (dot_seq(d, n) > 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
      double cos_i = fabs(dot_seq(d, n));
      double q[4];
      const int allow = allowed_kinds(S, P->allow, tri, has_s, has_d);
      if (!interaction_q(S->mats + S->matrow[tri], cos_i, P->q_d, allow, q)) {
        counters[OC_TERMINATED]++;
        break;
      }
      double uu = orc_philox_uniform(P->seed, 0, (uint64_t)depth, TAG_INTERACTION, g);
      double cum = 0.0;
      int code = 0;
      for (int k = 0; k < 4; ++k) { cum = k ? cum + q[k] : q[k]; code += (uu >= cum); }
      if (code > 3) code = 3;
      run_prob *= q[code];
      int32_t wid = -1;
      if (code == 3) {
        double foot[3];
        wid = project_wedge(S, tri, pt, foot);
        memcpy(pt, foot, sizeof foot);
        has_d = 1;
      }
      if (code == 0) {
        hr = 1373ULL * hr + S->hash_r[tri];
        hf = 1373ULL * hf + S->hash_f[tri];
      } else if (code == 3) {
        hr = 1373ULL * hr + S->w_hr[wid];
        hf = 1373ULL * hf + S->w_hf[wid];
      } else if (code == 1) {
        suffix = depth;
        has_s = 1;
      }
      Hist* h = H + (g - lo) * L + (depth - 1);
      memcpy(h->vertex, pt, sizeof pt);
      memcpy(h->normal, n, sizeof n);
      h->run_prob = run_prob; h->hr = hr; h->hf = hf; h->tri = (int32_t)tri;
      h->wedge = wid;
      h->code = (int8_t)code; h->suffix_start = (int8_t)suffix;
      if (depth == L) break;
      /* _continue_rays (paths.py:855-900) */
      if (code == 0) {
        double dn = dot_seq(d, n);
        for (int k = 0; k < 3; ++k) d[k] = d[k] - 2.0 * dn * n[k];
      } else if (code == 1) {
        double u0 = orc_philox_uniform(P->seed, 0, (uint64_t)depth, TAG_RESPAWN, 2 * g);
        double u1 = orc_philox_uniform(P->seed, 0, (uint64_t)depth, TAG_RESPAWN, 2 * g + 1);
        double cos_t = u0, azim = TWO_PI * u1;
        double x = 1.0 - cos_t * cos_t, sin_t = sqrt(x > 0.0 ? x : 0.0);
        double t1[3], t2[3];
        perp_batch(n, t1);
        cross3(n, t1, t2);
        double a = sin_t * cos(azim), b = sin_t * sin(azim);
        for (int k = 0; k < 3; ++k) d[k] = (a * t1[k] + b * t2[k]) + cos_t * n[k];
      } else if (code == 3) {
        /* Keller cone (paths.py:881-896) */
        const double* e = S->w_ehat + 3 * wid;
        double cb = dot_seq(d, e);
        cb = cb < -1.0 ? -1.0 : (cb > 1.0 ? 1.0 : cb);
        double x = 1.0 - cb * cb, sb = sqrt(x > 0.0 ? x : 0.0);
        if (sb < 1e-9) { counters[OC_TERMINATED]++; break; }
        double phi = orc_philox_uniform(P->seed, 0, (uint64_t)depth, TAG_CONE, g) *
                     S->w_nopen[wid] * PI_;
        double a = sb * cos(phi), b = sb * sin(phi);
        const double* t0 = S->w_t0 + 3 * wid;
        const double* n0 = S->w_n0 + 3 * wid;
        for (int k = 0; k < 3; ++k) d[k] = (a * t0[k] + b * n0[k]) + cb * e[k];
      }
      memcpy(o, pt, sizeof pt);
    }
  }
  return 0;
}

/* Test-infrastructure threading (orc_set_threads, default 1): samples are
 * independent, so the sweep and the visibility rows split over pthreads that
 * claim items from a shared counter, with per-thread counters; rows are
 * concatenated in (depth, sample, target) order, so every result is identical
 * to the single-threaded run. */
static int g_orc_threads = 1;
ORC_EXPORT void orc_set_threads(int n) { g_orc_threads = n > 0 ? n : 1; }

typedef int (*ItemFn)(void* ctx, int64_t item, uint64_t* counters);
typedef struct {
  ItemFn fn;
  void* ctx;
  int64_t n, next;
  uint64_t counters[OC_COUNT];
  int rc;
  pthread_mutex_t mu;
} ItemPool;

static void* item_worker(void* arg) {
  ItemPool* P = (ItemPool*)arg;
  uint64_t local[OC_COUNT] = {0};
  int rc = 0;
  for (;;) {
    const int64_t i = __atomic_fetch_add(&P->next, 1, __ATOMIC_RELAXED);
    if (i >= P->n || rc) break;
    rc = P->fn(P->ctx, i, local);
  }
  pthread_mutex_lock(&P->mu);
  for (int k = 0; k < OC_COUNT; ++k) P->counters[k] += local[k];
  if (rc) P->rc = rc;
  pthread_mutex_unlock(&P->mu);
  return NULL;
}

/* fn(ctx, i, counters) for i in [0, n) on g_orc_threads threads; returns the
 * first nonzero status; counters are summed into `counters` */
static int parallel_items(int64_t n, ItemFn fn, void* ctx, uint64_t* counters) {
  ItemPool P;
  memset(&P, 0, sizeof P);
  P.fn = fn; P.ctx = ctx; P.n = n;
  pthread_mutex_init(&P.mu, NULL);
  int nt = g_orc_threads;
  if (nt > n) nt = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  if (nt > 256) nt = 256;
  if (nt <= 1) {
    item_worker(&P);
  } else {
    for (int t = 0; t < nt; ++t) pthread_create(th + t, NULL, item_worker, &P);
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  }
  pthread_mutex_destroy(&P.mu);
  for (int k = 0; k < OC_COUNT; ++k) counters[k] += P.counters[k];
  return P.rc;
}

typedef struct {
  const OrcScene* S;
  const OrcCirParams* P;
  uint64_t lo, hi;
  Hist* H;
} SweepCtx;

static int sweep_item(void* c, int64_t b, uint64_t* counters) {
  SweepCtx* x = (SweepCtx*)c;
  const uint64_t g0 = x->lo + (uint64_t)b * 64, g1 = g0 + 64 < x->hi ? g0 + 64 : x->hi;
  for (uint64_t g = g0; g < g1; ++g) {
    const int rc = sweep_one(x->S, x->P, x->lo, g, x->H, counters);
    if (rc) return rc;
  }
  return 0;
}

static int cir_sweep(const OrcScene* S, const OrcCirParams* P, uint64_t lo, uint64_t hi, Hist* H,
                     uint64_t* counters) {
  const int L = P->max_depth;
  for (uint64_t i = 0; i < (hi - lo) * (uint64_t)(L > 0 ? L : 1); ++i) H[i].code = -1;
  SweepCtx x = {S, P, lo, hi, H};
  return parallel_items((int64_t)((hi - lo + 63) / 64), sweep_item, &x, counters);
}

/* visible rows of H in (depth, sample, target) order (_visible_pairs 657-683) */
typedef struct {
  Row* rows;
  int64_t n, cap;
} RowBuf;

/* rows of samples [g0, g1) at one depth, appended to B */
static int rows_block(const OrcScene* S, const OrcCirParams* P, uint64_t lo, int depth,
                      uint64_t g0, uint64_t g1, const Hist* H, RowBuf* B, uint64_t* counters) {
  const int L = P->max_depth, nt = P->nt;
  for (uint64_t g = g0; g < g1; ++g) {
    const Hist* h = H + (g - lo) * L + (depth - 1);
    if (h->code < 0) continue;
    for (int k = 0; k < nt; ++k) {
      const double* tg = P->targets + 3 * k;
      double diff[3] = {tg[0] - h->vertex[0], tg[1] - h->vertex[1], tg[2] - h->vertex[2]};
      double side = dot_seq(diff, h->normal);
      int ok = h->code == 2 ? side < 0.0 : side > 0.0;
      if (h->code == 3) ok = 1;
      if (!ok) continue;
      counters[OC_VIS]++;
      int occ;
      if (occluded1(S, h->vertex, tg, 1e-4, &occ)) return SBR_ERR_STACK;
      if (occ) continue;
      counters[OC_ROWS]++;
      if (B->n == B->cap) {
        B->cap = B->cap ? 2 * B->cap : 1024;
        B->rows = (Row*)realloc(B->rows, sizeof(Row) * (size_t)B->cap);
      }
      Row* r = B->rows + B->n++;
      r->g = (int64_t)g; r->depth = depth; r->k = k;
      r->diffuse = h->code == 1;
      r->chain = h->suffix_start == 0 && h->code != 1;
      r->pr = fnv1a_u64(h->hr, (uint64_t)k);
      r->pf = fnv1a_u64(h->hf, (uint64_t)k);
    }
  }
  return 0;
}

typedef struct {
  const OrcScene* S;
  const OrcCirParams* P;
  uint64_t lo, hi;
  int depth;
  const Hist* H;
  RowBuf* blk;
} RowsCtx;

static int rows_item(void* c, int64_t b, uint64_t* counters) {
  RowsCtx* x = (RowsCtx*)c;
  const uint64_t g0 = x->lo + (uint64_t)b * 256, g1 = g0 + 256 < x->hi ? g0 + 256 : x->hi;
  x->blk[b].n = 0;
  return rows_block(x->S, x->P, x->lo, x->depth, g0, g1, x->H, x->blk + b, counters);
}

static int cir_rows(const OrcScene* S, const OrcCirParams* P, uint64_t lo, uint64_t hi,
                    const Hist* H, Row** rows_out, int64_t* n_out, uint64_t* counters) {
  const int L = P->max_depth;
  const uint64_t span = hi - lo;
  const int64_t nblk = span == 0 ? 0 : (int64_t)((span + 255) / 256);
  RowBuf* blk = (RowBuf*)calloc((size_t)(nblk > 0 ? nblk : 1), sizeof(RowBuf));
  Row* rows = NULL;
  int64_t n = 0, cap = 0;
  int rc = 0;
  for (int depth = 1; depth <= L && !rc; ++depth) {
    RowsCtx x = {S, P, lo, hi, depth, H, blk};
    rc = parallel_items(nblk, rows_item, &x, counters);
    for (int64_t b = 0; b < nblk && !rc; ++b) {
      if (n + blk[b].n > cap) {
        cap = 2 * (n + blk[b].n) + 4096;
        rows = (Row*)realloc(rows, sizeof(Row) * (size_t)cap);
      }
      if (blk[b].n) memcpy(rows + n, blk[b].rows, sizeof(Row) * (size_t)blk[b].n);
      n += blk[b].n;
    }
  }
  for (int64_t b = 0; b < nblk; ++b) free(blk[b].rows);
  free(blk);
  if (rc) {
    free(rows);
    return rc;
  }
  *rows_out = rows;
  *n_out = n;
  return 0;
}

static int row_cmp(const void* a, const void* b) {
  const Row* x = (const Row*)a;
  const Row* y = (const Row*)b;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  if (x->g != y->g) return x->g < y->g ? -1 : 1;
  return x->k < y->k ? -1 : (x->k > y->k);
}

/* _emit_records dedup + truncation and DedupTable / PathBuffer registration
 * (paths.py:903-987, 174-226, 1036-1096) over rows sorted by (depth, sample,
 * target).  rec_row[i]: index into `rows`, or ~k for the LoS record of
 * target k.  los[k] = 1 when the source sees target k. */
static int64_t cir_select(const OrcCirParams* P, const Row* rows, int64_t n, const uint8_t* los,
                          int64_t* rec_row, uint64_t* counters) {
  PairSet seen = {0, 0, 0, 0};
  uint8_t* keep = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  int64_t emitted = 0, i = 0;
  while (i < n) {
    const int depth = rows[i].depth;
    int64_t j = i, depth_rows = 0;
    int64_t room = P->n_buffer - emitted;
    if (room < 0) room = 0;
    for (; j < n && rows[j].depth == depth; ++j) {
      if (rows[j].chain && !pairset_insert(&seen, rows[j].pr, rows[j].pf)) {
        counters[OC_DUP]++;
        continue;
      }
      if (depth_rows < room) keep[j] = 1;
      depth_rows++;
    }
    /* a depth cut to nothing returns no batch: its truncation is not counted */
    if (depth_rows > room) {
      if (room > 0) counters[OC_TRUNC] += (uint64_t)(depth_rows - room);
      emitted += room;
    } else {
      emitted += depth_rows;
    }
    i = j;
  }
  free(seen.k); free(seen.used);
  int32_t* counts = (int32_t*)calloc((size_t)P->n_hash, sizeof(int32_t));
  int64_t nrec = 0;
  for (int k = 0; k < P->nt; ++k) {
    if (!los[k]) continue;
    uint64_t i1 = fnv1a_u64(0ULL, (uint64_t)k) % P->n_hash;
    if (counts[i1] == 0) {
      counts[i1] += 2;
      counters[OC_REG]++;
    } else {
      counters[OC_DUP]++;
      continue;
    }
    if (nrec >= P->n_buffer) { counters[OC_OVERFLOW]++; continue; }
    rec_row[nrec++] = ~(int64_t)k;
  }
  for (int64_t r = 0; r < n; ++r) {
    if (!keep[r]) continue;
    if (rows[r].chain) {
      uint64_t i1 = rows[r].pr % P->n_hash, i2 = rows[r].pf % P->n_hash;
      if (counts[i1] == 0 && counts[i2] == 0) {
        counts[i1]++; counts[i2]++;
        counters[OC_REG]++;
      } else {
        counters[OC_DUP]++;
        continue;
      }
    }
    if (nrec >= P->n_buffer) { counters[OC_OVERFLOW]++; continue; }
    rec_row[nrec++] = r;
  }
  for (uint64_t s = 0; s < P->n_hash; ++s) counters[OC_SLOTS] += counts[s] != 0;
  counters[OC_CAND] += (uint64_t)nrec;
  free(counts); free(keep);
  return nrec;
}

static int cir_los(const OrcScene* S, const OrcCirParams* P, uint8_t* los) {
  for (int k = 0; k < P->nt; ++k) {
    int occ;
    if (occluded1(S, P->source, P->targets + 3 * k, 1e-4, &occ)) return SBR_ERR_STACK;
    los[k] = !occ;
  }
  return 0;
}

/* Visible rows of the sample range [lo, hi) for the multi-rank path: ordinal
 * key (depth << 60 | sample << 20 | target), pair hashes, chain flag. */
ORC_EXPORT int orc_cir_rows(const OrcScene* S, const OrcCirParams* P, uint64_t lo, uint64_t hi,
                            uint64_t* key, uint64_t* pr, uint64_t* pf, uint8_t* chain,
                            int64_t cap, int64_t* n_out, uint64_t* counters) {
  const int L = P->max_depth > 0 ? P->max_depth : 1;
  Hist* H = (Hist*)malloc(sizeof(Hist) * (size_t)((hi - lo) * L + 1));
  int rc = cir_sweep(S, P, lo, hi, H, counters);
  Row* rows = NULL;
  int64_t n = 0;
  if (!rc) rc = cir_rows(S, P, lo, hi, H, &rows, &n, counters);
  *n_out = n;
  if (!rc && n > cap) rc = SBR_ERR_NOMEM;
  for (int64_t i = 0; !rc && i < n; ++i) {
    key[i] = ((uint64_t)rows[i].depth << 60) | ((uint64_t)rows[i].g << 20) | (uint64_t)rows[i].k;
    pr[i] = rows[i].pr;
    pf[i] = rows[i].pf;
    chain[i] = rows[i].chain;
  }
  free(H); free(rows);
  return rc;
}

/* Selection over rows in any order (e.g. gathered from several ranks):
 * rec_row[i] indexes the caller's arrays, or ~target for LoS. */
ORC_EXPORT int orc_cir_select(const OrcScene* S, const OrcCirParams* P, const uint64_t* key,
                              const uint64_t* pr, const uint64_t* pf, const uint8_t* chain,
                              int64_t n, int64_t* rec_row, int64_t* n_rec, uint64_t* counters) {
  /* decorate rows with their input index, sort by (depth, sample, target) */
  typedef struct { Row r; int64_t i; } Dec;  /* Row first: row_cmp applies */
  Dec* dec = (Dec*)malloc(sizeof(Dec) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    dec[i].r.depth = (int32_t)(key[i] >> 60);
    dec[i].r.g = (int64_t)((key[i] >> 20) & ((1ULL << 40) - 1));
    dec[i].r.k = (int32_t)(key[i] & ((1ULL << 20) - 1));
    dec[i].r.pr = pr[i];
    dec[i].r.pf = pf[i];
    dec[i].r.chain = chain[i];
    dec[i].r.diffuse = 0;
    dec[i].i = i;
  }
  qsort(dec, (size_t)n, sizeof(Dec), row_cmp);
  Row* sorted = (Row*)malloc(sizeof(Row) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) sorted[i] = dec[i].r;
  uint8_t* los = (uint8_t*)malloc((size_t)P->nt);
  int rc = cir_los(S, P, los);
  int64_t nrec = 0;
  if (!rc) {
    nrec = cir_select(P, sorted, n, los, rec_row, counters);
    for (int64_t i = 0; i < nrec; ++i)
      if (rec_row[i] >= 0) rec_row[i] = dec[rec_row[i]].i;
  }
  *n_rec = nrec;
  free(dec); free(sorted); free(los);
  return rc;
}

ORC_EXPORT int orc_cir_generate(const OrcScene* S, const OrcCirParams* P, OrcRecords* R,
                                int64_t* n_out, uint64_t* counters) {
  const int L = P->max_depth > 0 ? P->max_depth : 1;
  const uint64_t N = P->num_samples;
  Hist* H = (Hist*)malloc(sizeof(Hist) * (size_t)(N * L + 1));
  if (!H) return SBR_ERR_NOMEM;
  int rc = cir_sweep(S, P, 0, N, H, counters);
  Row* rows = NULL;
  int64_t n = 0;
  if (!rc) rc = cir_rows(S, P, 0, N, H, &rows, &n, counters);
  uint8_t* los = (uint8_t*)malloc((size_t)P->nt);
  if (!rc) rc = cir_los(S, P, los);
  int64_t* rec_row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P->n_buffer > 0 ? P->n_buffer : 1));
  int64_t nrec = 0;
  if (!rc) nrec = cir_select(P, rows, n, los, rec_row, counters);
  const int Ls = R->L;
  for (int64_t i = 0; !rc && i < nrec; ++i) {
    const int64_t rr = rec_row[i];
    for (int j = 0; j < Ls; ++j) {
      R->kind[i * Ls + j] = -1;
      R->tri[i * Ls + j] = -1;
      R->wedge[i * Ls + j] = -1;
    }
    R->prefix_prob[i] = 1.0;
    memcpy(R->anchor + 3 * i, P->source, 3 * sizeof(double));
    if (rr < 0) {
      R->target[i] = (int32_t)(~rr); R->sample[i] = -1; R->depth[i] = 0;
      R->suffix_start[i] = 0; R->diffuse[i] = 0; R->chain_hash[i] = 0;
      continue;
    }
    const Row* r = rows + rr;
    const Hist* last = H + r->g * L + (r->depth - 1);
    R->target[i] = r->k; R->sample[i] = r->g; R->depth[i] = r->depth;
    R->suffix_start[i] = last->suffix_start; R->diffuse[i] = r->diffuse;
    R->chain_hash[i] = last->hr;
    if (last->suffix_start > 0) {
      const Hist* a = H + r->g * L + (last->suffix_start - 1);
      R->prefix_prob[i] = a->run_prob;
      memcpy(R->anchor + 3 * i, a->vertex, 3 * sizeof(double));
    }
    for (int j = 0; j < r->depth && j < Ls; ++j) {
      const Hist* h = H + r->g * L + j;
      const int64_t o = i * Ls + j;
      R->kind[o] = h->code; R->tri[o] = h->tri; R->wedge[o] = h->wedge;
      memcpy(R->vertex + 3 * o, h->vertex, 3 * sizeof(double));
      memcpy(R->normal + 3 * o, h->normal, 3 * sizeof(double));
    }
  }
  *n_out = nrec;
  free(H); free(rows); free(los); free(rec_row);
  return rc;
}

/* refine_candidate (paths.py:1123-1252), diffraction branch out of scope.
 * pv (n, L+2, 3) = [source, vertices..., target]; status SBR_REFINE_*. */
static void reflect_point(const double* p, const double* nrm, const double* on, double* out) {
  double rel[3] = {p[0] - on[0], p[1] - on[1], p[2] - on[2]};
  double f = dot_ddot(rel, nrm);
  for (int k = 0; k < 3; ++k) out[k] = p[k] - 2.0 * f * nrm[k];
}

static void rotate_about(const double* a, double angle, double R[9]) {
  /* _rotate_about (paths.py:557-565): c I + s K + (1 - c) a a^T */
  double c = cos(angle), sn = sin(angle);
  double K[9] = {0.0, -a[2], a[1], a[2], 0.0, -a[0], -a[1], a[0], 0.0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = (c * (i == j ? 1.0 : 0.0) + sn * K[3 * i + j]) + (1.0 - c) * (a[i] * a[j]);
}

/* solve_diffraction_point (paths.py:517-554); returns 0 ok, 1 degenerate */
static int solve_diffraction_point(const double* src, const double* tgt, const double* eo,
                                   const double* ed, double* x_out) {
  double en = sqrt(dot_ddot(ed, ed));
  double e[3] = {ed[0] / en, ed[1] / en, ed[2] / en};
  double sv[3] = {src[0] - eo[0], src[1] - eo[1], src[2] - eo[2]};
  double tv[3] = {tgt[0] - eo[0], tgt[1] - eo[1], tgt[2] - eo[2]};
  double es = dot_ddot(e, sv), et = dot_ddot(e, tv);
  double u1[3], u2[3];
  for (int k = 0; k < 3; ++k) { u1[k] = sv[k] - es * e[k]; u2[k] = tv[k] - et * e[k]; }
  double n1 = sqrt(dot_ddot(u1, u1)), n2 = sqrt(dot_ddot(u2, u2));
  if (n1 < 1e-12 || n2 < 1e-12) return 1;
  for (int k = 0; k < 3; ++k) { u1[k] /= n1; u2[k] /= n2; }
  double ax[3];
  cross3(u1, u2, ax);
  double na = sqrt(dot_ddot(ax, ax));
  if (na < 1e-12) memcpy(ax, e, sizeof ax);
  else for (int k = 0; k < 3; ++k) ax[k] /= na;
  double cu = dot_ddot(u1, u2);
  cu = cu < -1.0 ? -1.0 : (cu > 1.0 ? 1.0 : cu);
  double angle = PI_ - acos(cu);
  double R[9], tr[3];
  rotate_about(ax, angle, R);
  for (int i = 0; i < 3; ++i) tr[i] = dot_gemv(R + 3 * i, tv);
  double st[3] = {tr[0] - sv[0], tr[1] - sv[1], tr[2] - sv[2]};
  double guide[3], lever[3];
  cross3(e, st, guide);
  double ng = sqrt(dot_ddot(guide, guide));
  if (ng < 1e-12) return 1;
  cross3(sv, st, lever);
  double sign = dot_ddot(guide, lever) >= 0.0 ? 1.0 : -1.0;
  *x_out = sign * (sqrt(dot_ddot(lever, lever)) / ng);
  return 0;
}

static void reflect_vector(const double* v, const double* nrm, double* out) {
  double f = dot_ddot(v, nrm);
  for (int k = 0; k < 3; ++k) out[k] = v[k] - 2.0 * f * nrm[k];
}

ORC_EXPORT int orc_cir_refine(const OrcScene* S, const double* source, const double* targets,
                              const OrcRecords* R, int64_t n, double* pv, int32_t* status) {
  const int L = R->L;
  for (int64_t r = 0; r < n; ++r) {
    const int depth = R->depth[r], ss = R->suffix_start[r];
    const double* tg = targets + 3 * R->target[r];
    double* out = pv + r * (int64_t)(L + 2) * 3;
    memset(out, 0, sizeof(double) * 3 * (size_t)(L + 2));
    memcpy(out, source, 3 * sizeof(double));
    for (int j = 0; j < depth; ++j) memcpy(out + 3 * (j + 1), R->vertex + 3 * (r * L + j), 3 * sizeof(double));
    memcpy(out + 3 * (depth + 1), tg, 3 * sizeof(double));
    status[r] = SBR_REFINE_OK;
    if (R->diffuse[r] || ss >= depth) continue;
    const int ns = depth - ss;
    double img[17][3];
    memcpy(img[0], R->anchor + 3 * r, 3 * sizeof(double));
    int i_d = -1;
    for (int j = 0; j < ns; ++j) {
      int64_t o = r * L + ss + j;
      if (R->kind[o] == 0) reflect_point(img[j], R->normal + 3 * o, R->vertex + 3 * o, img[j + 1]);
      else memcpy(img[j + 1], img[j], sizeof img[j]);
      if (R->kind[o] == 3 && i_d < 0) i_d = j;
    }
    double eo[17][3], ee[17][3], x = 0.0, wlen = 0.0;
    int st = SBR_REFINE_OK;
    if (i_d >= 0) {
      const int w = R->wedge[r * L + ss + i_d];
      memcpy(eo[i_d], S->w_origin + 3 * w, sizeof eo[i_d]);
      memcpy(ee[i_d], S->w_ehat + 3 * w, sizeof ee[i_d]);
      wlen = S->w_len[w];
      for (int j = i_d + 1; j < ns; ++j) {
        int64_t o = r * L + ss + j;
        if (R->kind[o] == 0) {
          reflect_point(eo[j - 1], R->normal + 3 * o, R->vertex + 3 * o, eo[j]);
          reflect_vector(ee[j - 1], R->normal + 3 * o, ee[j]);
        } else {
          memcpy(eo[j], eo[j - 1], sizeof eo[j]);
          memcpy(ee[j], ee[j - 1], sizeof ee[j]);
        }
      }
      if (solve_diffraction_point(img[ns], tg, eo[ns - 1], ee[ns - 1], &x)) st = SBR_REFINE_DEGENERATE;
      else if (!(0.0 <= x && x <= wlen)) st = SBR_REFINE_OFF_EDGE;
    }
    double from[3], refined0[3];
    memcpy(from, tg, sizeof from);
    for (int j = ns - 1; st == SBR_REFINE_OK && j >= 0; --j) {
      int64_t o = r * L + ss + j;
      if (j == i_d) {
        double v[3] = {eo[i_d][0] + x * ee[i_d][0], eo[i_d][1] + x * ee[i_d][1], eo[i_d][2] + x * ee[i_d][2]};
        int occ;
        if (occluded1(S, from, v, 1e-4, &occ)) return SBR_ERR_STACK;
        if (occ) { st = SBR_REFINE_OCCLUDED; break; }
        memcpy(out + 3 * (ss + j + 1), v, sizeof v);
        memcpy(from, v, sizeof v);
        memcpy(refined0, v, sizeof v);
        continue;
      }
      double aim[3];
      if (i_d < 0 || j < i_d) memcpy(aim, img[j + 1], sizeof aim);
      else for (int k = 0; k < 3; ++k) aim[k] = eo[j][k] + x * ee[j][k];
      double ray[3] = {aim[0] - from[0], aim[1] - from[1], aim[2] - from[2]};
      double len = sqrt(dot_ddot(ray, ray));
      if (len < 1e-12) { st = SBR_REFINE_DEGENERATE; break; }
      for (int k = 0; k < 3; ++k) ray[k] = ray[k] / len;
      double t, u_, v_;
      int64_t tri;
      if (closest1(S, from, ray, 1e-4, INFINITY, &t, &tri, &u_, &v_)) return SBR_ERR_STACK;
      if (tri < 0) { st = SBR_REFINE_COPLANAR_MISS; break; }
      const double* sn = R->normal + 3 * o;
      double hp[3] = {from[0] + t * ray[0], from[1] + t * ray[1], from[2] + t * ray[2]};
      double rel[3] = {hp[0] - R->vertex[3 * o], hp[1] - R->vertex[3 * o + 1], hp[2] - R->vertex[3 * o + 2]};
      if (fabs(dot_ddot(S->normal + 3 * tri, sn)) < 1.0 - 1e-6 || !(fabs(dot_ddot(rel, sn)) <= 1e-6)) {
        st = SBR_REFINE_COPLANAR_MISS;
        break;
      }
      memcpy(out + 3 * (ss + j + 1), hp, sizeof hp);
      memcpy(from, hp, sizeof hp);
      memcpy(refined0, hp, sizeof hp);
    }
    if (st == SBR_REFINE_OK) {
      int occ;
      if (occluded1(S, R->anchor + 3 * r, refined0, 1e-4, &occ)) return SBR_ERR_STACK;
      if (occ) st = SBR_REFINE_OCCLUDED;
    }
    status[r] = st;
  }
  return 0;
}

/* ---- compute_path_fields (paths.py:1302-1399), Algorithm 2 ---------------- */
typedef struct {
  double wavelength, q_d;
  uint64_t num_samples, seed;
  int32_t allow;
  int32_t pad_;
  SbrAntenna tx;
  const SbrAntenna* rx;          /* per target */
  double tx_vel[3];
  const double* rx_vel;          /* per target (n,3) */
  const double* obj_vel;         /* per material row (nobj,3) or NULL */
} OrcFieldParams;

/* ---- UTD (materials.py:482-646) ------------------------------------------ */
/* Fresnel integrals S, C: power series below 1.5, continued fraction above
 * (scipy.special.fresnel semantics; agree to ~1e-12 relative). */
static void fresnel_sc(double x, double* s_out, double* c_out) {
  const double PIO2 = 1.5707963267948966;
  double ax = fabs(x), s, c;
  if (ax < 1.5) {
    double t = PIO2 * ax * ax, term = ax, sumc = 0.0, sums = 0.0;
    for (int k = 0; k < 60; ++k) {
      double contrib = term / (2 * k + 1);
      double sign = ((k / 2) % 2) ? -1.0 : 1.0;
      if (k % 2 == 0) sumc += sign * contrib; else sums += sign * contrib;
      term *= t / (k + 1);
      if (term < 1e-18 * (sumc + sums + 1e-300)) break;
    }
    c = sumc; s = sums;
  } else {
    double pix2 = PI_ * ax * ax;
    cpx b = C(1.0, -pix2), cc = C(1e300, 0.0);
    cpx d = cdiv(C(1.0, 0.0), b), h = d;
    int n = -1;
    for (int k = 2; k < 300; ++k) {
      n += 2;
      double a = -(double)n * (double)(n + 1);
      b = C(b.re + 4.0, b.im);
      d = cdiv(C(1.0, 0.0), cadd(cscale(a, d), b));
      cc = cadd(b, cdiv(C(a, 0.0), cc));
      cpx del = cmul(cc, d);
      h = cmul(h, del);
      if (fabs(del.re - 1.0) + fabs(del.im) < 1e-16) break;
    }
    h = cmul(h, C(ax, -ax));
    cpx w = cmul(C(cos(0.5 * pix2), sin(0.5 * pix2)), h);
    cpx cs = cmul(C(0.5, 0.5), C(1.0 - w.re, -w.im));
    c = cs.re; s = cs.im;
  }
  if (x < 0.0) { c = -c; s = -s; }
  *s_out = s; *c_out = c;
}

/* transition_function (materials.py:482-501) */
static cpx transition_f(double x) {
  double arg = sqrt(2.0 * x / PI_), s, c;
  fresnel_sc(arg, &s, &c);
  cpx a = cmul(C(cos(x), sin(x)), C(1.0 - 2.0 * s, 1.0 - 2.0 * c));
  return cscale(sqrt(PI_ * x / 2.0), a);
}

/* _cot_f_product (materials.py:504-528) */
static cpx cot_f(double beta, double n_open, double k, double l, double sign) {
  double n_round = nearbyint((beta + sign * PI_) / (2.0 * n_open * PI_));
  double eps = beta - (2.0 * n_open * PI_ * n_round - sign * PI_);
  if (fabs(eps) < 1e-6) {
    double sg = eps >= 0.0 ? 1.0 : -1.0, kl = k * l;
    cpx q = C(cos(PI_ / 4.0), sin(PI_ / 4.0));
    cpx inner = csub(C(sqrt(2.0 * PI_ * kl) * sg, 0.0), cscale(2.0 * kl * eps, q));
    return cscale(sign * n_open, cmul(q, inner));
  }
  double cot = 1.0 / tan((PI_ + sign * beta) / (2.0 * n_open));
  double cv = cos((2.0 * n_open * PI_ * n_round - beta) / 2.0);
  double a = 2.0 * cv * cv;
  return cscale(cot, transition_f(k * l * a));
}

/* fresnel_vacuum r_perp, r_par (materials.py:173-205) */
static void fresnel_vacuum_r(double c1, double eta_re, double eta_im, cpx* rp, cpx* rl) {
  cpx eta = C(eta_re, eta_im);
  double sin2 = 1.0 - c1 * c1;
  cpx root = csqrt_lossy(C(eta.re - sin2, eta.im));
  *rp = cdiv(C(c1 - root.re, -root.im), C(c1 + root.re, root.im));
  cpx ec = C(eta.re * c1, eta.im * c1);
  *rl = cdiv(csub(ec, root), cadd(ec, root));
  if (eta.im == 0.0 && sin2 >= cabs_(eta)) { *rp = C(1.0, 0.0); *rl = C(1.0, 0.0); }
}

typedef struct { cpx m[2][2]; } M2;
static M2 m2_mul(M2 a, M2 b) {
  M2 r;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) r.m[i][j] = cadd(cmul(a.m[i][0], b.m[0][j]), cmul(a.m[i][1], b.m[1][j]));
  return r;
}
static M2 m2_w(const double* a, const double* b, const double* q, const double* r) {
  M2 w;
  w.m[0][0] = C(dot_ddot(a, q), 0.0); w.m[0][1] = C(dot_ddot(a, r), 0.0);
  w.m[1][0] = C(dot_ddot(b, q), 0.0); w.m[1][1] = C(dot_ddot(b, r), 0.0);
  return w;
}
static void oblique_frame(const double* s_hat, const double* n_hat, const double* other,
                          double* e_perp, double* e_par) {
  double cr[3];
  cross3(s_hat, n_hat, cr);
  double nn = sqrt(dot_ddot(cr, cr));
  if (nn < 1e-9) {
    double axes[2][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}};
    for (int a = 0; a < 2; ++a) {
      double av = dot_ddot(axes[a], s_hat);
      double u[3] = {axes[a][0] - av * s_hat[0], axes[a][1] - av * s_hat[1], axes[a][2] - av * s_hat[2]};
      double un = sqrt(dot_ddot(u, u));
      if (un > 1e-9) { for (int k = 0; k < 3; ++k) e_perp[k] = u[k] / un; break; }
    }
  } else {
    for (int k = 0; k < 3; ++k) e_perp[k] = cr[k] / nn;
  }
  cross3(e_perp, other, e_par);
}

/* utd_transfer (materials.py:547-646); returns 0 ok, 1 degenerate geometry */
static int utd_transfer(const OrcScene* S, int w, const double* s_i, const double* s_o,
                        double dist_in, double dist_out, double lam, M2* out, double b_in[2][3],
                        double b_out[2][3]) {
  const double* e = S->w_ehat + 3 * w;
  const double n_open = S->w_nopen[w];
  double cos_beta = dot_ddot(s_i, e);
  double x = 1.0 - cos_beta * cos_beta, sb0 = sqrt(x > 0.0 ? x : 0.0);
  if (sb0 < 1e-9) return 1;
  double ci[3], so_neg[3] = {-s_o[0], -s_o[1], -s_o[2]}, co[3];
  cross3(s_i, e, ci);
  double nci = sqrt(dot_ddot(ci, ci));
  for (int k = 0; k < 3; ++k) b_in[0][k] = ci[k] / nci;
  cross3(b_in[0], s_i, b_in[1]);
  cross3(so_neg, e, co);
  double nco = sqrt(dot_ddot(co, co));
  if (nco < 1e-9) return 1;
  for (int k = 0; k < 3; ++k) b_out[0][k] = co[k] / nco;
  cross3(b_out[0], s_o, b_out[1]);
  const double* t0 = S->w_t0 + 3 * w;
  const double* n0 = S->w_n0 + 3 * w;
  double sit[3], sot[3], a1 = dot_ddot(s_i, e), a2 = dot_ddot(s_o, e);
  for (int k = 0; k < 3; ++k) { sit[k] = s_i[k] - a1 * e[k]; sot[k] = s_o[k] - a2 * e[k]; }
  double n1 = sqrt(dot_ddot(sit, sit)), n2 = sqrt(dot_ddot(sot, sot));
  for (int k = 0; k < 3; ++k) { sit[k] /= n1; sot[k] /= n2; }
  double msit[3] = {-sit[0], -sit[1], -sit[2]};
  double c_in = dot_ddot(msit, t0), c_out = dot_ddot(sot, t0);
  c_in = c_in < -1.0 ? -1.0 : (c_in > 1.0 ? 1.0 : c_in);
  c_out = c_out < -1.0 ? -1.0 : (c_out > 1.0 ? 1.0 : c_out);
  double phi_in = PI_ - (PI_ - acos(c_in)) * (dot_ddot(msit, n0) >= 0.0 ? 1.0 : -1.0);
  double phi_out = PI_ - (PI_ - acos(c_out)) * (dot_ddot(sot, n0) >= 0.0 ? 1.0 : -1.0);
  double k = TWO_PI / lam;
  double l = dist_in * dist_out / (dist_in + dist_out) * (sb0 * sb0);
  cpx pref = cdiv(C(-cos(-PI_ / 4.0), -sin(-PI_ / 4.0)),
                  C(2.0 * n_open * sqrt(2.0 * PI_ * k) * sb0, 0.0));
  cpx d1 = cmul(pref, cot_f(phi_out - phi_in, n_open, k, l, 1.0));
  cpx d2 = cmul(pref, cot_f(phi_out - phi_in, n_open, k, l, -1.0));
  cpx d3 = cmul(pref, cot_f(phi_out + phi_in, n_open, k, l, 1.0));
  cpx d4 = cmul(pref, cot_f(phi_out + phi_in, n_open, k, l, -1.0));
  const SbrMaterial* m0 = S->mats + S->w_mat0[w];
  const SbrMaterial* mn = S->mats + S->w_matn[w];
  double cos_r[2] = {fabs(sin(phi_in)), fabs(sin(n_open * PI_ - phi_out))};
  const double* nf[2] = {n0, S->w_nn + 3 * w};
  const SbrMaterial* mf[2] = {m0, mn};
  M2 refl[2];
  for (int f = 0; f < 2; ++f) {
    double ep[3] = {1.0, 0.0, 0.0}, el[3], er[3];
    oblique_frame(s_i, nf[f], s_i, ep, el);
    cross3(ep, s_o, er);
    cpx rp, rl;
    fresnel_vacuum_r(cos_r[f], mf[f]->eta_re, mf[f]->eta_im, &rp, &rl);
    M2 dg;
    dg.m[0][0] = rp; dg.m[0][1] = C(0.0, 0.0); dg.m[1][0] = C(0.0, 0.0); dg.m[1][1] = rl;
    refl[f] = m2_mul(m2_mul(m2_w(b_out[0], b_out[1], ep, er), dg), m2_w(ep, el, b_in[0], b_in[1]));
  }
  cpx d12 = cadd(d1, d2);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      cpx v = i == j ? d12 : C(0.0, 0.0);
      v = csub(csub(v, cmul(d3, refl[1].m[i][j])), cmul(d4, refl[0].m[i][j]));
      out->m[i][j] = C(-v.re, -v.im);
    }
  return 0;
}

/* pattern_to_gcs (em.py:198-219) for the built-in evaluators (c_phi_l = 0) */
static void pattern_gcs(const SbrAntenna* A, const double* d, double* c_th, double* c_ph,
                        double th_g[3], double ph_g[3]) {
  const double* R = A->rot;
  double dl[3];
  for (int k = 0; k < 3; ++k) dl[k] = R[0 * 3 + k] * d[0] + R[1 * 3 + k] * d[1] + R[2 * 3 + k] * d[2];
  double z = dl[2] < -1.0 ? -1.0 : (dl[2] > 1.0 ? 1.0 : dl[2]);
  double theta_l = acos(z), phi_l = atan2(dl[1], dl[0]);
  double amp = A->kind == SBR_PATTERN_TR38901 ? tr38901_amp(A->scale, theta_l, phi_l) : 1.0;
  transverse(d, th_g, ph_g);
  double th_l[3] = {cos(theta_l) * cos(phi_l), cos(theta_l) * sin(phi_l), -sin(theta_l)};
  double thw[3];
  for (int k = 0; k < 3; ++k) thw[k] = R[3 * k] * th_l[0] + R[3 * k + 1] * th_l[1] + R[3 * k + 2] * th_l[2];
  *c_th = dot_ddot(th_g, thw) * amp;
  *c_ph = dot_ddot(ph_g, thw) * amp;
}

static void basis_w(const double* a, const double* b, const double* q, const double* r, cpx c0,
                    cpx c1, cpx* o0, cpx* o1) {
  double w00 = dot_ddot(a, q), w01 = dot_ddot(a, r), w10 = dot_ddot(b, q), w11 = dot_ddot(b, r);
  *o0 = cadd(cscale(w00, c0), cscale(w01, c1));
  *o1 = cadd(cscale(w10, c0), cscale(w11, c1));
}

ORC_EXPORT int orc_cir_fields(const OrcScene* S, const OrcFieldParams* P, const OrcRecords* R,
                              const double* pv, const int32_t* status, int64_t n, double* gain,
                              double* delay, double* doppler, double* dep, double* arr) {
  const int L = R->L;
  const double lam = P->wavelength;
  for (int64_t r = 0; r < n; ++r) {
    if (status[r] != SBR_REFINE_OK) continue;
    const int depth = R->depth[r], tgt = R->target[r];
    const double* V = pv + r * (int64_t)(L + 2) * 3;
    double seg[17], kh[17][3], total = 0.0;
    for (int i = 0; i <= depth; ++i) {
      double s3[3] = {V[3 * (i + 1)] - V[3 * i], V[3 * (i + 1) + 1] - V[3 * i + 1], V[3 * (i + 1) + 2] - V[3 * i + 2]};
      seg[i] = norm_seq(s3);
      for (int k = 0; k < 3; ++k) kh[i][k] = s3[k] / seg[i];
      total += seg[i];
    }
    double cth, cph, fa[3], fb[3];
    pattern_gcs(&P->tx, kh[0], &cth, &cph, fa, fb);
    cpx c0 = C(cth, 0.0), c1 = C(cph, 0.0);
    double gamma_prob = 1.0, r_dist = 0.0, tube = FOUR_PI / (double)P->num_samples;
    int n_phase = 0;
    char tag[32];
    int len = 0;
    {
      const char* pre = "phase-";
      while (pre[len]) { tag[len] = pre[len]; ++len; }
      char dg[12];
      int nd = 0, v = depth;
      do { dg[nd++] = (char)('0' + v % 10); v /= 10; } while (v > 0);
      while (nd > 0) tag[len++] = dg[--nd];
      tag[len] = 0;
    }
    const uint64_t ptag = orc_tag_hash(tag);
    const uint64_t psample = R->sample[r] > 0 ? (uint64_t)R->sample[r] : 0ULL;
    int has_s = 0, has_d = 0, diffracted = 0;
    double s_dist = 0.0;
    double nu = dot_ddot(P->tx_vel, kh[0]) / lam;
    nu -= dot_ddot(P->rx_vel + 3 * tgt, kh[depth]) / lam;
    for (int i = 0; i < depth; ++i) {
      const int64_t o = r * L + i;
      const int kind = R->kind[o], slot = R->tri[o];
      const int row = S->matrow[slot];
      const SbrMaterial* m = S->mats + row;
      const double* k_in = kh[i];
      const double* k_out = kh[i + 1];
      r_dist += seg[i];
      const double* nrm = R->normal + 3 * o;
      double nh[3] = {nrm[0], nrm[1], nrm[2]};
      if (dot_ddot(k_in, nh) > 0.0) { nh[0] = -nh[0]; nh[1] = -nh[1]; nh[2] = -nh[2]; }
      double q[4];
      interaction_q(m, fabs(dot_ddot(k_in, nrm)), P->q_d,
                    allowed_kinds(S, P->allow, slot, has_s, has_d), q);
      gamma_prob *= q[kind];
      if (P->obj_vel) {
        const double* v = P->obj_vel + 3 * row;
        if (v[0] != 0.0 || v[1] != 0.0 || v[2] != 0.0) {
          double dk[3] = {k_out[0] - k_in[0], k_out[1] - k_in[1], k_out[2] - k_in[2]};
          nu += dot_ddot(v, dk) / lam;
        }
      }
      double ep[3], el[3];
      incidence_frame(k_in, nh, ep, el);
      double cos_t = fabs(dot_ddot(k_in, nh));
      Fresnel4 F = slab_fresnel(m, cos_t);
      if (kind == 3) {
        /* UTD wedge transfer (paths.py:1358-1373) */
        const int w = R->wedge[o];
        double remaining = 0.0;
        for (int q2 = i + 1; q2 <= depth; ++q2) remaining += seg[q2];
        M2 T;
        double bi[2][3], bo[2][3];
        if (utd_transfer(S, w, k_in, k_out, r_dist, remaining, lam, &T, bi, bo)) {
          c0 = c1 = C(0.0, 0.0);
        } else {
          cpx p0, p1;
          basis_w(bi[0], bi[1], fa, fb, c0, c1, &p0, &p1);
          cpx n0_ = cadd(cmul(T.m[0][0], p0), cmul(T.m[0][1], p1));
          cpx n1_ = cadd(cmul(T.m[1][0], p0), cmul(T.m[1][1], p1));
          c0 = n0_; c1 = n1_;
          double cr[3];
          cross3(bo[0], bo[1], cr);
          if (dot_ddot(cr, k_out) < 0.0) {
            cpx t = c0; c0 = c1; c1 = t;
            memcpy(fa, bo[1], sizeof fa); memcpy(fb, bo[0], sizeof fb);
          } else {
            memcpy(fa, bo[0], sizeof fa); memcpy(fb, bo[1], sizeof fb);
          }
        }
        s_dist = r_dist;
        r_dist = 0.0;
        diffracted = 1;
        has_d = 1;
        continue;
      }
      if (kind == 0 || kind == 2) {
        cpx p0, p1;
        basis_w(ep, el, fa, fb, c0, c1, &p0, &p1);
        double na[3], nb[3], kk[3];
        if (kind == 0) {
          double dn = dot_ddot(k_in, nh);
          for (int k = 0; k < 3; ++k) kk[k] = k_in[k] - 2.0 * dn * nh[k];
          double erp[3];
          cross3(ep, kk, erp);
          c0 = cscale(m->spec_amp, cmul(F.rp, p0));
          c1 = cscale(m->spec_amp, cmul(F.rl, p1));
          memcpy(na, ep, sizeof na); memcpy(nb, erp, sizeof nb);
        } else {
          memcpy(kk, k_in, sizeof kk);
          c0 = cmul(F.tp, p0);
          c1 = cmul(F.tl, p1);
          memcpy(na, ep, sizeof na); memcpy(nb, el, sizeof nb);
        }
        double cr[3];
        cross3(na, nb, cr);
        if (dot_ddot(cr, kk) < 0.0) { /* _right_handed (paths.py:1259-1273) */
          cpx t = c0; c0 = c1; c1 = t;
          memcpy(fa, nb, sizeof fa); memcpy(fb, na, sizeof fb);
        } else {
          memcpy(fa, na, sizeof fa); memcpy(fb, nb, sizeof fb);
        }
      } else {
        cpx p0, p1;
        basis_w(ep, el, fa, fb, c0, c1, &p0, &p1);
        double norm_in = sqrt(cabs2(p0) + cabs2(p1));
        double gam = norm_in == 0.0 ? 0.0 : sqrt(cabs2(cmul(F.rp, p0)) + cabs2(cmul(F.rl, p1))) / norm_in;
        double ci = -dot_ddot(k_in, nh);
        double patch = tube * (r_dist * r_dist) / (ci > 1e-12 ? ci : 1e-12);
        ci = ci < 0.0 ? 0.0 : (ci > 1.0 ? 1.0 : ci);
        double f_s = pattern_density(m, k_in, k_out, nh);
        double amp = m->scattering * gam * sqrt(f_s * ci * patch);
        double chi1 = 0.0, chi2 = 0.0;
        if (m->random_phases) {
          chi1 = TWO_PI * orc_philox_uniform(P->seed, psample, (uint64_t)tgt, ptag, 2 * n_phase);
          chi2 = TWO_PI * orc_philox_uniform(P->seed, psample, (uint64_t)tgt, ptag, 2 * n_phase + 1);
          ++n_phase;
        }
        double sq = sqrt(1.0 - m->xpd_kx), sk = sqrt(m->xpd_kx);
        double thi[3], phi_[3], ths[3], phs[3];
        transverse(k_in, thi, phi_);
        transverse(k_out, ths, phs);
        cpx q0, q1;
        basis_w(thi, phi_, fa, fb, c0, c1, &q0, &q1);
        cpx e1 = C(cos(chi1), sin(chi1)), e2 = C(cos(chi2), sin(chi2));
        cpx o0 = cscale(amp, cadd(cmul(cscale(sq, e1), q0), cmul(cscale(-sk, e1), q1)));
        cpx o1 = cscale(amp, cadd(cmul(cscale(sk, e2), q0), cmul(cscale(sq, e2), q1)));
        double inv = 1.0 / sqrt(gamma_prob);
        c0 = C(o0.re / r_dist * inv, o0.im / r_dist * inv);
        c1 = C(o1.re / r_dist * inv, o1.im / r_dist * inv);
        memcpy(fa, ths, sizeof fa); memcpy(fb, phs, sizeof fb);
        gamma_prob = 1.0;
        r_dist = 0.0;
        tube = TWO_PI;
        has_s = 1;
      }
    }
    r_dist += seg[depth];
    double na[3] = {-kh[depth][0], -kh[depth][1], -kh[depth][2]};
    double rc0, rc1, rth[3], rph[3];
    pattern_gcs(P->rx + tgt, na, &rc0, &rc1, rth, rph);
    cpx acc = C(0.0, 0.0);
    for (int k = 0; k < 3; ++k) {
      cpx e = cadd(cscale(fa[k], c0), cscale(fb[k], c1));
      double rv = rc0 * rth[k] + rc1 * rph[k];
      acc = cadd(acc, cscale(rv, e));
    }
    double sc = lam / FOUR_PI;
    double dv = diffracted ? sqrt(s_dist * r_dist * (s_dist + r_dist)) : r_dist;
    gain[2 * r] = acc.re * sc / dv;
    gain[2 * r + 1] = acc.im * sc / dv;
    delay[r] = total / 299792458.0;
    doppler[r] = nu;
    memcpy(dep + 3 * r, kh[0], 3 * sizeof(double));
    memcpy(arr + 3 * r, kh[depth], 3 * sizeof(double));
  }
  return 0;
}

/* frequency_response (paths.py:1519-1547), path order accumulation */
ORC_EXPORT void orc_cfr(const double* gain, const double* delay, const double* dep,
                        const double* arr, const int32_t* prx, const int32_t* ptx, int64_t np,
                        const double* freqs, int32_t nf, const double* txo, int32_t ntx,
                        const double* rxo, int32_t nrx, double wavelength, int32_t synthetic,
                        double* H) {
  memset(H, 0, sizeof(double) * 2 * (size_t)nrx * ntx * nf);
  const double kw = TWO_PI / wavelength;
  for (int64_t p = 0; p < np; ++p) {
    cpx a = C(gain[2 * p], gain[2 * p + 1]);
    for (int r = 0; r < nrx; ++r)
      for (int t = 0; t < ntx; ++t) {
        cpx v = a;
        if (synthetic) {
          double nk[3] = {-arr[3 * p], -arr[3 * p + 1], -arr[3 * p + 2]};
          double pr = kw * dot_gemv(rxo + 3 * r, nk), pt = kw * dot_gemv(txo + 3 * t, dep + 3 * p);
          v = cmul(cmul(v, C(cos(pr), sin(pr))), C(cos(pt), sin(pt)));
        } else if (prx[p] != r || ptx[p] != t) {
          continue;
        }
        for (int f = 0; f < nf; ++f) {
          double ang = -TWO_PI * freqs[f] * delay[p];
          cpx w = cmul(v, C(cos(ang), sin(ang)));
          double* h = H + 2 * (((int64_t)r * ntx + t) * nf + f);
          h[0] += w.re;
          h[1] += w.im;
        }
      }
  }
}

/* ========================================================================= */
/* Edge (diffraction) radio-map estimator: compute_radio_map_diffraction     */
/* (radiomap.py:842-965) with _cone_points / _weighting_rows / _utd_rows       */
/* ========================================================================= */
#define TAG_MAP_WEDGE 0x9115590451c40950ULL

static void cone_point(const OrcScene* S, int w, const double* src, double x, double phi,
                       double* v, double* s_in, double* k_i, double* k_s, double* sin_b) {
  const double* o = S->w_origin + 3 * w;
  const double* e = S->w_ehat + 3 * w;
  const double* t0 = S->w_t0 + 3 * w;
  const double* n0 = S->w_n0 + 3 * w;
  for (int k = 0; k < 3; ++k) v[k] = o[k] + x * e[k];
  double d[3] = {v[0] - src[0], v[1] - src[1], v[2] - src[2]};
  *s_in = norm_seq(d);
  for (int k = 0; k < 3; ++k) k_i[k] = d[k] / *s_in;
  double cb = dot_gemv(d, e) / *s_in;
  double xb = 1.0 - cb * cb;
  *sin_b = sqrt(xb > 0.0 ? xb : 0.0);
  double a = *sin_b * cos(phi), b = *sin_b * sin(phi);
  for (int k = 0; k < 3; ++k) k_s[k] = (a * t0[k] + b * n0[k]) + cb * e[k];
}

ORC_EXPORT int orc_radiomap_wedges(const OrcScene* S, const SbrMapParams* P, const double* offs,
                                   const double* prec, const int32_t* wedge_ids, int32_t nw,
                                   uint64_t wedge_samples, double* grid, uint64_t* counters) {
  const double* nh = P->normal;
  const double lam = P->wavelength;
  for (int wi = 0; wi < nw; ++wi) {
    const int w = wedge_ids[wi];
    const double len = S->w_len[w], nopen = S->w_nopen[w];
    const double norm = len * nopen * PI_ / (double)wedge_samples;
    const double hx = 1e-4 * (len > 1.0 ? len : 1.0), hp = 1e-4;
    for (uint64_t i = 0; i < wedge_samples; ++i) {
      const uint64_t block = i >> SBR_CHUNK_LOG2, slot = i & ((1ULL << SBR_CHUNK_LOG2) - 1);
      counters[SBR_MC_CONE_SAMPLES]++;
      double u0 = orc_philox_uniform(P->seed, (uint64_t)w, block, TAG_MAP_WEDGE, 2 * slot);
      double u1 = orc_philox_uniform(P->seed, (uint64_t)w, block, TAG_MAP_WEDGE, 2 * slot + 1);
      double xs = u0 * len, phis = u1 * nopen * PI_;
      double v[3], s_in, k_i[3], k_s[3], sin_b;
      cone_point(S, w, P->source, xs, phis, v, &s_in, k_i, k_s, &sin_b);
      if (!(sin_b >= 1e-9)) continue;
      double denom = dot_gemv(k_s, nh);
      if (!(fabs(denom) > 1e-9)) continue;
      double gamma = (P->plane_off - dot_gemv(v, nh)) / denom;
      if (!(gamma > 1e-4)) continue;
      double inc[3] = {-k_i[0], -k_i[1], -k_i[2]};
      double azim = atan2(dot_gemv(inc, S->w_n0 + 3 * w), dot_gemv(inc, S->w_t0 + 3 * w));
      if (azim < 0.0) azim += 2.0 * PI_;
      if (!(azim <= nopen * PI_)) continue;
      double pts[3] = {v[0] + gamma * k_s[0], v[1] + gamma * k_s[1], v[2] + gamma * k_s[2]};
      double rel[3] = {pts[0] - P->corner[0], pts[1] - P->corner[1], pts[2] - P->corner[2]};
      double fu = floor(dot_gemv(rel, P->u_hat) / P->cell_w);
      double fv = floor(dot_gemv(rel, P->v_hat) / P->cell_h);
      if (!(fu >= 0.0 && fu < (double)P->nx && fv >= 0.0 && fv < (double)P->ny)) continue;
      int occ;
      if (occluded1(S, P->source, v, 1e-4, &occ)) return SBR_ERR_STACK;
      if (occ) continue;
      if (occluded1(S, v, pts, 1e-4, &occ)) return SBR_ERR_STACK;
      if (occ) continue;
      M2 T;
      double bi[2][3], bo[2][3];
      if (utd_transfer(S, w, k_i, k_s, s_in, gamma, lam, &T, bi, bo)) continue;
      /* _weighting_rows: central differences of the plane crossing */
      double cr[4][3];
      const double xv[4] = {xs + hx, xs - hx, xs, xs}, pvv[4] = {phis, phis, phis + hp, phis - hp};
      int bad = 0;
      for (int q = 0; q < 4; ++q) {
        double vq[3], sq, kiq[3], ksq[3], sbq;
        cone_point(S, w, P->source, xv[q], pvv[q], vq, &sq, kiq, ksq, &sbq);
        double dq = dot_gemv(ksq, nh);
        if (fabs(dq) < 1e-9) { bad = 1; dq = 1.0; }
        double gq = (P->plane_off - dot_gemv(vq, nh)) / dq;
        for (int k = 0; k < 3; ++k) cr[q][k] = vq[k] + gq * ksq[k];
      }
      if (bad) continue;
      double ddx[3], ddp[3], cx[3];
      for (int k = 0; k < 3; ++k) {
        ddx[k] = (cr[0][k] - cr[1][k]) / (2.0 * hx);
        ddp[k] = (cr[2][k] - cr[3][k]) / (2.0 * hp);
      }
      cross3(ddx, ddp, cx);
      double factor = norm_seq(cx);
      cpx E[3];
      pattern_field(&P->pattern, k_i, E);
      cpx c0 = cdot_real(E, bi[0]), c1 = cdot_real(E, bi[1]);
      cpx o0 = cadd(cmul(T.m[0][0], c0), cmul(T.m[0][1], c1));
      cpx o1 = cadd(cmul(T.m[1][0], c0), cmul(T.m[1][1], c1));
      double spread = s_in * gamma * (s_in + gamma);
      double e_p = (cabs2(o0) + cabs2(o1)) / spread;
      double a_sq = alpha_sq(P, offs, prec, k_i);
      grid[(int64_t)fv * P->nx + (int64_t)fu] += norm * P->scale * e_p * factor * a_sq;
      counters[SBR_MC_DEPOSITS]++;
    }
  }
  return 0;
}
