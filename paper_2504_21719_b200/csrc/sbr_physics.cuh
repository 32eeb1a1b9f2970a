// sbr_physics.cuh -- per-hit electromagnetic operators (float64 / complex128).
//
// Device versions of the reference's numpy material and antenna math:
//   slab_fresnel        ITU-R P.2040 slab over vacuum Fresnel (materials.py:163-245)
//   pattern_density     Lambertian / directive / backscattering lobes (354-397)
//   antenna_field       isotropic / TR 38.901 launch field (em.py:258-308,
//                       radiomap.py:266-277), precoding |alpha|^2 (253-259)
//   incidence_frame     (e_perp, e_par) with the deterministic perpendicular
//                       fallback (radiomap.py:291-300, em.py:96-107)
//   perp_batch / transverse_rows (sampling.py:179-190, radiomap.py:280-288)
// Operation order follows the numpy expressions so a float64 result differs
// from the reference only where CUDA's libm differs from numpy's by an ulp.
#pragma once

#include "sbr_common.cuh"

namespace sbr {

#ifndef SBR_FRESNEL_EXP_LOOP
#define SBR_FRESNEL_EXP_LOOP 0
#endif

struct Fresnel4 {
  cplx rp, rl, tp, tl;
};

__device__ __forceinline__ cplx csqrt_lossy(cplx z) {
  const cplx s = csqrt_(z);
  return s.im > 0.0 ? C(-s.re, -s.im) : s;
}

__device__ __forceinline__ Fresnel4 slab_fresnel(const SbrMaterial& m, double c0) {
  Fresnel4 f;
  const cplx eta = C(m.eta_re, m.eta_im);
  const double sin2 = 1.0 - c0 * c0;
  const cplx root = csqrt_lossy(C(eta.re - sin2, eta.im));
  if (m.thickness == 0.0) {
    f.rp = C(0.0, 0.0);
    f.rl = C(0.0, 0.0);
    f.tp = C(1.0, 0.0);
    f.tl = C(1.0, 0.0);
    return f;
  }
  const cplx c_plus = C(c0 + root.re, root.im);
  const cplx ec = C(eta.re * c0, eta.im * c0);
  cplx r_perp = cdiv(C(c0 - root.re, -root.im), c_plus);
  cplx r_par = cdiv(ec - root, ec + root);
  if (eta.im == 0.0 && sin2 >= cabs_np(eta)) {
    r_perp = C(1.0, 0.0);
    r_par = C(1.0, 0.0);
  }
  const cplx q = m.kd * root;
#if SBR_FRESNEL_EXP_LOOP
  // both exponentials through one inlined cexp_ (a 2-trip loop): half the
  // code of two inlined copies, no call
  cplx phase2, phase1;
#pragma unroll 1
  for (int k = 0; k < 2; ++k) {
    const cplx e = cexp_(k == 0 ? C(2.0 * q.im, -2.0 * q.re) : C(q.im, -q.re));
    if (k == 0) phase2 = e;  // exp(-2j q)
    else phase1 = e;         // exp(-1j q)
  }
#else
  const cplx phase2 = cexp_(C(2.0 * q.im, -2.0 * q.re));  // exp(-2j q)
  const cplx phase1 = cexp_(C(q.im, -q.re));              // exp(-1j q)
#endif
  const cplx one_m_p2 = C(1.0 - phase2.re, -phase2.im);
  {
    const cplx r1sq = r_perp * r_perp;
    const cplx z = r1sq * phase2;
    const cplx den = C(1.0 - z.re, -z.im);
#if SBR_CDIV2
    const cplx2 q = cdiv2(r_perp * one_m_p2, C(1.0 - r1sq.re, -r1sq.im) * phase1, den);
    f.rp = q.x;
    f.tp = q.y;
#else
    f.rp = cdiv(r_perp * one_m_p2, den);
    f.tp = cdiv(C(1.0 - r1sq.re, -r1sq.im) * phase1, den);
#endif
  }
  {
    const cplx r1sq = r_par * r_par;
    const cplx z = r1sq * phase2;
    const cplx den = C(1.0 - z.re, -z.im);
#if SBR_CDIV2
    const cplx2 q = cdiv2(r_par * one_m_p2, C(1.0 - r1sq.re, -r1sq.im) * phase1, den);
    f.rl = q.x;
    f.tl = q.y;
#else
    f.rl = cdiv(r_par * one_m_p2, den);
    f.tl = cdiv(C(1.0 - r1sq.re, -r1sq.im) * phase1, den);
#endif
  }
  return f;
}

__device__ __forceinline__ double binom(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
  return floor(r + 0.5);
}

static __device__ double lobe_norm(int alpha, double cos_ti) {
  double sin2 = 1.0 - cos_ti * cos_ti;
  if (sin2 < 0.0) sin2 = 0.0;
  double total = 0.0;
  for (int k = 0; k <= alpha; ++k) {
    double ik;
    if ((k & 1) == 0) {
      ik = kTwoPi / (double)(k + 1);
    } else {
      double inner = 0.0;
      for (int w = 0; w <= (k - 1) / 2; ++w)
        inner = inner + binom(2 * w, w) * pow(sin2 / 4.0, (double)w);
      ik = kTwoPi / (double)(k + 1) * cos_ti * inner;
    }
    total = total + binom(alpha, k) * ik;
  }
  return total / pow(2.0, (double)alpha);
}

__device__ __forceinline__ double clamp1(double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); }

// the Lambertian lobe of pattern_density (materials.py:354-397)
__device__ __forceinline__ double lambert_density(double3 ks, double3 n) {
  double c = dot_seq(ks, n);
  c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
  return c / kPi;
}

static __device__ double pattern_density(const SbrMaterial& m, double3 ki, double3 ks, double3 n) {
  if (m.pattern_kind == SBR_SCAT_LAMBERTIAN) return lambert_density(ks, n);
  const double ci = clamp1(-dot_seq(ki, n));
  const double kn = dot_seq(ki, n);
  const double3 kr = ki - (2.0 * kn) * n;
  const double lobe_r = pow((1.0 + dot_seq(kr, ks)) / 2.0, (double)m.alpha_r);
  if (m.pattern_kind == SBR_SCAT_DIRECTIVE) return lobe_r / lobe_norm(m.alpha_r, ci);
  const double lobe_i = pow((1.0 - dot_seq(ki, ks)) / 2.0, (double)m.alpha_i);
  const double lam = m.lambda_mix;
  const double nrm = lam * lobe_norm(m.alpha_r, ci) + (1.0 - lam) * lobe_norm(m.alpha_i, ci);
  return (lam * lobe_r + (1.0 - lam) * lobe_i) / nrm;
}

// zenith / azimuth unit vectors of a direction (radiomap.py:280-288)
__device__ __forceinline__ void transverse_rows(double3 d, double3& th, double3& ph) {
  const double theta = acos(clamp1(d.z));
  const double phi = atan2(d.y, d.x);
  double st, ct, sp, cp;
  sincos(theta, &st, &ct);
  sincos(phi, &sp, &cp);
  th = make_double3(ct * cp, ct * sp, -st);
  ph = make_double3(-sp, cp, 0.0);
}

__device__ __forceinline__ double tr38901_amp(double scale, double theta, double phi) {
  const double theta_deg = theta * (180.0 / kPi);
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double phi_deg = atan2(sp, cp) * (180.0 / kPi);
  const double a = (theta_deg - 90.0) / 65.0;
  double av = 12.0 * (a * a);
  av = -(av < 30.0 ? av : 30.0);
  const double b = phi_deg / 65.0;
  double ah = 12.0 * (b * b);
  ah = -(ah < 30.0 ? ah : 30.0);
  const double s = -(av + ah);
  const double g = -(s < 30.0 ? s : 30.0) + 8.0;
  return scale * pow(10.0, g / 20.0);
}

// World-frame launch field of a departure direction (radiomap.py:266-277).
static __device__ cvec3 antenna_field(const SbrAntenna& a, double3 d) {
  double3 local;
  if (a.identity) {
    local = d;
  } else {
    local = make_double3(dot_gemv(d, make_double3(a.rot[0], a.rot[3], a.rot[6])),
                         dot_gemv(d, make_double3(a.rot[1], a.rot[4], a.rot[7])),
                         dot_gemv(d, make_double3(a.rot[2], a.rot[5], a.rot[8])));
  }
  const double theta = acos(clamp1(local.z));
  const double phi = atan2(local.y, local.x);
  const double cth = a.kind == SBR_PATTERN_TR38901 ? tr38901_amp(a.scale, theta, phi) : 1.0;
  double st, ct, sp, cp;
  sincos(theta, &st, &ct);
  sincos(phi, &sp, &cp);
  double3 th = make_double3(ct * cp, ct * sp, -st);
  if (!a.identity) {
    th = make_double3(dot_gemv(th, make_double3(a.rot[0], a.rot[1], a.rot[2])),
                      dot_gemv(th, make_double3(a.rot[3], a.rot[4], a.rot[5])),
                      dot_gemv(th, make_double3(a.rot[6], a.rot[7], a.rot[8])));
  }
  cvec3 E;
  E.x = C(cth * th.x, 0.0);
  E.y = C(cth * th.y, 0.0);
  E.z = C(cth * th.z, 0.0);
  return E;
}

// antenna_field for an isotropic, unrotated pattern: the same operations on
// local = d with cth = 1 (bit-identical), without the other patterns' code
__device__ __forceinline__ cvec3 antenna_iso(double3 d) {
  const double theta = acos(clamp1(d.z));
  const double phi = atan2(d.y, d.x);
  double st, ct, sp, cp;
  sincos(theta, &st, &ct);
  sincos(phi, &sp, &cp);
  cvec3 E;
  E.x = C(1.0 * (ct * cp), 0.0);
  E.y = C(1.0 * (ct * sp), 0.0);
  E.z = C(1.0 * -st, 0.0);
  return E;
}

// |sum_m exp(j k d.o_m) u_m|^2 (radiomap.py:253-259)
static __device__ double alpha_sq(const SbrMapParams& P, double3 d) {
  if (P.n_elements <= 0) return 1.0;
  const double k = kTwoPi / P.wavelength;
  cplx acc = C(0.0, 0.0);
  for (int m = 0; m < P.n_elements; ++m) {
    const double ph = k * dot_gemv(d, ldg3(P.elem_offsets_dev + 3 * m));
    double s, c;
    sincos(ph, &s, &c);
    const cplx u = C(__ldg(P.precoder_dev + 2 * m), __ldg(P.precoder_dev + 2 * m + 1));
    acc = acc + C(c, s) * u;
  }
  return cabs2(acc);
}

// deterministic_perpendicular (em.py:96-107): projected x, else y axis --
// the normal-incidence branch of incidence_frame, kept out of line (cold)
static __device__ __noinline__ double3 deterministic_perp(double3 k) {
  const double ax = k.x;  // x_axis . k via ddot == k.x exactly
  double3 u = make_double3(1.0 - ax * k.x, 0.0 - ax * k.y, 0.0 - ax * k.z);
  double un = sqrt(dot_ddot(u, u));
  if (!(un > 1e-9)) {
    const double ay = k.y;
    u = make_double3(0.0 - ay * k.x, 1.0 - ay * k.y, 0.0 - ay * k.z);
    un = sqrt(dot_ddot(u, u));
  }
  return make_double3(u.x / un, u.y / un, u.z / un);
}

// (e_perp, e_par) of an incident ray on a surface (radiomap.py:291-300)
__device__ __forceinline__ void incidence_frame(double3 k, double3 n, double3& e_perp,
                                                double3& e_par) {
  double3 cr = cross3(k, n);
  double nrm = norm_seq(cr);
  if (nrm < 1e-9) {
    cr = deterministic_perp(k);
    nrm = 1.0;
  }
  e_perp = SBR_DIV3(cr, nrm);
  e_par = cross3(e_perp, k);
}

// _perpendicular_batch (sampling.py:179-190)
__device__ __forceinline__ double3 perp_batch(double3 v) {
  double3 c = make_double3(1.0 - v.x * v.x, 0.0 - v.x * v.y, 0.0 - v.x * v.z);
  double nrm = norm_seq(c);
  if (nrm <= 1e-9) {
    c = make_double3(0.0 - v.y * v.x, 1.0 - v.y * v.y, 0.0 - v.y * v.z);
    nrm = norm_seq(c);
  }
  return make_double3(c.x / nrm, c.y / nrm, c.z / nrm);
}

}  // namespace sbr
