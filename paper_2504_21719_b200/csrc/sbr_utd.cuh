// sbr_utd.cuh -- first-order diffraction on the device (SURVEY.md §8f "next" #1).
//
//   project_wedge        _project_diffractions (paths.py:831-852)
//   allowed_kinds        interaction masks (paths.py:743-748, 1276-1299)
//   solve_diffraction_point, rotate_about (paths.py:517-565)
//   fresnel_sc, transition_f, cot_f, fresnel_vacuum_r, utd_transfer
//                        (materials.py:173-205, 482-646; scipy.special.fresnel)
// Float64 throughout; the CPU oracle (oracle/sbr_oracle.c) carries the same
// restatement and both are pinned to the reference's golden diffraction paths.
#pragma once

#include "sbr_physics.cuh"

namespace sbr {

constexpr uint64_t TAG_CONE = 0x0bc9fb91195d708aULL;  // fnv1a("cone")

__device__ __forceinline__ bool owns_wedge(const DevScene& S, int tri) {
  return S.n_wedges > 0 && __ldg(S.slot_woff + tri + 1) > __ldg(S.slot_woff + tri);
}

// bit0 R, bit1 S, bit2 T, bit3 D
__device__ __forceinline__ int allowed_kinds(const DevScene& S, int allow, int tri, bool has_s,
                                             bool has_d) {
  int a = allow & 15;
  if (has_d) a &= ~2;
  if (has_d || has_s) a &= ~8;
  if (!owns_wedge(S, tri)) a &= ~8;
  return a;
}

// nearest owned wedge of a slot, clamped foot point (first minimum in CSR order)
__device__ __forceinline__ int project_wedge(const DevScene& S, int tri, double3 p, double3& foot) {
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int bw = -1;
  for (int k = __ldg(S.slot_woff + tri); k < __ldg(S.slot_woff + tri + 1); ++k) {
    const int w = __ldg(S.slot_wids + k);
    const double3 o = ldg3(S.w_origin + 3 * w), e = ldg3(S.w_ehat + 3 * w);
    double x = dot_seq(p - o, e);
    const double len = __ldg(S.w_len + w);
    x = x < 0.0 ? 0.0 : (x > len ? len : x);
    const double3 f = o + x * e;
    const double dist = norm_seq(p - f);
    if (dist < best) {
      best = dist;
      bw = w;
      foot = f;
    }
  }
  return bw;
}

__device__ __forceinline__ double3 reflect_vec(double3 v, double3 nrm) {
  const double f = dot_ddot(v, nrm);
  return v - (2.0 * f) * nrm;
}

// returns false when degenerate
__device__ __forceinline__ bool solve_diffraction_point(double3 src, double3 tgt, double3 eo,
                                                        double3 ed, double& x_out) {
  const double en = sqrt(dot_ddot(ed, ed));
  const double3 e = make_double3(ed.x / en, ed.y / en, ed.z / en);
  const double3 sv = src - eo, tv = tgt - eo;
  double3 u1 = sv - dot_ddot(e, sv) * e, u2 = tv - dot_ddot(e, tv) * e;
  const double n1 = sqrt(dot_ddot(u1, u1)), n2 = sqrt(dot_ddot(u2, u2));
  if (n1 < 1e-12 || n2 < 1e-12) return false;
  u1 = make_double3(u1.x / n1, u1.y / n1, u1.z / n1);
  u2 = make_double3(u2.x / n2, u2.y / n2, u2.z / n2);
  double3 ax = cross3(u1, u2);
  const double na = sqrt(dot_ddot(ax, ax));
  ax = na < 1e-12 ? e : make_double3(ax.x / na, ax.y / na, ax.z / na);
  const double angle = kPi - acos(clamp1(dot_ddot(u1, u2)));
  double sa, ca;
  sincos(angle, &sa, &ca);
  const double a[3] = {ax.x, ax.y, ax.z};
  const double K[9] = {0.0, -a[2], a[1], a[2], 0.0, -a[0], -a[1], a[0], 0.0};
  double R[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = (ca * (i == j ? 1.0 : 0.0) + sa * K[3 * i + j]) + (1.0 - ca) * (a[i] * a[j]);
  const double3 tr = make_double3(dot_gemv(make_double3(R[0], R[1], R[2]), tv),
                                  dot_gemv(make_double3(R[3], R[4], R[5]), tv),
                                  dot_gemv(make_double3(R[6], R[7], R[8]), tv));
  const double3 st = tr - sv;
  const double3 guide = cross3(e, st);
  const double ng = sqrt(dot_ddot(guide, guide));
  if (ng < 1e-12) return false;
  const double3 lever = cross3(sv, st);
  const double sign = dot_ddot(guide, lever) >= 0.0 ? 1.0 : -1.0;
  x_out = sign * (sqrt(dot_ddot(lever, lever)) / ng);
  return true;
}

// Fresnel integrals S, C (power series below 1.5, continued fraction above)
__device__ __forceinline__ void fresnel_sc(double x, double& s_out, double& c_out) {
  const double ax = fabs(x);
  double s, c;
  if (ax < 1.5) {
    const double t = 1.5707963267948966 * ax * ax;
    double term = ax, sumc = 0.0, sums = 0.0;
    for (int k = 0; k < 60; ++k) {
      const double contrib = term / (2 * k + 1);
      const double sign = ((k / 2) % 2) ? -1.0 : 1.0;
      if (k % 2 == 0) sumc += sign * contrib;
      else sums += sign * contrib;
      term *= t / (k + 1);
      if (term < 1e-18 * (sumc + sums + 1e-300)) break;
    }
    c = sumc;
    s = sums;
  } else {
    const double pix2 = kPi * ax * ax;
    cplx b = C(1.0, -pix2), cc = C(1e300, 0.0);
    cplx d = cdiv(C(1.0, 0.0), b), h = d;
    int n = -1;
    for (int k = 2; k < 300; ++k) {
      n += 2;
      const double a = -(double)n * (double)(n + 1);
      b = C(b.re + 4.0, b.im);
      d = cdiv(C(1.0, 0.0), a * d + b);
      cc = b + cdiv(C(a, 0.0), cc);
      const cplx del = cc * d;
      h = h * del;
      if (fabs(del.re - 1.0) + fabs(del.im) < 1e-16) break;
    }
    h = h * C(ax, -ax);
    double sp, cp;
    sincos(0.5 * pix2, &sp, &cp);
    const cplx w = C(cp, sp) * h;
    const cplx cs = C(0.5, 0.5) * C(1.0 - w.re, -w.im);
    c = cs.re;
    s = cs.im;
  }
  if (x < 0.0) {
    c = -c;
    s = -s;
  }
  s_out = s;
  c_out = c;
}

__device__ __forceinline__ cplx transition_f(double x) {
  double s, c;
  fresnel_sc(sqrt(2.0 * x / kPi), s, c);
  double sx, cx;
  sincos(x, &sx, &cx);
  return sqrt(kPi * x / 2.0) * (C(cx, sx) * C(1.0 - 2.0 * s, 1.0 - 2.0 * c));
}

__device__ __forceinline__ cplx cot_f(double beta, double n_open, double k, double l, double sign) {
  const double n_round = nearbyint((beta + sign * kPi) / (2.0 * n_open * kPi));
  const double eps = beta - (2.0 * n_open * kPi * n_round - sign * kPi);
  if (fabs(eps) < 1e-6) {
    const double sg = eps >= 0.0 ? 1.0 : -1.0, kl = k * l;
    const cplx q = C(cos(kPi / 4.0), sin(kPi / 4.0));
    const cplx inner = C(sqrt(2.0 * kPi * kl) * sg, 0.0) - (2.0 * kl * eps) * q;
    return (sign * n_open) * (q * inner);
  }
  const double cot = 1.0 / tan((kPi + sign * beta) / (2.0 * n_open));
  const double cv = cos((2.0 * n_open * kPi * n_round - beta) / 2.0);
  return cot * transition_f(k * l * (2.0 * cv * cv));
}

__device__ __forceinline__ void fresnel_vacuum_r(double c1, double eta_re, double eta_im,
                                                 cplx& rp, cplx& rl) {
  const double sin2 = 1.0 - c1 * c1;
  const cplx root = csqrt_lossy(C(eta_re - sin2, eta_im));
  rp = cdiv(C(c1 - root.re, -root.im), C(c1 + root.re, root.im));
  const cplx ec = C(eta_re * c1, eta_im * c1);
  rl = cdiv(ec - root, ec + root);
  if (eta_im == 0.0 && sin2 >= cabs_np(C(eta_re, eta_im))) {
    rp = C(1.0, 0.0);
    rl = C(1.0, 0.0);
  }
}

struct M2 {
  cplx m[2][2];
};

__device__ __forceinline__ M2 m2_mul(const M2& a, const M2& b) {
  M2 r;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j];
  return r;
}

__device__ __forceinline__ M2 m2_w(double3 a, double3 b, double3 q, double3 r) {
  M2 w;
  w.m[0][0] = C(dot_ddot(a, q), 0.0);
  w.m[0][1] = C(dot_ddot(a, r), 0.0);
  w.m[1][0] = C(dot_ddot(b, q), 0.0);
  w.m[1][1] = C(dot_ddot(b, r), 0.0);
  return w;
}

__device__ __forceinline__ void oblique_frame(double3 s_hat, double3 n_hat, double3 other,
                                              double3& e_perp, double3& e_par) {
  const double3 cr = cross3(s_hat, n_hat);
  const double nn = sqrt(dot_ddot(cr, cr));
  if (nn < 1e-9) {
    const double av = s_hat.x;
    double3 u = make_double3(1.0 - av * s_hat.x, 0.0 - av * s_hat.y, 0.0 - av * s_hat.z);
    double un = sqrt(dot_ddot(u, u));
    if (!(un > 1e-9)) {
      const double ay = s_hat.y;
      u = make_double3(0.0 - ay * s_hat.x, 1.0 - ay * s_hat.y, 0.0 - ay * s_hat.z);
      un = sqrt(dot_ddot(u, u));
    }
    e_perp = make_double3(u.x / un, u.y / un, u.z / un);
  } else {
    e_perp = make_double3(cr.x / nn, cr.y / nn, cr.z / nn);
  }
  e_par = cross3(e_perp, other);
}

// utd_transfer; false on edge-parallel (degenerate) geometry
static __device__ bool utd_transfer(const DevScene& S, int w, double3 s_i, double3 s_o, double dist_in,
                             double dist_out, double lam, M2& out, double3 b_in[2],
                             double3 b_out[2]) {
  const double3 e = ldg3(S.w_ehat + 3 * w);
  const double n_open = __ldg(S.w_nopen + w);
  const double cos_beta = dot_ddot(s_i, e);
  const double xb = 1.0 - cos_beta * cos_beta;
  const double sb0 = sqrt(xb > 0.0 ? xb : 0.0);
  if (sb0 < 1e-9) return false;
  const double3 ci = cross3(s_i, e);
  const double nci = sqrt(dot_ddot(ci, ci));
  b_in[0] = make_double3(ci.x / nci, ci.y / nci, ci.z / nci);
  b_in[1] = cross3(b_in[0], s_i);
  const double3 co = cross3(neg(s_o), e);
  const double nco = sqrt(dot_ddot(co, co));
  if (nco < 1e-9) return false;
  b_out[0] = make_double3(co.x / nco, co.y / nco, co.z / nco);
  b_out[1] = cross3(b_out[0], s_o);
  const double3 t0 = ldg3(S.w_t0 + 3 * w), n0 = ldg3(S.w_n0 + 3 * w);
  double3 sit = s_i - dot_ddot(s_i, e) * e, sot = s_o - dot_ddot(s_o, e) * e;
  const double n1 = sqrt(dot_ddot(sit, sit)), n2 = sqrt(dot_ddot(sot, sot));
  sit = make_double3(sit.x / n1, sit.y / n1, sit.z / n1);
  sot = make_double3(sot.x / n2, sot.y / n2, sot.z / n2);
  const double3 msit = neg(sit);
  const double phi_in =
      kPi - (kPi - acos(clamp1(dot_ddot(msit, t0)))) * (dot_ddot(msit, n0) >= 0.0 ? 1.0 : -1.0);
  const double phi_out =
      kPi - (kPi - acos(clamp1(dot_ddot(sot, t0)))) * (dot_ddot(sot, n0) >= 0.0 ? 1.0 : -1.0);
  const double k = kTwoPi / lam;
  const double l = dist_in * dist_out / (dist_in + dist_out) * (sb0 * sb0);
  const cplx pref = cdiv(C(-cos(-kPi / 4.0), -sin(-kPi / 4.0)),
                         C(2.0 * n_open * sqrt(2.0 * kPi * k) * sb0, 0.0));
  const cplx d1 = pref * cot_f(phi_out - phi_in, n_open, k, l, 1.0);
  const cplx d2 = pref * cot_f(phi_out - phi_in, n_open, k, l, -1.0);
  const cplx d3 = pref * cot_f(phi_out + phi_in, n_open, k, l, 1.0);
  const cplx d4 = pref * cot_f(phi_out + phi_in, n_open, k, l, -1.0);
  const double cos_r[2] = {fabs(sin(phi_in)), fabs(sin(n_open * kPi - phi_out))};
  const double3 nf[2] = {n0, ldg3(S.w_nn + 3 * w)};
  const int mrow[2] = {__ldg(S.w_mat0 + w), __ldg(S.w_matn + w)};
  M2 refl[2];
  for (int f = 0; f < 2; ++f) {
    double3 ep, el;
    oblique_frame(s_i, nf[f], s_i, ep, el);
    const double3 er = cross3(ep, s_o);
    const SbrMaterial m = S.mats[mrow[f]];
    cplx rp, rl;
    fresnel_vacuum_r(cos_r[f], m.eta_re, m.eta_im, rp, rl);
    M2 dg;
    dg.m[0][0] = rp;
    dg.m[0][1] = C(0.0, 0.0);
    dg.m[1][0] = C(0.0, 0.0);
    dg.m[1][1] = rl;
    refl[f] = m2_mul(m2_mul(m2_w(b_out[0], b_out[1], ep, er), dg), m2_w(ep, el, b_in[0], b_in[1]));
  }
  const cplx d12 = d1 + d2;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const cplx v = (i == j ? d12 : C(0.0, 0.0)) - d3 * refl[1].m[i][j] - d4 * refl[0].m[i][j];
      out.m[i][j] = C(-v.re, -v.im);
    }
  return true;
}

}  // namespace sbr
