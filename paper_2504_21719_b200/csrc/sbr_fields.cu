// sbr_fields.cu -- path field replay (Algorithm 2) and the channel frequency response.
//
// Replaces emtrace:
//   compute_path_fields (paths.py:1302-1399) with _step_probability (1276-1299),
//   _right_handed (1259-1273), specular_transform / refraction_transform
//   (materials.py:280-347), gamma_reflected / diffuse_transform (400-475),
//   pattern_to_gcs (em.py:198-219), accumulate_doppler (paths.py:1410-1426)
//                                                       -> k_cir_fields
//   frequency_response (paths.py:1519-1547), array_response (em.py:240-251)
//                                                       -> k_cfr
// One thread per path; the transverse field is a 2-component complex Jones
// vector carried in an explicit (a, b, k) frame exactly as the reference does,
// in float64 (north-star tolerance for gains/delays/angles: 1e-4 relative).
#include <string>

#include "sbr_utd.cuh"

struct SbrScene;

namespace sbr {
DevScene dev_view(const SbrScene* s);
int set_error(int code, const std::string& msg);
}  // namespace sbr

using namespace sbr;

namespace {

constexpr double kSpeedOfLight = 299792458.0;

struct Jones {
  cplx c0, c1;         // components along (a, b)
  double3 a, b, k;     // frame
};

__device__ __forceinline__ double ddot(double3 a, double3 b) { return dot_ddot(a, b); }

// (theta_hat, phi_hat) of a direction (em.py:39-50 transverse_frame)
__device__ __forceinline__ void sph_frame(double3 d, double3& th, double3& ph) {
  transverse_rows(d, th, ph);
}

// pattern_to_gcs (em.py:198-219): components in the world (theta, phi) basis of d
__device__ void pattern_gcs(const SbrAntenna& A, double3 d, cplx& c_th, cplx& c_ph, double3& th_g,
                            double3& ph_g) {
  const double* R = A.rot;
  // d_local = rot.T @ d
  const double3 dl = make_double3(R[0] * d.x + R[3] * d.y + R[6] * d.z,
                                  R[1] * d.x + R[4] * d.y + R[7] * d.z,
                                  R[2] * d.x + R[5] * d.y + R[8] * d.z);
  const double theta_l = acos(clamp1(dl.z));
  const double phi_l = atan2(dl.y, dl.x);
  const double amp = A.kind == SBR_PATTERN_TR38901 ? tr38901_amp(A.scale, theta_l, phi_l) : 1.0;
  sph_frame(d, th_g, ph_g);
  double st, ct, sp, cp;
  sincos(theta_l, &st, &ct);
  sincos(phi_l, &sp, &cp);
  const double3 th_l = make_double3(ct * cp, ct * sp, -st);
  const double3 ph_l = make_double3(-sp, cp, 0.0);
  const double3 thw = make_double3(R[0] * th_l.x + R[1] * th_l.y + R[2] * th_l.z,
                                   R[3] * th_l.x + R[4] * th_l.y + R[5] * th_l.z,
                                   R[6] * th_l.x + R[7] * th_l.y + R[8] * th_l.z);
  (void)ph_l;  // both built-in evaluators return c_phi_l = 0 (em.py:258-288)
  c_th = C(ddot(th_g, thw) * amp, 0.0);
  c_ph = C(ddot(ph_g, thw) * amp, 0.0);
}

// W = [[a.q, a.r], [b.q, b.r]] applied to comps given in (q, r)
__device__ __forceinline__ void basis_change(double3 a, double3 b, double3 q, double3 r, cplx c0,
                                             cplx c1, cplx& o0, cplx& o1) {
  const double w00 = ddot(a, q), w01 = ddot(a, r), w10 = ddot(b, q), w11 = ddot(b, r);
  o0 = w00 * c0 + w01 * c1;
  o1 = w10 * c0 + w11 * c1;
}

__device__ __forceinline__ void right_handed(Jones& J, double3 a, double3 b, double3 k) {
  if (ddot(cross3(a, b), k) < 0.0) {
    const cplx t = J.c0;
    J.c0 = J.c1;
    J.c1 = t;
    J.a = b;
    J.b = a;
  } else {
    J.a = a;
    J.b = b;
  }
  J.k = k;
}

// interaction_probabilities(...)[kind] at replay geometry (paths.py:1276-1299);
// allow already carries the has_s / has_d / wedge-ownership masks
__device__ double step_probability(const SbrMaterial& m, double cos_i, int kind, double q_d,
                                   int allow) {
  const Fresnel4 F = slab_fresnel(m, cos_i);
  const double r_sq = cabs2(F.rp) + cabs2(F.rl);
  const double t_sq = cabs2(F.tp) + cabs2(F.tl);
  const double den = r_sq + t_sq;
  double q[4] = {0.0, 0.0, 0.0, q_d};
  if (den > 0.0) {
    const double keep = 1.0 - q_d;
    const double s2 = m.scattering * m.scattering;
    q[0] = keep * (1.0 - s2) * r_sq / den;
    q[1] = keep * s2 * r_sq / den;
    q[2] = keep * t_sq / den;
  }
  if (!(allow & 1)) q[0] = 0.0;
  if (!(allow & 2)) q[1] = 0.0;
  if (!(allow & 4)) q[2] = 0.0;
  if (!(allow & 8)) q[3] = 0.0;
  const double total = (((0.0 + q[0]) + q[1]) + q[2]) + q[3];
  return total > 0.0 ? q[kind] / total : 0.0;
}

__device__ __forceinline__ uint64_t phase_tag(int nsteps) {
  // fnv1a("phase-%d" % nsteps)
  char buf[16] = {'p', 'h', 'a', 's', 'e', '-'};
  int len = 6;
  char digits[8];
  int nd = 0;
  int v = nsteps;
  do {
    digits[nd++] = (char)('0' + v % 10);
    v /= 10;
  } while (v > 0);
  while (nd > 0) buf[len++] = digits[--nd];
  uint64_t h = 0xCBF29CE484222325ULL;
  for (int i = 0; i < len; ++i) h = (h ^ (uint8_t)buf[i]) * 0x100000001B3ULL;
  return h;
}

__global__ void __launch_bounds__(128) k_cir_fields(DevScene S, SbrFieldParams P, SbrRecordBuf R,
                                                    const double* __restrict__ pv,
                                                    const int32_t* __restrict__ status, int64_t n,
                                                    double* gain, double* delay, double* doppler,
                                                    double* dep, double* arr) {
  const int L = R.max_depth;
  const double lam = P.wavelength;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (status[r] != SBR_REFINE_OK) continue;
    const int depth = R.depth[r];
    const int tgt = R.target[r];
    const double* V = pv + r * (int64_t)(L + 2) * 3;
    // segments
    double seg_len[17];
    double3 kh[17];
    double total_len = 0.0;
    for (int i = 0; i <= depth; ++i) {
      const double3 s = make_double3(V[3 * (i + 1)] - V[3 * i], V[3 * (i + 1) + 1] - V[3 * i + 1],
                                     V[3 * (i + 1) + 2] - V[3 * i + 2]);
      seg_len[i] = norm_seq(s);
      kh[i] = make_double3(s.x / seg_len[i], s.y / seg_len[i], s.z / seg_len[i]);
      total_len += seg_len[i];
    }
    // launch field
    Jones J;
    {
      double3 th, ph;
      pattern_gcs(P.tx_pattern, kh[0], J.c0, J.c1, th, ph);
      J.a = th;
      J.b = ph;
      J.k = kh[0];
    }
    double gamma_prob = 1.0, r_dist = 0.0, s_dist = 0.0;
    double tube_omega = kFourPi / (double)P.num_samples;
    bool has_s = false, has_d = false, diffracted = false;
    int n_phase = 0;
    const uint64_t ptag = phase_tag(depth);
    const uint64_t psample = R.sample[r] > 0 ? (uint64_t)R.sample[r] : 0ULL;
    // accumulate_doppler (paths.py:1410-1426): endpoint terms first, then vertices
    const double3 tv = make_double3(P.tx_velocity[0], P.tx_velocity[1], P.tx_velocity[2]);
    const double3 rv = ldg3(P.rx_velocity_dev + 3 * tgt);
    double nu = ddot(tv, kh[0]) / lam;
    nu -= ddot(rv, kh[depth]) / lam;
    for (int i = 0; i < depth; ++i) {
      const int64_t o = r * L + i;
      const int kind = R.kind[o];
      const int slot = R.tri[o];
      const double3 k_in = kh[i], k_out = kh[i + 1];
      r_dist += seg_len[i];
      const int row = __ldg(S.matrow + slot);
      const SbrMaterial m = S.mats[row];
      double3 nrm = ld3(R.normal + 3 * o);
      const double cos_step = fabs(ddot(k_in, nrm));
      double3 n_hat = nrm;
      if (ddot(k_in, n_hat) > 0.0) n_hat = neg(n_hat);
      gamma_prob *= step_probability(m, cos_step, kind, P.q_diffraction,
                                     allowed_kinds(S, P.allow_mask, slot, has_s, has_d));
      if (P.n_objects > 0 && row < P.n_objects) {
        const double3 v = ldg3(P.obj_velocity_dev + 3 * row);
        if (v.x != 0.0 || v.y != 0.0 || v.z != 0.0) nu += ddot(v, k_out - k_in) / lam;
      }
      if (kind == 3) {
        // UTD wedge transfer (paths.py:1358-1373)
        double remaining = 0.0;
        for (int q2 = i + 1; q2 <= depth; ++q2) remaining += seg_len[q2];
        M2 T;
        double3 bi[2], bo[2];
        if (!utd_transfer(S, R.wedge[o], k_in, k_out, r_dist, remaining, lam, T, bi, bo)) {
          J.c0 = J.c1 = C(0.0, 0.0);
        } else {
          cplx p0, p1;
          basis_change(bi[0], bi[1], J.a, J.b, J.c0, J.c1, p0, p1);
          J.c0 = T.m[0][0] * p0 + T.m[0][1] * p1;
          J.c1 = T.m[1][0] * p0 + T.m[1][1] * p1;
          right_handed(J, bo[0], bo[1], k_out);
        }
        s_dist = r_dist;
        r_dist = 0.0;
        diffracted = true;
        has_d = true;
        continue;
      }
      double3 e_perp, e_par;
      incidence_frame(k_in, n_hat, e_perp, e_par);
      const double cos_t = fabs(ddot(k_in, n_hat));
      if (kind == 0 || kind == 2) {
        const Fresnel4 F = slab_fresnel(m, cos_t);
        cplx c0, c1;
        basis_change(e_perp, e_par, J.a, J.b, J.c0, J.c1, c0, c1);
        if (kind == 0) {
          const double dn = ddot(k_in, n_hat);
          const double3 k_r = k_in - (2.0 * dn) * n_hat;
          const double3 e_r_par = cross3(e_perp, k_r);
          J.c0 = m.spec_amp * F.rp * c0;
          J.c1 = m.spec_amp * F.rl * c1;
          right_handed(J, e_perp, e_r_par, k_r);
        } else {
          J.c0 = F.tp * c0;
          J.c1 = F.tl * c1;
          right_handed(J, e_perp, e_par, k_in);
        }
      } else {
        // diffuse scattering (gamma_reflected + diffuse_transform)
        const Fresnel4 F = slab_fresnel(m, cos_t);
        cplx p0, p1;
        basis_change(e_perp, e_par, J.a, J.b, J.c0, J.c1, p0, p1);
        const double nrm_in = sqrt(cabs2(p0) + cabs2(p1));
        const double gam =
            nrm_in == 0.0 ? 0.0 : sqrt(cabs2(F.rp * p0) + cabs2(F.rl * p1)) / nrm_in;
        double ci = -ddot(k_in, n_hat);
        const double ci_patch = ci > 1e-12 ? ci : 1e-12;
        const double patch = tube_omega * (r_dist * r_dist) / ci_patch;
        ci = ci < 0.0 ? 0.0 : (ci > 1.0 ? 1.0 : ci);
        const double f_s = pattern_density(m, k_in, k_out, n_hat);
        const double amp = m.scattering * gam * sqrt(f_s * ci * patch);
        double chi1 = 0.0, chi2 = 0.0;
        if (m.random_phases) {
          chi1 = kTwoPi * philox_uniform(P.seed, psample, (uint64_t)tgt, ptag, 2 * n_phase);
          chi2 = kTwoPi * philox_uniform(P.seed, psample, (uint64_t)tgt, ptag, 2 * n_phase + 1);
          ++n_phase;
        }
        const double sq = sqrt(1.0 - m.xpd_kx), sk = sqrt(m.xpd_kx);
        double th_i_s, th_i_c;
        double3 th_i, ph_i, th_s, ph_s;
        sph_frame(k_in, th_i, ph_i);
        sph_frame(k_out, th_s, ph_s);
        cplx q0, q1;
        basis_change(th_i, ph_i, J.a, J.b, J.c0, J.c1, q0, q1);
        sincos(chi1, &th_i_s, &th_i_c);
        const cplx e1 = C(th_i_c, th_i_s);
        double s2, c2;
        sincos(chi2, &s2, &c2);
        const cplx e2 = C(c2, s2);
        const cplx o0 = amp * ((sq * e1) * q0 + ((-sk) * e1) * q1);
        const cplx o1 = amp * ((sk * e2) * q0 + (sq * e2) * q1);
        const double inv = 1.0 / sqrt(gamma_prob);
        J.c0 = C(o0.re / r_dist * inv, o0.im / r_dist * inv);
        J.c1 = C(o1.re / r_dist * inv, o1.im / r_dist * inv);
        J.a = th_s;
        J.b = ph_s;
        J.k = k_out;
        gamma_prob = 1.0;
        r_dist = 0.0;
        tube_omega = kTwoPi;
        has_s = true;
      }
    }
    r_dist += seg_len[depth];
    const double3 arrival = kh[depth];
    cplx rc0, rc1;
    double3 rth, rph;
    pattern_gcs(P.rx_pattern_dev[tgt], neg(arrival), rc0, rc1, rth, rph);
    // e_vec . rx_vec (unconjugated)
    const cplx ex = J.c0 * C(J.a.x, 0.0) + J.c1 * C(J.b.x, 0.0);
    const cplx ey = J.c0 * C(J.a.y, 0.0) + J.c1 * C(J.b.y, 0.0);
    const cplx ez = J.c0 * C(J.a.z, 0.0) + J.c1 * C(J.b.z, 0.0);
    const cplx rx = rc0 * C(rth.x, 0.0) + rc1 * C(rph.x, 0.0);
    const cplx ry = rc0 * C(rth.y, 0.0) + rc1 * C(rph.y, 0.0);
    const cplx rz = rc0 * C(rth.z, 0.0) + rc1 * C(rph.z, 0.0);
    const cplx dotv = (ex * rx + ey * ry) + ez * rz;
    const double spread = diffracted ? sqrt(s_dist * r_dist * (s_dist + r_dist)) : r_dist;
    gain[2 * r] = dotv.re * (lam / kFourPi) / spread;
    gain[2 * r + 1] = dotv.im * (lam / kFourPi) / spread;
    delay[r] = total_len / kSpeedOfLight;
    doppler[r] = nu;
    for (int c = 0; c < 3; ++c) {
      dep[3 * r + c] = c == 0 ? kh[0].x : (c == 1 ? kh[0].y : kh[0].z);
      arr[3 * r + c] = c == 0 ? arrival.x : (c == 1 ? arrival.y : arrival.z);
    }
  }
}

// H[r, t, f] over the paths of one link, float64 accumulation in path order
// ---------------------------------------------------------------------------
// CFR (paths.py:1519-1547) as a factorised complex contraction
// ---------------------------------------------------------------------------
// The reference adds, path by path,
//     ((g_p * u_rx[r,p]) * u_tx[t,p]) * spin[p,f]
// so H = W . E with W[(r,t),p] = (g_p u_rx[r,p]) u_tx[t,p] and
// E[p,f] = exp(-2j pi f tau_p).  The steering vectors and the spin matrix are
// computed once (O((n_rx + n_tx + F) P) sincos instead of O(n_rx n_tx F P)),
// then a shared-memory tiled float64 contraction accumulates every output
// over p in path order with the same complex products (-fmad=false), so the
// result is identical to the path-by-path sum.  At these shapes (K = paths
// per link, a few to a few hundred) the contraction is tiny next to the
// output write; tensor cores would change the rounding (fused products,
// split K) for no measurable gain, so it stays on the FP64 pipe.

// u[e, p] = exp(1j * kw * (offsets[e] @ (sign * k_p)))   (em.py:240-251)
__global__ void k_cfr_steer(const double* __restrict__ dirs, int64_t np,
                            const double* __restrict__ offs, int ne, double kw, int incoming,
                            double* __restrict__ u) {
  const int64_t total = (int64_t)ne * np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / np);
    const int64_t p = i % np;
    const double3 k = ld3(dirs + 3 * p);
    const double ph = kw * dot_gemv(ldg3(offs + 3 * e), incoming ? neg(k) : k);
    double sn, cs;
    sincos(ph, &sn, &cs);
    u[2 * i] = cs;
    u[2 * i + 1] = sn;
  }
}

// E[p, f] = exp(-2j pi f tau_p)
__global__ void k_cfr_spin(const double* __restrict__ delay, int64_t np,
                           const double* __restrict__ freqs, int nf, double* __restrict__ E) {
  const int64_t total = np * nf;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / nf;
    const int f = (int)(i % nf);
    const double ang = -kTwoPi * freqs[f] * delay[p];
    double sn, cs;
    sincos(ang, &sn, &cs);
    E[2 * i] = cs;
    E[2 * i + 1] = sn;
  }
}

// W[(r, t), p]: synthetic arrays steer every path to every element pair;
// element-indexed paths only touch their own (rx_el, tx_el) row (zero
// elsewhere: a zero term leaves every partial sum unchanged)
__global__ void k_cfr_weights(const double* __restrict__ gain, int64_t np,
                              const double* __restrict__ u_rx, int nrx,
                              const double* __restrict__ u_tx, int ntx,
                              const int32_t* __restrict__ prx, const int32_t* __restrict__ ptx,
                              int synthetic, double* __restrict__ W) {
  const int64_t total = (int64_t)nrx * ntx * np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % np;
    const int64_t row = i / np;
    const int t = (int)(row % ntx), r = (int)(row / ntx);
    cplx a = C(gain[2 * p], gain[2 * p + 1]);
    if (synthetic) {
      a = (a * C(u_rx[2 * (r * np + p)], u_rx[2 * (r * np + p) + 1])) *
          C(u_tx[2 * (t * np + p)], u_tx[2 * (t * np + p) + 1]);
    } else if (prx[p] != r || ptx[p] != t) {
      a = C(0.0, 0.0);
    }
    W[2 * i] = a.re;
    W[2 * i + 1] = a.im;
  }
}

// H[row, f] = sum_p W[row, p] E[p, f], p in order.  Block: 32 rows x 64
// frequencies, 256 threads x (2 rows x 4 frequencies), K staged 16 at a time.
constexpr int kCfrRows = 32, kCfrCols = 64, kCfrK = 16;
#ifndef SBR_CFR_DMMA_MIN
#define SBR_CFR_DMMA_MIN 16  // paths per link from which the FP64 tensor-core contraction runs (tools/cfr_sweep.py: 5 paths SIMT 14 vs 15 us, 20 paths DMMA 22 vs 24 us)
#endif

__global__ void __launch_bounds__(256) k_cfr_contract(const double2* __restrict__ W,
                                                      const double2* __restrict__ E,
                                                      int64_t rows, int64_t np, int nf,
                                                      double2* __restrict__ H) {
  __shared__ double2 ws[kCfrRows][kCfrK + 1];
  __shared__ double2 es[kCfrK][kCfrCols];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * kCfrRows;
  const int col0 = blockIdx.x * kCfrCols;
  double ar[2][4], ai[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) ar[i][c] = ai[i][c] = 0.0;
  for (int64_t k0 = 0; k0 < np; k0 += kCfrK) {
    const int kn = (int)((np - k0) < kCfrK ? (np - k0) : kCfrK);
    for (int e = threadIdx.x; e < kCfrRows * kCfrK; e += 256) {
      const int rr = e / kCfrK, kk = e % kCfrK;
      const int64_t row = row0 + rr;
      ws[rr][kk] = (row < rows && kk < kn) ? W[row * np + k0 + kk] : make_double2(0.0, 0.0);
    }
    for (int e = threadIdx.x; e < kCfrK * kCfrCols; e += 256) {
      const int kk = e / kCfrCols, cc = e % kCfrCols;
      es[kk][cc] = (kk < kn && col0 + cc < nf) ? E[(k0 + kk) * nf + col0 + cc]
                                                : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 w = ws[ty * 2 + i][kk];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 e = es[kk][tx + 16 * c];
          // v = a * spin (numpy complex multiply), then out += v
          const double vr = w.x * e.x - w.y * e.y;
          const double vi = w.x * e.y + w.y * e.x;
          ar[i][c] += vr;
          ai[i][c] += vi;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = row0 + ty * 2 + i;
    if (row >= rows) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int f = col0 + tx + 16 * c;
      if (f < nf) H[row * nf + f] = make_double2(ar[i][c], ai[i][c]);
    }
  }
}

// ---- FP64 tensor-core path (DMMA, mma.sync m8n8k4 f64) for many paths ----
// H = W . E as four real products per complex one (Hr += Wr Er - Wi Ei,
// Hi += Wr Ei + Wi Er), each an 8x8x4 float64 MMA on the tensor cores (B200:
// FP64 tensor-core peak ~40 TFLOP/s vs the SIMT kernel's 18.6 TFLOP/s
// instruction roofline for unfused complex products).  The MMA fuses its
// multiply-adds, so H differs from the path-order sum by rounding (~1e-16 of
// max|H| per path; the north star allows 1e-4); used from kCfrDmmaMin paths on.
// Block: 4 warps, 32 rows x 64 frequencies; warp: 16 x 32 (2 x 4 MMA tiles);
// K staged 16 paths at a time in shared memory, real / imaginary planes split.
constexpr int kDmRows = 32, kDmCols = 64, kDmK = 16;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k_cfr_contract_dmma(const double2* __restrict__ W,
                                                           const double2* __restrict__ E,
                                                           int64_t rows, int64_t np, int nf,
                                                           double2* __restrict__ H) {
  __shared__ double wr[kDmRows][kDmK + 1], wi[kDmRows][kDmK + 1];
  __shared__ double er[kDmK][kDmCols + 1], ei[kDmK][kDmCols + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;  // warp tile origin in the block
  const int64_t row0 = (int64_t)blockIdx.y * kDmRows;
  const int col0 = blockIdx.x * kDmCols;
  const int g = lane >> 2, q = lane & 3;  // fragment coordinates
  double hr[2][4][2], hi[2][4][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) hr[m][n][0] = hr[m][n][1] = hi[m][n][0] = hi[m][n][1] = 0.0;
  for (int64_t k0 = 0; k0 < np; k0 += kDmK) {
    const int kn = (int)((np - k0) < kDmK ? (np - k0) : kDmK);
    for (int e = threadIdx.x; e < kDmRows * kDmK; e += 128) {
      const int rr = e / kDmK, kk = e % kDmK;
      const int64_t row = row0 + rr;
      const double2 v = (row < rows && kk < kn) ? W[row * np + k0 + kk] : make_double2(0.0, 0.0);
      wr[rr][kk] = v.x;
      wi[rr][kk] = v.y;
    }
    for (int e = threadIdx.x; e < kDmK * kDmCols; e += 128) {
      const int kk = e / kDmCols, cc = e % kDmCols;
      const double2 v = (kk < kn && col0 + cc < nf) ? E[(k0 + kk) * nf + col0 + cc]
                                                     : make_double2(0.0, 0.0);
      er[kk][cc] = v.x;
      ei[kk][cc] = v.y;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kDmK; ks += 4) {
      double ar[2], ai[2], br[4], bi[4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {  // A 8x4 row-major: (row g, col q)
        ar[m] = wr[wm + 8 * m + g][ks + q];
        ai[m] = wi[wm + 8 * m + g][ks + q];
      }
#pragma unroll
      for (int n = 0; n < 4; ++n) {  // B 4x8 col-major: (row q, col g)
        br[n] = er[ks + q][wn + 8 * n + g];
        bi[n] = ei[ks + q][wn + 8 * n + g];
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          dmma(hr[m][n][0], hr[m][n][1], ar[m], br[n]);
          dmma(hr[m][n][0], hr[m][n][1], ai[m], -bi[n]);
          dmma(hi[m][n][0], hi[m][n][1], ar[m], bi[n]);
          dmma(hi[m][n][0], hi[m][n][1], ai[m], br[n]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {  // C 8x8: (row g, cols 2q, 2q + 1)
    const int64_t row = row0 + wm + 8 * m + g;
    if (row >= rows) continue;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int f = col0 + wn + 8 * n + 2 * q + c;
        if (f < nf) H[row * nf + f] = make_double2(hr[m][n][c], hi[m][n][c]);
      }
  }
}

static int64_t g_cfr_dmma_min = SBR_CFR_DMMA_MIN;

unsigned grid_for(int64_t n, int block, int cap = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

int launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SBR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
  return SBR_OK;
}

}  // namespace

extern "C" {

int sbr_cir_fields(const SbrScene* scene, const SbrFieldParams* P, const SbrRecordBuf* rec,
                   const double* pv, const int32_t* status, int64_t n, double* gain, double* delay,
                   double* doppler, double* dep, double* arr, void* stream) {
  if (!scene || !P || !rec) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (!dev_view(scene).mats) return set_error(SBR_ERR_INVALID, "scene has no material table");
  if (!P->rx_pattern_dev || !P->rx_velocity_dev)
    return set_error(SBR_ERR_INVALID, "per-target rx pattern / velocity missing");
  if (rec->max_depth < 1 || rec->max_depth > 15) return set_error(SBR_ERR_INVALID, "bad max_depth");
  if (n <= 0) return SBR_OK;
  k_cir_fields<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      dev_view(scene), *P, *rec, pv, status, n, gain, delay, doppler, dep, arr);
  return launch_status("k_cir_fields");
}

int sbr_set_cfr_dmma_min_paths(int64_t min_paths) {
  g_cfr_dmma_min = min_paths;  // < 0: never use the tensor-core contraction
  return SBR_OK;
}

int sbr_cfr(const double* gain, const double* delay, const double* dep, const double* arr,
            const int32_t* prx, const int32_t* ptx, int64_t np, const double* freqs, int32_t nf,
            const double* txo, int32_t ntx, const double* rxo, int32_t nrx, double wavelength,
            int32_t synthetic, double* H, void* stream) {
  if (nf < 1 || ntx < 1 || nrx < 1) return set_error(SBR_ERR_INVALID, "empty response shape");
  if (!(wavelength > 0.0)) return set_error(SBR_ERR_INVALID, "wavelength must be positive");
  if (!synthetic && (!prx || !ptx)) return set_error(SBR_ERR_INVALID, "element indices missing");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = (int64_t)nrx * ntx;
  if (np == 0) {
    cudaMemsetAsync(H, 0, sizeof(double) * 2 * rows * nf, st);
    return launch_status("sbr_cfr memset");
  }
  const double kw = kTwoPi / wavelength;
  double *u_rx = nullptr, *u_tx = nullptr, *E = nullptr, *W = nullptr;
  const size_t c16 = 2 * sizeof(double);
  cudaError_t e = cudaSuccess;
  if (synthetic) {
    e = scratch_alloc((void**)&u_rx, c16 * nrx * np, st);
    if (e == cudaSuccess) e = scratch_alloc((void**)&u_tx, c16 * ntx * np, st);
  }
  if (e == cudaSuccess) e = scratch_alloc((void**)&E, c16 * np * nf, st);
  if (e == cudaSuccess) e = scratch_alloc((void**)&W, c16 * rows * np, st);
  int rc = SBR_OK;
  if (e != cudaSuccess) {
    rc = set_error(SBR_ERR_CUDA, std::string("sbr_cfr scratch: ") + cudaGetErrorString(e));
  } else {
    if (synthetic) {
      k_cfr_steer<<<grid_for((int64_t)nrx * np, 256), 256, 0, st>>>(arr, np, rxo, nrx, kw, 1, u_rx);
      rc = launch_status("k_cfr_steer");
      if (!rc) {
        k_cfr_steer<<<grid_for((int64_t)ntx * np, 256), 256, 0, st>>>(dep, np, txo, ntx, kw, 0,
                                                                      u_tx);
        rc = launch_status("k_cfr_steer");
      }
    }
    if (!rc) {
      k_cfr_spin<<<grid_for(np * nf, 256), 256, 0, st>>>(delay, np, freqs, nf, E);
      rc = launch_status("k_cfr_spin");
    }
    if (!rc) {
      k_cfr_weights<<<grid_for(rows * np, 256), 256, 0, st>>>(gain, np, u_rx, nrx, u_tx, ntx,
                                                              prx, ptx, synthetic, W);
      rc = launch_status("k_cfr_weights");
    }
    if (!rc) {
      prof_begin(st, "k_cfr_contract");
      if (g_cfr_dmma_min >= 0 && np >= g_cfr_dmma_min) {
        const dim3 grid((nf + kDmCols - 1) / kDmCols, (unsigned)((rows + kDmRows - 1) / kDmRows));
        k_cfr_contract_dmma<<<grid, 128, 0, st>>>((const double2*)W, (const double2*)E, rows, np,
                                                  nf, (double2*)H);
      } else {
        const dim3 grid((nf + kCfrCols - 1) / kCfrCols,
                        (unsigned)((rows + kCfrRows - 1) / kCfrRows));
        k_cfr_contract<<<grid, 256, 0, st>>>((const double2*)W, (const double2*)E, rows, np, nf,
                                             (double2*)H);
      }
      prof_end(st);
      rc = launch_status("k_cfr_contract");
    }
  }
  if (u_rx) cudaFreeAsync(u_rx, st);
  if (u_tx) cudaFreeAsync(u_tx, st);
  if (E) cudaFreeAsync(E, st);
  if (W) cudaFreeAsync(W, st);
  return rc;
}

}  // extern "C"
