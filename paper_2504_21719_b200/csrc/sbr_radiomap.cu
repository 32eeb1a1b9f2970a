// sbr_radiomap.cu -- radio-map SBR megakernel and the analytic direct term.
//
// Replaces emtrace radiomap.py:_map_chunk (347-563) and _direct_cells
// (566-583).  One persistent kernel runs the full segment loop per ray:
//   trace (closest hit) -> plane crossing + deposit (float64 atomics into the
//   L2-resident grid) -> escape / depth exit -> threshold + Russian roulette
//   -> slab Fresnel energies -> inverse-CDF draw (Philox keyed by global
//   sample id) -> R / S / T field and direction update.
// Rays live in registers for their whole life: there is no per-bounce ray
// state traffic to HBM.  Warps are kept full by "warp refill": after every
// segment, lanes whose ray ended fetch fresh sample ids with one atomicAdd
// per warp, so divergence in path length never idles lanes (the live-ray
// compaction of the north star, done in registers instead of through HBM).
//
// Work order: work item w -> global sample g = c + k*F (F = 233, a Fibonacci
// number), k = w % Q, c = w / Q.  Consecutive lanes therefore launch
// neighbouring lattice directions (coherent primary rays); the RNG is keyed
// by g, so the order has no effect on the result.
#include <string>

#include "sbr_physics.cuh"

struct SbrScene;

namespace sbr {
DevScene dev_view(const SbrScene* s);
int set_error(int code, const std::string& msg);
}  // namespace sbr

using namespace sbr;

namespace {

constexpr uint64_t kCombStride = 233;

struct MapRay {
  double3 o, d;
  cvec3 E;
  double r_dist, omega, weight;
  uint64_t g;
  int seg;
  bool alive;
};

struct LaneCounters {
  unsigned rb, deposits, escaped, respawns;
};

__device__ __forceinline__ void init_ray(const SbrMapParams& P, uint64_t g, MapRay& R) {
  R.g = g;
  R.seg = 0;
  R.d = fibonacci_dir(P.num_samples, g);
  R.o = make_double3(P.source[0], P.source[1], P.source[2]);
  R.E = antenna_field(P.pattern, R.d);
  R.r_dist = 0.0;
  R.omega = P.omega0;
  R.weight = alpha_sq(P, R.d);
  R.alive = true;
}

// One segment of the _map_chunk loop for one ray.
__device__ __forceinline__ void map_step(const DevScene& S, const SbrMapParams& P, MapRay& R,
                                         double* __restrict__ grid, LaneCounters& K,
                                         unsigned long long* sc) {
  const int seg = R.seg;
  const uint64_t chunk = R.g >> SBR_CHUNK_LOG2;
  const uint64_t slot = R.g & ((1ULL << SBR_CHUNK_LOG2) - 1);
  K.rb++;
  HitRecord h;
  if (!trace_closest(S, R.o, R.d, 1e-4, __longlong_as_double(0x7ff0000000000000LL), h)) {
    flag_error(S, kErrStack);
    atomicAdd(sc + SBR_MC_STACK_OVERFLOW, 1ULL);
    R.alive = false;
    return;
  }
  const double3 n_hat = make_double3(P.normal[0], P.normal[1], P.normal[2]);
  if (seg >= 1) {
    // plane crossing before the hit (escaped rays have t = inf and deposit)
    const double denom = dot_gemv(R.d, n_hat);
    double s = -1.0;
    if (fabs(denom) > 1e-12) s = (P.plane_off - dot_gemv(R.o, n_hat)) / denom;
    if (s > 1e-4 && s < h.t) {
      const double3 pt = R.o + s * R.d;
      const double3 rel = make_double3(pt.x - P.corner[0], pt.y - P.corner[1], pt.z - P.corner[2]);
      const double fu = floor(dot_gemv(rel, make_double3(P.u_hat[0], P.u_hat[1], P.u_hat[2])) / P.cell_w);
      const double fv = floor(dot_gemv(rel, make_double3(P.v_hat[0], P.v_hat[1], P.v_hat[2])) / P.cell_h);
      if (fu >= 0.0 && fu < (double)P.nx && fv >= 0.0 && fv < (double)P.ny) {
        const double val = P.scale * field_energy(R.E) * R.omega / fabs(denom) * R.weight;
        atomicAdd(grid + (int64_t)fv * P.nx + (int64_t)fu, val);
        K.deposits++;
      }
    }
  }
  if (h.tri < 0) {
    K.escaped++;
    R.alive = false;
    return;
  }
  if (seg == P.max_depth) {
    R.alive = false;
    return;
  }
  const double r_hit = R.r_dist + h.t;
  if (seg >= P.cull_from && (P.gain_threshold > 0.0 || P.rr_depth >= 0)) {
    const double e_sq = field_energy(R.E);
    bool keep = true;
    if (P.gain_threshold > 0.0) {
      keep = e_sq >= P.gain_threshold * (r_hit * r_hit);
      if (!keep) atomicAdd(sc + SBR_MC_THRESHOLD_KILLED, 1ULL);
    }
    if (P.rr_depth >= 0 && seg >= P.rr_depth) {
      const double surv = e_sq < P.rr_max ? e_sq : P.rr_max;
      const double u_rr = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_ROULETTE, slot);
      if (keep && u_rr >= surv) atomicAdd(sc + SBR_MC_ROULETTE_KILLED, 1ULL);
      keep = keep && (u_rr < surv);
      if (keep) R.weight /= surv;
    }
    if (!keep) {
      R.alive = false;
      return;
    }
  }
  const double3 pt = R.o + h.t * R.d;
  double3 n = ldg3(S.normals + 3 * (int64_t)h.tri);
  if (dot_seq(R.d, n) > 0.0) n = neg(n);
  const double cos_i = fabs(dot_seq(R.d, n));
  const SbrMaterial m = S.mats[__ldg(S.matrow + h.tri)];
  const Fresnel4 F = slab_fresnel(m, cos_i);
  const double r_sq = cabs2(F.rp) + cabs2(F.rl);
  const double t_sq = cabs2(F.tp) + cabs2(F.tl);
  // _interaction_rows with q_D = 0 (paths.py:572-595)
  double q0 = 0.0, q1 = 0.0, q2 = 0.0;
  const double den = r_sq + t_sq;
  if (den > 0.0) {
    const double s_sq = m.scattering * m.scattering;
    q0 = 1.0 * (1.0 - s_sq) * r_sq / den;
    q1 = 1.0 * s_sq * r_sq / den;
    q2 = 1.0 * t_sq / den;
  }
  if (!(P.allow_mask & 1)) q0 = 0.0;
  if (!(P.allow_mask & 2)) q1 = 0.0;
  if (!(P.allow_mask & 4)) q2 = 0.0;
  const double total = ((q0 + q1) + q2) + 0.0;
  if (!(total > 0.0)) {
    atomicAdd(sc + SBR_MC_TERMINATED, 1ULL);
    R.alive = false;
    return;
  }
  q0 /= total;
  q1 /= total;
  q2 /= total;
  const double q3 = 0.0 / total;
  const double u = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_INTERACTION, slot);
  const double c0 = q0, c1 = c0 + q1, c2 = c1 + q2, c3 = c2 + q3;
  int code = (u >= c0) + (u >= c1) + (u >= c2) + (u >= c3);
  if (code > 3) code = 3;
  R.weight /= (code == 0 ? q0 : code == 1 ? q1 : code == 2 ? q2 : q3);

  double3 e_perp, e_par;
  incidence_frame(R.d, n, e_perp, e_par);
  const cplx c_perp = cdot_real(R.E, e_perp), c_par = cdot_real(R.E, e_par);
  double3 nd = R.d;
  if (code == 0) {
    const double dn = dot_seq(R.d, n);
    const double3 kr = R.d - (2.0 * dn) * n;
    const double3 e_par_r = cross3(e_perp, kr);
    const cplx a = F.rp * c_perp, b = F.rl * c_par;
    R.E.x = m.spec_amp * (e_perp.x * a + e_par_r.x * b);
    R.E.y = m.spec_amp * (e_perp.y * a + e_par_r.y * b);
    R.E.z = m.spec_amp * (e_perp.z * a + e_par_r.z * b);
    nd = kr;
  } else if (code == 2) {
    const cplx a = F.tp * c_perp, b = F.tl * c_par;
    R.E.x = e_perp.x * a + e_par.x * b;
    R.E.y = e_perp.y * a + e_par.y * b;
    R.E.z = e_perp.z * a + e_par.z * b;
  }
  R.r_dist = r_hit;
  if (code == 1) {
    const double u0 = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot);
    const double u1 = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot + 1);
    const double cos_t = u0, azim = kTwoPi * u1;
    const double x = 1.0 - cos_t * cos_t;
    const double sin_t = sqrt(x > 0.0 ? x : 0.0);
    const double3 t1 = perp_batch(n);
    const double3 t2 = cross3(n, t1);
    double sa, ca;
    sincos(azim, &sa, &ca);
    const double a = sin_t * ca, b = sin_t * sa;
    const double3 ks = make_double3((a * t1.x + b * t2.x) + cos_t * n.x,
                                    (a * t1.y + b * t2.y) + cos_t * n.y,
                                    (a * t1.z + b * t2.z) + cos_t * n.z);
    const double g_num = sqrt(cabs2(F.rp * c_perp) + cabs2(F.rl * c_par));
    const double g_den = sqrt(cabs2(c_perp) + cabs2(c_par));
    const double gamma = g_den > 0.0 ? g_num / g_den : 0.0;
    const double f_s = pattern_density(m, R.d, ks, n);
    const double patch = R.omega * (r_hit * r_hit) / (cos_i > 1e-12 ? cos_i : 1e-12);
    const double amp = m.scattering * gamma * sqrt(f_s * cos_i * patch);
    double3 th_i, ph_i;
    transverse_rows(R.d, th_i, ph_i);
    const cplx ci0 = cdot_real(R.E, th_i), ci1 = cdot_real(R.E, ph_i);
    double chi1 = 0.0, chi2 = 0.0;
    if (P.any_random_phase && m.random_phases) {
      chi1 = kTwoPi * philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot);
      chi2 = kTwoPi * philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot + 1);
    }
    const double sq = sqrt(1.0 - m.xpd_kx), sk = sqrt(m.xpd_kx);
    double s1, k1, s2, k2;
    sincos(chi1, &s1, &k1);
    sincos(chi2, &s2, &k2);
    const cplx co0 = C(amp * k1, amp * s1) * (sq * ci0 - sk * ci1);
    const cplx co1 = C(amp * k2, amp * s2) * (sk * ci0 + sq * ci1);
    double3 th_s, ph_s;
    transverse_rows(ks, th_s, ph_s);
    const cplx inv_r = C(r_hit, 0.0);
    R.E.x = cdiv(th_s.x * co0 + ph_s.x * co1, inv_r);
    R.E.y = cdiv(th_s.y * co0 + ph_s.y * co1, inv_r);
    R.E.z = cdiv(th_s.z * co0 + ph_s.z * co1, inv_r);
    nd = ks;
    R.r_dist = 0.0;
    R.omega = kTwoPi;
    K.respawns++;
  }
  R.o = pt;
  R.d = nd;
  R.seg = seg + 1;
}

__global__ void __launch_bounds__(128) k_radiomap(DevScene S, SbrMapParams P, uint64_t begin,
                                                  uint64_t count, uint64_t comb_q,
                                                  unsigned long long* __restrict__ work,
                                                  double* __restrict__ grid,
                                                  unsigned long long* __restrict__ counters) {
  __shared__ unsigned long long sc[SBR_MC_COUNT];
  for (int i = threadIdx.x; i < SBR_MC_COUNT; i += blockDim.x) sc[i] = 0ULL;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint64_t total_items = comb_q * kCombStride;
  MapRay R;
  R.alive = false;
  LaneCounters K = {0u, 0u, 0u, 0u};
  bool more = true;
  while (true) {
    const unsigned dead = __ballot_sync(0xffffffffu, !R.alive);
    if (dead && more) {
      const unsigned nd = __popc(dead);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(work, (unsigned long long)nd);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + nd >= total_items) more = false;
      if (!R.alive) {
        const uint64_t w = base + __popc(dead & lt_mask);
        if (w < total_items) {
          const uint64_t k = w % comb_q, c = w / comb_q;
          const uint64_t local = c + k * kCombStride;
          if (local < count) init_ray(P, begin + local, R);
        }
      }
    }
    if (!__any_sync(0xffffffffu, R.alive)) {
      if (!more) break;
      continue;
    }
    if (R.alive) map_step(S, P, R, grid, K, sc);
  }
  // warp-reduce the per-lane counters, then one shared atomic per warp
  unsigned v[4] = {K.rb, K.deposits, K.escaped, K.respawns};
  const int idx[4] = {SBR_MC_RAY_BOUNCES, SBR_MC_DEPOSITS, SBR_MC_ESCAPED, SBR_MC_RESPAWNS};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v[k]);
    if (lane == 0) atomicAdd(sc + idx[k], (unsigned long long)s);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SBR_MC_COUNT; i += blockDim.x)
    if (sc[i]) atomicAdd(counters + i, sc[i]);
}

__global__ void __launch_bounds__(128) k_direct(DevScene S, SbrMapParams P,
                                                double* __restrict__ out,
                                                unsigned long long* __restrict__ counters) {
  const int64_t ncell = (int64_t)P.nx * P.ny;
  unsigned visible = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(c % P.nx), j = (int)(c / P.nx);
    const double uu = ((double)i + 0.5) * P.cell_w, vv = ((double)j + 0.5) * P.cell_h;
    const double3 ctr = make_double3((P.corner[0] + uu * P.u_hat[0]) + vv * P.v_hat[0],
                                     (P.corner[1] + uu * P.u_hat[1]) + vv * P.v_hat[1],
                                     (P.corner[2] + uu * P.u_hat[2]) + vv * P.v_hat[2]);
    const double3 src = make_double3(P.source[0], P.source[1], P.source[2]);
    const double3 diff = ctr - src;
    const double dist = norm_seq(diff);
    double val = 0.0;
    if (dist > 1e-9) {
      const double3 d = make_double3(diff.x / dist, diff.y / dist, diff.z / dist);
      const double e_sq = field_energy(antenna_field(P.pattern, d));
      const double a_sq = alpha_sq(P, d);
      const double x = P.wavelength / (kFourPi * dist);
      const double gain = x * x * e_sq * a_sq;
      bool ok;
      const bool occ = occluded_segment(S, src, ctr, 1e-4, ok);
      if (!ok) flag_error(S, kErrStack);
      val = occ ? 0.0 : gain;
    }
    out[c] = val;
    visible += val > 0.0;
  }
  const unsigned s = __reduce_add_sync(0xffffffffu, visible);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(counters + SBR_MC_DIRECT_VISIBLE, (unsigned long long)s);
}

int launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(SBR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
  return SBR_OK;
}

int check_params(const SbrScene* scene, const SbrMapParams* P) {
  if (!scene || !P) return set_error(SBR_ERR_INVALID, "NULL argument");
  const DevScene S = dev_view(scene);
  if (!S.mats) return set_error(SBR_ERR_INVALID, "scene has no material table");
  if (P->nx < 1 || P->ny < 1) return set_error(SBR_ERR_INVALID, "grid shape must be positive");
  if (P->num_samples < 1) return set_error(SBR_ERR_INVALID, "num_samples must be positive");
  if (P->n_elements > 0 && (!P->elem_offsets_dev || !P->precoder_dev))
    return set_error(SBR_ERR_INVALID, "array without offsets / precoder");
  return SBR_OK;
}

}  // namespace

extern "C" {

int sbr_radiomap_bounce(const SbrScene* scene, const SbrMapParams* P, uint64_t sample_begin,
                        uint64_t sample_end, double* grid, uint64_t* counters, void* stream) {
  int rc = check_params(scene, P);
  if (rc) return rc;
  if (sample_end > P->num_samples || sample_begin > sample_end)
    return set_error(SBR_ERR_INVALID, "bad sample range");
  const uint64_t count = sample_end - sample_begin;
  if (count == 0) return SBR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* work;
  if (cudaMallocAsync(&work, sizeof(unsigned long long), st) != cudaSuccess)
    return set_error(SBR_ERR_NOMEM, "work counter");
  cudaMemsetAsync(work, 0, sizeof(unsigned long long), st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_radiomap, 128, 0);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t warps_needed = (count + 31) / 32;
  if (blocks * 4 > warps_needed) blocks = (warps_needed + 3) / 4;
  if (blocks < 1) blocks = 1;
  const uint64_t comb_q = (count + kCombStride - 1) / kCombStride;
  k_radiomap<<<(unsigned)blocks, 128, 0, st>>>(dev_view(scene), *P, sample_begin, count, comb_q,
                                               work, grid, (unsigned long long*)counters);
  rc = launch_status("k_radiomap");
  cudaFreeAsync(work, st);
  return rc;
}

int sbr_radiomap_direct(const SbrScene* scene, const SbrMapParams* P, double* direct,
                        uint64_t* counters, void* stream) {
  int rc = check_params(scene, P);
  if (rc) return rc;
  const int64_t ncell = (int64_t)P->nx * P->ny;
  int64_t blocks = (ncell + 127) / 128;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_direct<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(dev_view(scene), *P, direct,
                                                              (unsigned long long*)counters);
  return launch_status("k_direct");
}

}  // extern "C"
