// sbr_cir.cu -- path-solver (CIR) candidate generation, selection and refinement.
//
// Replaces emtrace paths.py:
//   _sweep_chunk / _continue_rays (704-828, 855-900)  -> k_cir_sweep
//   _visible_pairs (657-683)                          -> k_cir_visibility
//   _emit_records dedup + truncation (903-987),
//   DedupTable / PathBuffer (174-226),
//   generate_candidates registration loop (1019-1103) -> sbr_cir_select (CUB sorts
//                                                        + greedy slot kernels)
//   _record_from_batch (990-1016)                      -> k_cir_records
//   refine_candidate (1110-1252)                       -> k_cir_refine
//
// Design (B200): the sweep writes one 80-byte vertex per interaction into an
// HBM vertex buffer with a parent link (the reference keeps per-row history
// arrays and copies them on every select()); the O(vertices x targets)
// visibility stage -- the dominant cost at many receivers -- is a flat
// (vertex, target) grid with targets fastest so a warp shares one origin;
// candidate rows are 12 bytes (ordinal key + vertex index).  The reference's
// order-dependent dedup is reproduced exactly with sorts: stable radix sorts
// give "first occurrence in (depth, sample, target) order" and the
// both-slot DedupTable greedy is resolved by fixed-point rounds over the slot
// conflict lists.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <string>
#include <vector>

#include "sbr_utd.cuh"

namespace cg = cooperative_groups;

struct SbrScene;

namespace sbr {
DevScene dev_view(const SbrScene* s);
int set_error(int code, const std::string& msg);
}  // namespace sbr

using namespace sbr;

namespace {

constexpr uint64_t TAG_INTERACTION = 0x5c798e00ad8012ebULL;  // fnv1a("interaction")
constexpr uint64_t TAG_RESPAWN = 0x742c480a24ff9b7fULL;      // fnv1a("respawn")
constexpr uint64_t kFnvPrime = 0x100000001B3ULL;
constexpr uint64_t kHashBase = 1373ULL;                      // HASH_CHAIN_BASE
constexpr uint32_t kCirShardLog2 = SBR_CIR_SHARD_LOG2;  // CIR shard chunks of 4096 ids
constexpr int kTargetBits = 20;
constexpr int kSampleBits = 40;
constexpr uint64_t kTargetMask = (1ULL << kTargetBits) - 1;
constexpr uint64_t kSampleMask = (1ULL << kSampleBits) - 1;

// fnv1a_u64(value, seed) (paths.py:68-75)
__device__ __forceinline__ uint64_t fnv1a_u64(uint64_t v, uint64_t h) {
#pragma unroll
  for (int s = 0; s < 64; s += 8) h = (h ^ ((v >> s) & 0xFFULL)) * kFnvPrime;
  return h;
}

__device__ __forceinline__ uint64_t ordinal_key(int depth, int64_t sample, int target) {
  return ((uint64_t)depth << 60) | (((uint64_t)sample & kSampleMask) << kTargetBits) |
         ((uint64_t)target & kTargetMask);
}

// warp-aggregated append: one atomic per coalesced group
__device__ __forceinline__ unsigned long long append_slot(unsigned long long* counter) {
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(counter, (unsigned long long)g.size());
  base = g.shfl(base, 0);
  return base + g.thread_rank();
}

struct CirCounters {
  unsigned escaped, terminated, rb;
};

// _interaction_rows for one hit (paths.py:572-595), D never allowed (no wedges)
__device__ __forceinline__ bool interaction_probs(const SbrMaterial& m, double r_sq, double t_sq,
                                                  double q_d, int allow, double q[4]) {
  q[0] = q[1] = q[2] = 0.0;
  q[3] = q_d;
  const double den = r_sq + t_sq;
  if (den > 0.0) {
    const double keep = 1.0 - q_d;
    const double s_sq = m.scattering * m.scattering;
    q[0] = keep * (1.0 - s_sq) * r_sq / den;
    q[1] = keep * s_sq * r_sq / den;
    q[2] = keep * t_sq / den;
  }
  if (!(allow & 1)) q[0] = 0.0;
  if (!(allow & 2)) q[1] = 0.0;
  if (!(allow & 4)) q[2] = 0.0;
  if (!(allow & 8)) q[3] = 0.0;  // masked by has_s / has_d / wedge ownership
  const double total = ((q[0] + q[1]) + q[2]) + q[3];
  if (!(total > 0.0)) return false;
  q[0] /= total;
  q[1] /= total;
  q[2] /= total;
  q[3] /= total;
  return true;
}

// ---------------------------------------------------------------------------
// sweep
// ---------------------------------------------------------------------------
#ifndef SBR_SWEEP_MINB
#define SBR_SWEEP_MINB 8  // 64 registers: config-5 sweep 3.5 -> 2.0 ms
#endif
__global__ void __launch_bounds__(128, SBR_SWEEP_MINB) k_cir_sweep(DevScene S, SbrCirParams P, uint64_t begin,
                                                   uint64_t end, SbrVertexBuf vb,
                                                   unsigned long long* __restrict__ counters,
                                                   ShardMap sh, CombMap comb) {
  CirCounters K = {0u, 0u, 0u};
  const double3 src = make_double3(P.source[0], P.source[1], P.source[2]);
  // Warp-uniform loop over batches of 32 samples; every depth step traces the
  // batch's live rays together with the while-while closest hit (parked
  // leaves, full-warp triangle tests) instead of one scalar walk per thread.
  const unsigned lane_id = threadIdx.x & 31u;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  alignas(8) int sn[(SBR_PACKED_STACK ? 2 : 1) * kStackSize];
  float st[SBR_PACKED_STACK ? 1 : kStackSize];
  // comb order: the 32 lanes of a batch take lattice neighbours (ids F apart)
  const uint64_t slots = comb.slots();
  for (uint64_t base = warp0 * 32; base < slots; base += nwarps * 32) {
    const uint64_t off = base + lane_id < slots ? comb.sample(base + lane_id) : ~0ULL;
    const uint64_t l = begin + off;
    bool alive = off < end - begin;
    const uint64_t g = sh.gid(alive ? l : begin);  // global sample id (RNG key, ordinal)
    double3 o = src;
    double3 d = fibonacci_dir(P.num_samples, g);
    uint64_t hr = 0, hf = 0;
    double run_prob = 1.0;
    int suffix_start = 0;
    int parent = -1;
    bool has_s = false, has_d = false;
    for (int depth = 1; depth <= P.max_depth; ++depth) {
      if (!__any_sync(0xffffffffu, alive)) break;
      ClosestTravT<false> T(sn, st);
      if (alive) {
        K.rb++;
        T.start(S, o, d, 1e-4, __longlong_as_double(0x7ff0000000000000LL));
      } else {
        T.idle();
      }
      while (__any_sync(0xffffffffu, !T.done())) T.template round_u<true>(S);  // 1.08 -> 1.05 ms at config 3
      if (!alive) continue;
      HitRecord h;
      T.result(h);
      if (!T.ok) {
        flag_error(S, kErrStack);
        atomicAdd(counters + SBR_CC_STACK_OVERFLOW, 1ULL);
        alive = false;
        continue;
      }
      if (h.tri < 0) {
        K.escaped++;
        alive = false;
        continue;
      }
      double3 pt = o + h.t * d;
      double3 n = ldg3(S.normals + 3 * (int64_t)h.tri);
      if (dot_seq(d, n) > 0.0) n = neg(n);
      const double cos_i = fabs(dot_seq(d, n));
      const SbrMaterial m = S.mats[__ldg(S.matrow + h.tri)];
      const Fresnel4 F = slab_fresnel(m, cos_i);
      const double r_sq = cabs2(F.rp) + cabs2(F.rl);
      const double t_sq = cabs2(F.tp) + cabs2(F.tl);
      double q[4];
      if (!interaction_probs(m, r_sq, t_sq, P.q_diffraction,
                             allowed_kinds(S, P.allow_mask, h.tri, has_s, has_d), q)) {
        K.terminated++;
        alive = false;
        continue;
      }
      const double u = philox_uniform(P.seed, 0, (uint64_t)depth, TAG_INTERACTION, g);
      const double c0 = q[0], c1 = c0 + q[1], c2 = c1 + q[2], c3 = c2 + q[3];
      int code = (u >= c0) + (u >= c1) + (u >= c2) + (u >= c3);
      if (code > 3) code = 3;
      run_prob *= q[code];
      int wid = -1;
      if (code == 3) {
        double3 foot;
        wid = project_wedge(S, h.tri, pt, foot);
        pt = foot;
        has_d = true;
        hr = kHashBase * hr + __ldg(S.w_hr + wid);
        hf = kHashBase * hf + __ldg(S.w_hf + wid);
      } else if (code == 0) {
        hr = kHashBase * hr + __ldg(S.hash_r + h.tri);
        hf = kHashBase * hf + __ldg(S.hash_f + h.tri);
      } else if (code == 1) {
        suffix_start = depth;
        has_s = true;
      }
      const unsigned long long vi = append_slot(counters + SBR_CC_VERTICES);
      if ((int64_t)vi < vb.capacity) {
        vb.point[3 * vi] = pt.x;
        vb.point[3 * vi + 1] = pt.y;
        vb.point[3 * vi + 2] = pt.z;
        vb.normal[3 * vi] = n.x;
        vb.normal[3 * vi + 1] = n.y;
        vb.normal[3 * vi + 2] = n.z;
        vb.run_prob[vi] = run_prob;
        vb.sample[vi] = (int64_t)g;
        vb.hash_r[vi] = hr;
        vb.hash_f[vi] = hf;
        vb.parent[vi] = parent;
        vb.tri[vi] = h.tri;
        vb.code[vi] = (uint8_t)code;
        vb.depth[vi] = (uint8_t)depth;
        vb.suffix_start[vi] = (uint8_t)suffix_start;
        vb.wedge[vi] = wid;
        parent = (int)vi;
      } else {
        atomicAdd(counters + SBR_CC_VERTEX_OVERFLOW, 1ULL);
        alive = false;
        continue;
      }
      if (depth == P.max_depth) {
        alive = false;
        continue;
      }
      // _continue_rays (paths.py:855-900)
      if (code == 0) {
        const double dn = dot_seq(d, n);
        d = d - (2.0 * dn) * n;
      } else if (code == 1) {
        const double u0 = philox_uniform(P.seed, 0, (uint64_t)depth, TAG_RESPAWN, 2 * g);
        const double u1 = philox_uniform(P.seed, 0, (uint64_t)depth, TAG_RESPAWN, 2 * g + 1);
        const double cos_t = u0, azim = kTwoPi * u1;
        const double x = 1.0 - cos_t * cos_t;
        const double sin_t = sqrt(x > 0.0 ? x : 0.0);
        const double3 t1 = perp_batch(n);
        const double3 t2 = cross3(n, t1);
        double sa, ca;
        sincos(azim, &sa, &ca);
        const double a = sin_t * ca, b = sin_t * sa;
        d = make_double3((a * t1.x + b * t2.x) + cos_t * n.x, (a * t1.y + b * t2.y) + cos_t * n.y,
                         (a * t1.z + b * t2.z) + cos_t * n.z);
      } else if (code == 3) {
        // Keller cone (paths.py:881-896); edge-grazing rays terminate
        const double3 e = ldg3(S.w_ehat + 3 * wid);
        const double cb = clamp1(dot_seq(d, e));
        const double xb = 1.0 - cb * cb;
        const double sb = sqrt(xb > 0.0 ? xb : 0.0);
        if (sb < 1e-9) {
          K.terminated++;
          alive = false;
          continue;
        }
        const double phi =
            philox_uniform(P.seed, 0, (uint64_t)depth, TAG_CONE, g) * __ldg(S.w_nopen + wid) * kPi;
        double sp, cp;
        sincos(phi, &sp, &cp);
        const double a = sb * cp, b = sb * sp;
        const double3 t0 = ldg3(S.w_t0 + 3 * wid), n0 = ldg3(S.w_n0 + 3 * wid);
        d = make_double3((a * t0.x + b * n0.x) + cb * e.x, (a * t0.y + b * n0.y) + cb * e.y,
                         (a * t0.z + b * n0.z) + cb * e.z);
      }
      o = pt;
    }
  }
  const unsigned lane = threadIdx.x & 31u;
  const unsigned v[3] = {K.escaped, K.terminated, K.rb};
  const int idx[3] = {SBR_CC_SAMPLES_ESCAPED, SBR_CC_SAMPLES_TERMINATED, SBR_CC_RAY_BOUNCES};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v[k]);
    if (lane == 0 && s) atomicAdd(counters + idx[k], (unsigned long long)s);
  }
}

// ---------------------------------------------------------------------------
// vertex order: 63-bit Morton code of the interaction point
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t spread21(uint64_t x) {
  x &= 0x1fffffULL;
  x = (x | (x << 32)) & 0x1f00000000ffffULL;
  x = (x | (x << 16)) & 0x1f0000ff0000ffULL;
  x = (x | (x << 8)) & 0x100f00f00f00f00fULL;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ULL;
  x = (x | (x << 2)) & 0x1249249249249249ULL;
  return x;
}

__global__ void k_vertex_morton(const double* __restrict__ point, int64_t n, double3 lo,
                                double3 inv_ext, uint64_t* keys, int32_t* ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double p[3] = {point[3 * i], point[3 * i + 1], point[3 * i + 2]};
    const double l[3] = {lo.x, lo.y, lo.z}, ie[3] = {inv_ext.x, inv_ext.y, inv_ext.z};
    uint64_t q[3];
    for (int k = 0; k < 3; ++k) {
      double f = (p[k] - l[k]) * ie[k];
      f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
      q[k] = (uint64_t)(f * 2097151.0);
    }
    keys[i] = (spread21(q[0]) << 2) | (spread21(q[1]) << 1) | spread21(q[2]);
    ids[i] = (int32_t)i;
  }
}

// ---------------------------------------------------------------------------
// visibility: (vertex, target) pairs
// ---------------------------------------------------------------------------
// Pair p -> (group of kVisGroup tiles of 32 spatially sorted vertices,
// target, tile, vertex in tile).  A warp claims one group x target at a time
// and walks its tiles: 32 neighbouring vertices looking at the same target,
// so the occlusion rays are nearly parallel and walk the same BVH nodes.  The
// half-space side test runs first; survivors are pushed into a per-warp queue
// in shared memory and cast 32 at a time with the while-while any-hit, so
// dead lanes never enter traversal and no pair list goes through HBM.
//
// Occluder sharing (97 % of config-3 rays are occluded): a lane that finds an
// occluder publishes it to the lanes still traversing (tested at once) and to
// a two-entry per-warp ring that the next tiles of the same target test before
// traversing, and in a small per-target table (global memory, racy by
// design) that every warp working on that target tests too.  Any triangle
// with t_min < t < limit decides "occluded", so the result is exactly the
// traversal's.
constexpr int kVisWarps = 4;
#ifndef SBR_VIS_HINTS
#define SBR_VIS_HINTS 2
#endif
#ifndef SBR_VIS_GROUP
#define SBR_VIS_GROUP 8
#endif
#ifndef SBR_VIS_GHINTS
#define SBR_VIS_GHINTS 2  // per-target occluder table shared by all warps (ring 2 + table 2: 66.4 -> 63.4 ms vs 4 + 4)
#endif
constexpr int kVisGHints = SBR_VIS_GHINTS;
constexpr int kVisHints = SBR_VIS_HINTS;
constexpr int kVisGroup = SBR_VIS_GROUP;

// the visibility slab's vertices (point, facing normal, code) gathered into
// Morton order once, so every (tile, target) unit reads contiguous memory
__global__ void k_vis_view(SbrVertexBuf vb, int64_t v_begin, int64_t nv,
                           const int32_t* __restrict__ order, double* vpt, double* vnr,
                           uint8_t* vcode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = order ? order[v_begin + i] : v_begin + i;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vpt[3 * i + c] = vb.point[3 * v + c];
      vnr[3 * i + c] = vb.normal[3 * v + c];
    }
    vcode[i] = vb.code[v];
  }
}

#ifndef SBR_VIS_PACK
#define SBR_VIS_PACK 1  // config 3: 62.8 -> 60.9 ms (no 64-bit div/mod per ray)
#endif
#ifndef SBR_VIS_GHINT_EARLY
#define SBR_VIS_GHINT_EARLY 1  // config 3: 64.2 -> 62.8 ms (2: early __ldcg, 63.9)
#endif
#ifndef SBR_VIS_MINB
#define SBR_VIS_MINB 8  // 64 registers: 220 -> 180 ms at config 3
#endif
__global__ void __launch_bounds__(128, SBR_VIS_MINB) k_cir_visibility(DevScene S, SbrCirParams P,
                                                        SbrVertexBuf vb, int64_t v_begin,
                                                        int64_t v_end, uint64_t* row_key,
                                                        int32_t* row_vtx, int64_t row_cap,
                                                        unsigned long long* counters,
                                                        unsigned long long* work,
                                                        const int32_t* __restrict__ order,
                                                        int* ghint,
                                                        const double* __restrict__ vpt,
                                                        const double* __restrict__ vnr,
                                                        const uint8_t* __restrict__ vcode) {
  // vpt / vnr / vcode: point, facing normal and code of the slab's vertices in
  // Morton order (k_vis_view), so tiles read contiguous memory
  __shared__ int64_t sq[kVisWarps][64];
  __shared__ int shint[kVisWarps][kVisHints > 0 ? kVisHints : 1];
  __shared__ int shpos[kVisWarps];
  const unsigned lane = threadIdx.x & 31u;
  const unsigned wid = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t nt = P.n_targets;
  const int64_t nv = v_end - v_begin;
  const int64_t ntiles = (nv + 31) / 32;
  const int64_t ngroups = (ntiles + kVisGroup - 1) / kVisGroup;
  const int64_t total = ngroups * nt;  // claim units: (group, target)
  if ((int)lane < kVisHints) shint[wid][lane] = -1;
  if (lane == 0) shpos[wid] = 0;
  __syncwarp();
  int qn = 0;  // warp-uniform queue length
  unsigned vis = 0, dup_local = 0;
  bool more = true;
  int64_t unit = 0, g_tile0 = 0;
  int tile_cur = kVisGroup, tile_end = kVisGroup, k_cur = -1;
  while (more || qn > 0) {
    // ---- refill: side test on the next tile of the claimed (group, target)
    if (more && qn < 32) {
      if (tile_cur >= tile_end) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(work, 1ULL);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)base >= total) {
          more = false;
        } else {
          unit = (int64_t)base;
          const int64_t grp = unit / nt;
          const int k_new = (int)(unit % nt);
          const bool same_target = k_new == k_cur;
          k_cur = k_new;
          g_tile0 = grp * kVisGroup;
          tile_cur = 0;
          const int64_t left = ntiles - g_tile0;
          tile_end = left < kVisGroup ? (int)left : kVisGroup;
          if (kVisHints > 0 && !same_target) {  // hints of another target rarely help
            if ((int)lane < kVisHints) shint[wid][lane] = -1;
            __syncwarp();
          }
        }
      }
      if (more) {
        const int64_t pos = (g_tile0 + tile_cur) * 32 + lane;
        const int k = k_cur;
        ++tile_cur;
        bool pass = false;
        if (pos < nv) {
          const double3 p = ldg3(vpt + 3 * pos);
          const double3 n = ldg3(vnr + 3 * pos);
          const double3 tg = ldg3(P.targets_dev + 3 * k);
          const double side = dot_seq(tg - p, n);
          const int code = __ldg(vcode + pos);
          pass = code == 3 ? true : (code == 2 ? side < 0.0 : side > 0.0);
        }
        const unsigned m = __ballot_sync(0xffffffffu, pass);
#if SBR_VIS_PACK
        // (slab vertex, target) as two 32-bit halves: shifts, not a 64-bit div/mod
        SBR_DCHECK(S, !pass || qn + __popc(m & lt_mask) < 64);
        if (pass) sq[wid][qn + __popc(m & lt_mask)] = (int64_t)(((uint64_t)pos << 32) | (uint32_t)k);
#else
        if (pass) sq[wid][qn + __popc(m & lt_mask)] = pos * nt + k;  // (slab vertex, target)
#endif
        qn += __popc(m);
        __syncwarp();
        if (qn < 32 && more) continue;
      }
    }
    // ---- cast up to 32 queued occlusion rays
    const int take = qn < 32 ? qn : 32;
    const bool active = (int)lane < take;
    int64_t pi = 0;
    if (active) pi = sq[wid][qn - take + lane];
    __syncwarp();
    qn -= take;
    int64_t v = 0;
    int k = 0;
    double3 a = make_double3(0.0, 0.0, 0.0), b = a;
    bool cast = false;
    int sn[kStackSize];
    AnyTrav T(sn);
#if SBR_VIS_GHINT_EARLY
    // the per-target occluder table is read before the ray setup so its
    // latency overlaps the setup arithmetic; plain (L1-cacheable) loads: a
    // stale entry is still a valid candidate occluder
    int gh[kVisGHints > 0 ? kVisGHints : 1];
#endif
    if (active) {
#if SBR_VIS_PACK
      v = (int64_t)((uint64_t)pi >> 32);  // position in the slab's Morton order
      k = (int)(uint32_t)pi;
#else
      v = pi / nt;  // position in the slab's Morton order
      k = (int)(pi % nt);
#endif
#if SBR_VIS_GHINT_EARLY
#pragma unroll
      for (int h = 0; h < kVisGHints; ++h)
        gh[h] = SBR_VIS_GHINT_EARLY == 2 ? __ldcg(ghint + (int64_t)k * kVisGHints + h)
                                         : ghint[(int64_t)k * kVisGHints + h];
#endif
      a = ldg3(vpt + 3 * v);
      b = ldg3(P.targets_dev + 3 * k);
      vis++;
    }
    // occluded_batch (geometry.py:187-201): open segment, endpoints offset by eps
    if (active) {
      const double3 dd = b - a;
      const double len = norm_seq(dd);
      if (len > 2.0 * 1e-4) {
        const double3 dn = make_double3(dd.x / len, dd.y / len, dd.z / len);
        const double3 o = make_double3(a.x + 1e-4 * dn.x, a.y + 1e-4 * dn.y, a.z + 1e-4 * dn.z);
        T.start(S, o, dn, 0.0, len - 2.0 * 1e-4);
        cast = true;
      }
    }
    if (!cast) {
      T.idle();
      T.found = false;
      T.ok = true;
    }
    // occluders any warp found for this target (racy table: hints only); on
    // config 3 these settle 87 % of all rays, the warp ring below another 3 %
    for (int h = 0; h < kVisGHints; ++h) {
      if (cast && !T.found) {
#if SBR_VIS_GHINT_EARLY
        const int j = gh[h];
#else
        const int j = __ldcg(ghint + (int64_t)k * kVisGHints + h);
#endif
        if (j >= 0) T.try_occluder(S, j);
      }
    }
    // occluders found by this warp for earlier tiles of the same target
    for (int h = 0; h < kVisHints; ++h) {
      const int j = shint[wid][h];
      if (cast && !T.found && j >= 0) T.try_occluder(S, j);
    }
    while (!T.done()) {
      const bool before = T.found;
      T.round(S);
      if (kVisHints > 0) {
        const unsigned am = __activemask();
        const unsigned fresh = __ballot_sync(am, T.found && !before);
        if (fresh) {
          const int src = __ffs(fresh) - 1;
          const int j = __shfl_sync(am, T.hit_tri, src);
          if (!T.done()) T.try_occluder(S, j);
          if ((int)lane == src) {
            shint[wid][shpos[wid] % kVisHints] = j;
            if (kVisGHints > 0)
              __stcg(ghint + (int64_t)k * kVisGHints + (shpos[wid] % (kVisGHints > 0 ? kVisGHints : 1)), j);
            shpos[wid] = shpos[wid] + 1;
          }
        }
      }
    }
    __syncwarp();
    if (active && !T.ok) {
      flag_error(S, kErrStack);
      atomicAdd(counters + SBR_CC_STACK_OVERFLOW, 1ULL);
    }
    // Visible pairs become rows.  Within the batch, a chain row whose
    // (pair_r, pair_f) key another lane holds with a smaller ordinal is a
    // duplicate by construction (the selection keeps only each key's first
    // occurrence in ordinal order, and only kept rows reach truncation and
    // the DedupTable), so it is counted here instead of emitted: neighbouring
    // vertices on one facade usually share the chain and the target.
    const bool visible = active && !T.found;
    if (__any_sync(0xffffffffu, visible)) {
      int64_t vg = 0;
      uint64_t okey = ~0ULL, pr = 0, pf = 0;
      bool chain_row = false;
      if (visible) {
        vg = order ? order[v_begin + v] : v_begin + v;  // vertex buffer index
        okey = ordinal_key(vb.depth[vg], vb.sample[vg], k);
        chain_row = vb.suffix_start[vg] == 0 && vb.code[vg] != 1;
        if (chain_row) {
          pr = fnv1a_u64(vb.hash_r[vg], (uint64_t)k);
          pf = fnv1a_u64(vb.hash_f[vg], (uint64_t)k);
        }
      }
      const unsigned cand = __ballot_sync(0xffffffffu, chain_row);
      unsigned same = 0;
      if (chain_row) same = __match_any_sync(cand, pr) & __match_any_sync(cand, pf);
      bool first = true;
      if (chain_row && __popc(same) > 1) {
        // smallest ordinal of the key group (labeled-partition reductions)
        const unsigned hi = (unsigned)(okey >> 32), lo = (unsigned)okey;
        const unsigned mhi = __reduce_min_sync(same, hi);
        const unsigned top = __ballot_sync(same, hi == mhi);
        if (hi == mhi) first = lo == __reduce_min_sync(top, lo);
        else first = false;
      }
      if (visible) {
        if (chain_row && !first) {
          dup_local++;
        } else {
          const unsigned long long r = append_slot(counters + SBR_CC_ROWS);
          if ((int64_t)r < row_cap) {
            row_key[r] = okey;
            row_vtx[r] = (int32_t)vg;
          }
        }
      }
    }
  }
  const unsigned s = __reduce_add_sync(0xffffffffu, vis);
  if (lane == 0 && s) atomicAdd(counters + SBR_CC_VIS_RAYS, (unsigned long long)s);
  const unsigned sd = __reduce_add_sync(0xffffffffu, dup_local);
  if (lane == 0 && sd) atomicAdd(counters + SBR_CC_DUPLICATES, (unsigned long long)sd);
}

// ---------------------------------------------------------------------------
// selection kernels
// ---------------------------------------------------------------------------
// per row: pair hashes and the chain flag (_emit_records 919-924)
__global__ void k_row_pairs(SbrVertexBuf vb, const uint64_t* __restrict__ key,
                            const int32_t* __restrict__ row_vtx, int64_t n, uint64_t* pr,
                            uint64_t* pf, uint8_t* chain) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = row_vtx[i];
    const uint64_t k = key[i] & kTargetMask;
    pr[i] = fnv1a_u64(vb.hash_r[v], k);
    pf[i] = fnv1a_u64(vb.hash_f[v], k);
    chain[i] = (vb.suffix_start[v] == 0 && vb.code[v] != 1) ? 1 : 0;
  }
}

__global__ void k_gather_u8(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx,
                            int64_t n, uint8_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// record (row or LoS) -> (vertex, target) for k_cir_records
__global__ void k_resolve_records(const int64_t* __restrict__ rec_row,
                                  const uint64_t* __restrict__ key,
                                  const int32_t* __restrict__ row_vtx, int64_t n, int32_t* rec_vtx,
                                  int32_t* rec_target) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rec_row[i];
    if (r < 0) {
      rec_vtx[i] = -1;
      rec_target[i] = (int32_t)(~r);
    } else {
      rec_vtx[i] = row_vtx[r];
      rec_target[i] = (int32_t)(key[r] & kTargetMask);
    }
  }
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const int32_t* __restrict__ idx,
                             int64_t n, uint64_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// first occurrence of each (pr, pf) among chain rows sorted by (pr, pf, ordinal)
// First occurrence of each (pr, pf) among chain rows sorted stably by the top
// 32 bits of pr (ordinal order inside a run): a row is first unless an
// earlier row of its run has the same (pr, pf).  pr and pf are two hashes of
// one (chain, target) key, so a run almost always holds a single key and the
// scan stops at the neighbour; prefix or hash collisions between different
// keys only lengthen the scan, the result stays exact.
__global__ void k_first_flags_pr(const uint64_t* __restrict__ spr, const uint64_t* __restrict__ spf,
                                 const int32_t* __restrict__ order, int64_t n,
                                 uint8_t* keep_chain, unsigned long long* counters) {
  // spr / spf: (pr, pf) already in sorted order (contiguous reads); order:
  // the row each sorted position came from
  unsigned dup = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t ka = spr[i], fa = spf[i];
    bool first = true;
    for (int64_t j = i - 1; j >= 0; --j) {
      const uint64_t kb = spr[j];
      if ((kb >> 32) != (ka >> 32)) break;
      if (kb == ka && spf[j] == fa) {
        first = false;
        break;
      }
    }
    keep_chain[order[i]] = first ? 1 : 0;
    dup += first ? 0u : 1u;
  }
  const unsigned s = __reduce_add_sync(0xffffffffu, dup);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(counters + SBR_CC_DUPLICATES, (unsigned long long)s);
}

// Ordinal keys depth<<60 | sample<<20 | target re-packed densely (depth,
// sample and target fields only as wide as this call needs) so the radix sort
// runs over ~33 instead of 64 bits; the order is unchanged.
__global__ void k_dense_keys(const uint64_t* __restrict__ key, int64_t n, int tb, int sb,
                             uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    out[i] = ((k >> 60) << (sb + tb)) | (((k >> kTargetBits) & kSampleMask) << tb) |
             (k & kTargetMask);
  }
}

// kept rows per depth (the reference truncates depth by depth, _emit_records 954-960)
__global__ void k_kept_per_depth(const uint64_t* __restrict__ skey, const int32_t* __restrict__ kept,
                                 int64_t n, int depth_shift, unsigned long long* per_depth) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (kept[i]) atomicAdd(per_depth + (skey[i] >> depth_shift), 1ULL);
}

// kept = non-chain or first occurrence (ordinal order)
__global__ void k_kept(const uint8_t* __restrict__ chain, const uint8_t* __restrict__ keep_chain,
                       int64_t n, int32_t* kept) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    kept[i] = (!chain[i] || keep_chain[i]) ? 1 : 0;
}

// registration keys: LoS first (target order), then kept chain rows under the
// truncation cap, in ordinal order.  reg_src: >= 0 sorted-row index, < 0 ~target.
__global__ void k_reg_keys_los(const uint8_t* __restrict__ los, const int32_t* __restrict__ los_pos,
                               int n_targets, uint64_t* rk1, uint64_t* rk2, int64_t* reg_src) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_targets; k += gridDim.x * blockDim.x) {
    if (!los[k]) continue;
    const int j = los_pos[k];
    const uint64_t key = fnv1a_u64(0ULL, (uint64_t)k);  // pair_with_target(0, k)
    rk1[j] = key;
    rk2[j] = key;
    reg_src[j] = ~(int64_t)k;
  }
}

__global__ void k_reg_flags(const uint8_t* __restrict__ chain, const int32_t* __restrict__ kept,
                            const int32_t* __restrict__ kept_pos, int64_t n, int64_t n_buffer,
                            int32_t* is_reg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    is_reg[i] = (chain[i] && kept[i] && kept_pos[i] < n_buffer) ? 1 : 0;
}

__global__ void k_reg_keys_rows(const int32_t* __restrict__ is_reg, const int32_t* __restrict__ reg_pos,
                                const uint64_t* __restrict__ pr, const uint64_t* __restrict__ pf,
                                int64_t n, int64_t base, uint64_t* rk1, uint64_t* rk2,
                                int64_t* reg_src, int32_t* row_reg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!is_reg[i]) {
      row_reg[i] = -1;
      continue;
    }
    const int64_t j = base + reg_pos[i];
    rk1[j] = pr[i];
    rk2[j] = pf[i];
    reg_src[j] = i;
    row_reg[i] = (int32_t)j;
  }
}

// slot entries: (slot, key) for both slots (one entry when they coincide)
__global__ void k_slot_entries(const uint64_t* __restrict__ rk1, const uint64_t* __restrict__ rk2,
                               int64_t nreg, uint64_t n_hash, uint64_t* slot, int32_t* owner) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nreg;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t s1 = rk1[j] % n_hash, s2 = rk2[j] % n_hash;
    slot[2 * j] = s1;
    owner[2 * j] = (int32_t)j;
    // a coincident second slot becomes a sentinel sorted past every real slot
    slot[2 * j + 1] = s2 == s1 ? ~0ULL : s2;
    owner[2 * j + 1] = (int32_t)j;
  }
}

__global__ void k_entry_pos(const int32_t* __restrict__ owner, const uint64_t* __restrict__ slot,
                            int64_t ne, int32_t* pos1, int32_t* pos2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (slot[e] == ~0ULL) continue;
    const int32_t j = owner[e];
    // entries of one key: the smaller position is written to pos1 by whichever
    // lands first; use atomics so both slots get recorded
    if (atomicCAS(pos1 + j, -1, (int32_t)e) != -1) pos2[j] = (int32_t)e;
  }
}

// state: 0 undecided, 1 accepted, 2 rejected (DedupTable.register both-slot rule)
__device__ __forceinline__ int scan_slot(const uint64_t* slot, const int32_t* owner,
                                         const uint8_t* state, int32_t e) {
  // 1: some earlier key in this slot accepted; 0: all earlier rejected / none;
  // -1: an earlier key is still undecided
  const uint64_t s = slot[e];
  int res = 0;
  for (int32_t f = e - 1; f >= 0 && slot[f] == s; --f) {
    const uint8_t st = state[owner[f]];
    if (st == 1) return 1;
    if (st == 0) res = -1;
  }
  return res;
}

__global__ void k_greedy_round(const uint64_t* __restrict__ slot, const int32_t* __restrict__ owner,
                               const int32_t* __restrict__ pos1, const int32_t* __restrict__ pos2,
                               int64_t nreg, uint8_t* state, int* changed, int* undecided) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nreg;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (state[j] != 0) continue;
    const int a = scan_slot(slot, owner, state, pos1[j]);
    const int b = pos2[j] >= 0 ? scan_slot(slot, owner, state, pos2[j]) : 0;
    if (a == 1 || b == 1) {
      state[j] = 2;
      *changed = 1;
    } else if (a == 0 && b == 0) {
      state[j] = 1;
      *changed = 1;
    } else {
      *undecided = 1;
    }
  }
}

// claimed slots: slot runs holding an accepted key (DedupTable.load_factor numerator)
__global__ void k_claimed(const uint64_t* __restrict__ slot, const int32_t* __restrict__ owner,
                          const uint8_t* __restrict__ state, int64_t ne,
                          unsigned long long* counters) {
  unsigned c = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t s = slot[e];
    if (s == ~0ULL || state[owner[e]] != 1) continue;
    bool first = true;
    for (int64_t f = e - 1; f >= 0 && slot[f] == s; --f)
      if (state[owner[f]] == 1) {
        first = false;
        break;
      }
    c += first ? 1u : 0u;
  }
  const unsigned sc = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && sc) atomicAdd(counters + SBR_CC_HASH_SLOTS, (unsigned long long)sc);
}

__global__ void k_add_counter(unsigned long long* counters, int idx, unsigned long long v) {
  counters[idx] += v;
}

__global__ void k_count_states(const uint8_t* __restrict__ state, int64_t nreg,
                               unsigned long long* counters) {
  unsigned acc = 0, rej = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nreg;
       j += (int64_t)gridDim.x * blockDim.x) {
    acc += state[j] == 1;
    rej += state[j] == 2;
  }
  const unsigned a = __reduce_add_sync(0xffffffffu, acc);
  const unsigned r = __reduce_add_sync(0xffffffffu, rej);
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(counters + SBR_CC_HASH_REGISTERED, (unsigned long long)a);
    if (r) atomicAdd(counters + SBR_CC_DUPLICATES, (unsigned long long)r);
  }
}

// buffer flags: rows entering the PathBuffer (after LoS)
__global__ void k_buffer_flags(const uint8_t* __restrict__ chain, const int32_t* __restrict__ kept,
                               const int32_t* __restrict__ kept_pos,
                               const int32_t* __restrict__ row_reg,
                               const uint8_t* __restrict__ state, int64_t n, int64_t n_buffer,
                               int32_t* in_buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool b = kept[i] && kept_pos[i] < n_buffer;
    if (b && chain[i]) b = state[row_reg[i]] == 1;
    in_buf[i] = b ? 1 : 0;
  }
}

__global__ void k_los_buffer(const int64_t* __restrict__ reg_src, const uint8_t* __restrict__ state,
                             const int32_t* __restrict__ los_acc_pos, int n_los_keys,
                             int64_t n_buffer, int64_t* rec_row) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_los_keys; j += gridDim.x * blockDim.x) {
    if (state[j] != 1) continue;
    const int p = los_acc_pos[j];
    if (p >= n_buffer) continue;
    rec_row[p] = reg_src[j];  // ~target
  }
}

__global__ void k_row_buffer(const int32_t* __restrict__ in_buf, const int32_t* __restrict__ buf_pos,
                             const int32_t* __restrict__ sidx, int64_t n, int64_t base,
                             int64_t n_buffer, int64_t* rec_row) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!in_buf[i]) continue;
    const int64_t p = base + buf_pos[i];
    if (p >= n_buffer) continue;
    rec_row[p] = sidx[i];  // index into the caller's row arrays
  }
}

__global__ void k_iota64(int64_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

__global__ void k_iota(int32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// records
// ---------------------------------------------------------------------------
__global__ void k_cir_records(SbrCirParams P, SbrVertexBuf vb, const int32_t* __restrict__ rec_vtx,
                              const int32_t* __restrict__ rec_target, int64_t n, SbrRecordBuf R) {
  const int L = R.max_depth;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int v = rec_vtx[r];
    R.target[r] = rec_target[r];
    for (int j = 0; j < L; ++j) {
      R.kind[r * L + j] = -1;
      R.tri[r * L + j] = -1;
      R.wedge[r * L + j] = -1;
    }
    if (v < 0) {
      R.sample[r] = -1;
      R.depth[r] = 0;
      R.suffix_start[r] = 0;
      R.diffuse[r] = 0;
      R.chain_hash[r] = 0;
      R.prefix_prob[r] = 1.0;
      for (int c = 0; c < 3; ++c) R.anchor[3 * r + c] = P.source[c];
      continue;
    }
    const int depth = vb.depth[v];
    const int ss = vb.suffix_start[v];
    R.sample[r] = vb.sample[v];
    R.depth[r] = depth;
    R.suffix_start[r] = ss;
    R.diffuse[r] = vb.code[v] == 1 ? 1 : 0;
    R.chain_hash[r] = vb.hash_r[v];
    R.prefix_prob[r] = 1.0;
    for (int c = 0; c < 3; ++c) R.anchor[3 * r + c] = P.source[c];
    int w = v;
    for (int j = depth - 1; j >= 0 && w >= 0; --j) {
      const int64_t o = r * L + j;
      R.kind[o] = (int8_t)vb.code[w];
      R.tri[o] = vb.tri[w];
      R.wedge[o] = vb.wedge[w];
      for (int c = 0; c < 3; ++c) {
        R.vertex[3 * o + c] = vb.point[3 * w + c];
        R.normal[3 * o + c] = vb.normal[3 * w + c];
      }
      if (ss > 0 && j + 1 == ss) {
        R.prefix_prob[r] = vb.run_prob[w];
        for (int c = 0; c < 3; ++c) R.anchor[3 * r + c] = vb.point[3 * w + c];
      }
      w = vb.parent[w];
    }
  }
}

// ---------------------------------------------------------------------------
// refinement (image method)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double3 reflect_point(double3 p, double3 nrm, double3 on) {
  const double f = dot_ddot(p - on, nrm);
  return p - (2.0 * f) * nrm;
}

__global__ void __launch_bounds__(128) k_cir_refine(DevScene S, SbrCirParams P, SbrRecordBuf R,
                                                    int64_t n, double* __restrict__ pv,
                                                    int32_t* __restrict__ status,
                                                    unsigned long long* counters) {
  const int L = R.max_depth;
  const double3 src = make_double3(P.source[0], P.source[1], P.source[2]);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int depth = R.depth[r];
    const int ss = R.suffix_start[r];
    const int k = R.target[r];
    const double3 tg = ldg3(P.targets_dev + 3 * k);
    double* out = pv + r * (int64_t)(L + 2) * 3;
    for (int j = 0; j < (L + 2) * 3; ++j) out[j] = 0.0;
    out[0] = src.x;
    out[1] = src.y;
    out[2] = src.z;
    for (int j = 0; j < depth; ++j)
      for (int c = 0; c < 3; ++c) out[3 * (j + 1) + c] = R.vertex[3 * (r * L + j) + c];
    out[3 * (depth + 1)] = tg.x;
    out[3 * (depth + 1) + 1] = tg.y;
    out[3 * (depth + 1) + 2] = tg.z;
    if (R.diffuse[r] || ss >= depth) {
      status[r] = SBR_REFINE_OK;
      continue;
    }
    const int ns = depth - ss;
    const double3 anchor = ld3(R.anchor + 3 * r);
    double3 img[16];
    img[0] = anchor;
    int i_d = -1;
    for (int j = 0; j < ns; ++j) {
      const int64_t o = r * L + ss + j;
      img[j + 1] = R.kind[o] == 0
                       ? reflect_point(img[j], ld3(R.normal + 3 * o), ld3(R.vertex + 3 * o))
                       : img[j];
      if (R.kind[o] == 3 && i_d < 0) i_d = j;
    }
    int st = SBR_REFINE_OK;
    // diffraction: the edge seen through every later reflection (paths.py:1163-1191)
    double3 eo[16], ee[16];
    double x = 0.0;
    if (i_d >= 0) {
      const int w = R.wedge[r * L + ss + i_d];
      eo[i_d] = ldg3(S.w_origin + 3 * w);
      ee[i_d] = ldg3(S.w_ehat + 3 * w);
      for (int j = i_d + 1; j < ns; ++j) {
        const int64_t o = r * L + ss + j;
        if (R.kind[o] == 0) {
          const double3 nn = ld3(R.normal + 3 * o);
          eo[j] = reflect_point(eo[j - 1], nn, ld3(R.vertex + 3 * o));
          ee[j] = reflect_vec(ee[j - 1], nn);
        } else {
          eo[j] = eo[j - 1];
          ee[j] = ee[j - 1];
        }
      }
      if (!solve_diffraction_point(img[ns], tg, eo[ns - 1], ee[ns - 1], x))
        st = SBR_REFINE_DEGENERATE;
      else if (!(0.0 <= x && x <= __ldg(S.w_len + w)))
        st = SBR_REFINE_OFF_EDGE;
    }
    double3 from = tg;
    double3 first = tg;
    for (int j = ns - 1; st == SBR_REFINE_OK && j >= 0; --j) {
      const int64_t o = r * L + ss + j;
      if (j == i_d) {
        const double3 vtx = eo[i_d] + x * ee[i_d];
        bool fine;
        if (occluded_segment(S, from, vtx, 1e-4, fine)) st = SBR_REFINE_OCCLUDED;
        if (!fine) flag_error(S, kErrStack);
        if (st != SBR_REFINE_OK) break;
        out[3 * (ss + j + 1)] = vtx.x;
        out[3 * (ss + j + 1) + 1] = vtx.y;
        out[3 * (ss + j + 1) + 2] = vtx.z;
        from = vtx;
        first = vtx;
        continue;
      }
      const double3 aim = (i_d < 0 || j < i_d) ? img[j + 1] : eo[j] + x * ee[j];
      double3 ray = aim - from;
      const double len = sqrt(dot_ddot(ray, ray));
      if (len < 1e-12) {
        st = SBR_REFINE_DEGENERATE;
        break;
      }
      ray = make_double3(ray.x / len, ray.y / len, ray.z / len);
      HitRecord h;
      if (!trace_closest(S, from, ray, 1e-4, __longlong_as_double(0x7ff0000000000000LL), h)) {
        flag_error(S, kErrStack);
        atomicAdd(counters + SBR_CC_STACK_OVERFLOW, 1ULL);
      }
      if (h.tri < 0) {
        st = SBR_REFINE_COPLANAR_MISS;
        break;
      }
      const double3 hn = ldg3(S.normals + 3 * (int64_t)h.tri);
      const double3 sn = ld3(R.normal + 3 * o);
      const double3 hp = from + h.t * ray;
      if (fabs(dot_ddot(hn, sn)) < 1.0 - 1e-6 ||
          !(fabs(dot_ddot(hp - ld3(R.vertex + 3 * o), sn)) <= 1e-6)) {
        st = SBR_REFINE_COPLANAR_MISS;
        break;
      }
      out[3 * (ss + j + 1)] = hp.x;
      out[3 * (ss + j + 1) + 1] = hp.y;
      out[3 * (ss + j + 1) + 2] = hp.z;
      from = hp;
      first = hp;
    }
    if (st == SBR_REFINE_OK) {
      bool fine;
      if (occluded_segment(S, anchor, first, 1e-4, fine)) st = SBR_REFINE_OCCLUDED;
      if (!fine) flag_error(S, kErrStack);
    }
    status[r] = st;
    if (st == SBR_REFINE_COPLANAR_MISS) atomicAdd(counters + SBR_CC_REJ_COPLANAR, 1ULL);
    if (st == SBR_REFINE_OCCLUDED) atomicAdd(counters + SBR_CC_REJ_OCCLUDED, 1ULL);
    if (st == SBR_REFINE_DEGENERATE) atomicAdd(counters + SBR_CC_REJ_DEGENERATE, 1ULL);
    if (st == SBR_REFINE_OFF_EDGE) atomicAdd(counters + SBR_CC_REJ_OFF_EDGE, 1ULL);
  }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
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

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess) {                                                             \
      rc = set_error(SBR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
      goto done;                                                                         \
    }                                                                                    \
  } while (0)

#define LK(what)                                 \
  do {                                           \
    if ((rc = launch_status(what)) != SBR_OK) goto done; \
  } while (0)

// stream-ordered scratch arena (freed at the end of a call)
struct Arena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  bool ok = true;
  explicit Arena(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(int64_t count) {
    void* p = nullptr;
    if (scratch_alloc(&p, sizeof(T) * (size_t)(count > 0 ? count : 1), st) != cudaSuccess) {
      ok = false;
      return nullptr;
    }
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

int check_cir(const SbrScene* scene, const SbrCirParams* P) {
  if (!P) return set_error(SBR_ERR_INVALID, "NULL params");
  if (scene && !dev_view(scene).mats) return set_error(SBR_ERR_INVALID, "scene has no material table");
  if (P->max_depth < 0 || P->max_depth > 15) return set_error(SBR_ERR_INVALID, "max_depth must lie in [0, 15]");

  if (P->n_targets < 1 || P->n_targets > (1 << kTargetBits))
    return set_error(SBR_ERR_INVALID, "need 1 .. 2^20 targets");
  if (P->num_samples < 1 || P->num_samples > kSampleMask)
    return set_error(SBR_ERR_INVALID, "num_samples must lie in [1, 2^40)");
  return SBR_OK;
}

}  // namespace

extern "C" {

int sbr_cir_sweep(const SbrScene* scene, const SbrCirParams* P, uint64_t begin, uint64_t end,
                  const SbrVertexBuf* vb, uint64_t* counters, void* stream) {
  int rc = check_cir(scene, P);
  if (rc) return rc;
  if (!scene || !vb) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (end > P->num_samples || begin > end) return set_error(SBR_ERR_INVALID, "bad sample range");
  if (end == begin || P->max_depth == 0) return SBR_OK;
  prof_begin(stream, "k_cir_sweep");
  const uint64_t F = comb_stride(P->num_samples);
  k_cir_sweep<<<grid_for((int64_t)(end - begin), 128, 148 * 16), 128, 0, (cudaStream_t)stream>>>(
      dev_view(scene), *P, begin, end, *vb, (unsigned long long*)counters,
      ShardMap{0u, 1u, kCirShardLog2}, CombMap{(end - begin + F - 1) / F, F});
  prof_end(stream);
  return launch_status("k_cir_sweep");
}

int sbr_cir_sweep_sharded(const SbrScene* scene, const SbrCirParams* P, int32_t shard_index,
                          int32_t shard_count, const SbrVertexBuf* vb, uint64_t* counters,
                          void* stream) {
  int rc = check_cir(scene, P);
  if (rc) return rc;
  if (!scene || !vb) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
    return set_error(SBR_ERR_INVALID, "bad shard");
  const uint64_t n = shard_size(P->num_samples, (uint32_t)shard_index, (uint32_t)shard_count,
                                kCirShardLog2);
  if (n == 0 || P->max_depth == 0) return SBR_OK;
  prof_begin(stream, "k_cir_sweep");
  const uint64_t F = comb_stride(P->num_samples);
  k_cir_sweep<<<grid_for((int64_t)n, 128, 148 * 16), 128, 0, (cudaStream_t)stream>>>(
      dev_view(scene), *P, 0, n, *vb, (unsigned long long*)counters,
      ShardMap{(uint32_t)shard_index, (uint32_t)shard_count, kCirShardLog2},
      CombMap{(n + F - 1) / F, F});
  prof_end(stream);
  return launch_status("k_cir_sweep");
}

int sbr_cir_vertex_order(const SbrScene* scene, const SbrVertexBuf* vb, int64_t nv,
                         int32_t* order, void* stream) {
  if (!scene || !vb || !order) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (nv <= 0) return SBR_OK;
  if (nv >= (1LL << 31)) return set_error(SBR_ERR_INVALID, "too many vertices");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = SBR_OK;
  const DevScene S = dev_view(scene);
  double3 lo = make_double3(S.bounds_lo[0], S.bounds_lo[1], S.bounds_lo[2]);
  double3 ie;
  {
    const double ex = S.bounds_hi[0] - S.bounds_lo[0], ey = S.bounds_hi[1] - S.bounds_lo[1],
                 ez = S.bounds_hi[2] - S.bounds_lo[2];
    // one cubic grid (not per-axis stretching): a tile of 32 Morton-adjacent
    // vertices is then spatially compact in flat scenes (config-3
    // visibility 150 -> 125 ms)
    const double e = fmax(fmax(ex, ey), ez);
    ie = make_double3(e > 0 ? 1.0 / e : 0.0, e > 0 ? 1.0 / e : 0.0, e > 0 ? 1.0 / e : 0.0);
  }
  Arena A(st);
  uint64_t* keys = A.get<uint64_t>(nv);
  uint64_t* keys2 = A.get<uint64_t>(nv);
  int32_t* ids = A.get<int32_t>(nv);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "vertex order scratch");
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, ids, order, (int)nv, 0, 63, st);
  void* tmp = A.get<uint8_t>((int64_t)tb);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "vertex order scratch");
  k_vertex_morton<<<grid_for(nv, 256), 256, 0, st>>>(vb->point, nv, lo, ie, keys, ids);
  LK("k_vertex_morton");
  CK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, ids, order, (int)nv, 0, 63, st));
  count_launch();
done:
  return rc;
}

int sbr_cir_visibility(const SbrScene* scene, const SbrCirParams* P, const SbrVertexBuf* vb,
                       int64_t v_begin, int64_t v_end, const int32_t* order, uint64_t* row_key,
                       int32_t* row_vtx, int64_t row_cap, uint64_t* counters, void* stream) {
  int rc = check_cir(scene, P);
  if (rc) return rc;
  if (!scene || !vb) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (v_end <= v_begin) return SBR_OK;
  if (v_end - v_begin > INT32_MAX)  // queue entries pack the slab position in 32 bits
    return set_error(SBR_ERR_INVALID, "visibility slab larger than 2^31 vertices");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* work = nullptr;
  if (scratch_alloc((void**)&work, sizeof(unsigned long long), st) != cudaSuccess)
    return set_error(SBR_ERR_NOMEM, "work counter");
  cudaMemsetAsync(work, 0, sizeof(unsigned long long), st);
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cir_visibility, 128, 0);
  if (per_sm < 1) per_sm = 1;
  prof_begin(stream, "k_cir_visibility");
  int* ghint = nullptr;
  if (kVisGHints > 0) {
    const size_t gb = sizeof(int) * (size_t)P->n_targets * kVisGHints;
    if (scratch_alloc((void**)&ghint, gb, st) != cudaSuccess) {
      cudaFreeAsync(work, st);
      return set_error(SBR_ERR_NOMEM, "occluder hints");
    }
    cudaMemsetAsync(ghint, 0xff, gb, st);
  }
  const int64_t nvs = v_end - v_begin;
  double *vpt = nullptr, *vnr = nullptr;
  uint8_t* vcode = nullptr;
  if (scratch_alloc((void**)&vpt, sizeof(double) * 3 * nvs, st) != cudaSuccess ||
      scratch_alloc((void**)&vnr, sizeof(double) * 3 * nvs, st) != cudaSuccess ||
      scratch_alloc((void**)&vcode, nvs, st) != cudaSuccess) {
    if (vpt) cudaFreeAsync(vpt, st);
    if (vnr) cudaFreeAsync(vnr, st);
    cudaFreeAsync(work, st);
    if (ghint) cudaFreeAsync(ghint, st);
    return set_error(SBR_ERR_NOMEM, "visibility vertex view");
  }
  k_vis_view<<<grid_for(nvs, 256), 256, 0, st>>>(*vb, v_begin, nvs, order, vpt, vnr, vcode);
  count_launch();
  k_cir_visibility<<<sms * per_sm, 128, 0, st>>>(dev_view(scene), *P, *vb, v_begin, v_end,
                                                 row_key, row_vtx, row_cap,
                                                 (unsigned long long*)counters, work, order,
                                                 ghint, vpt, vnr, vcode);
  prof_end(stream);
  rc = launch_status("k_cir_visibility");
  cudaFreeAsync(work, st);
  if (ghint) cudaFreeAsync(ghint, st);
  cudaFreeAsync(vpt, st);
  cudaFreeAsync(vnr, st);
  cudaFreeAsync(vcode, st);
  return rc;
}

int sbr_cir_row_pairs(const SbrVertexBuf* vb, const uint64_t* row_key, const int32_t* row_vtx,
                      int64_t n, uint64_t* pr, uint64_t* pf, uint8_t* chain, void* stream) {
  if (!vb) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (n <= 0) return SBR_OK;
  k_row_pairs<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*vb, row_key, row_vtx, n, pr,
                                                                  pf, chain);
  return launch_status("k_row_pairs");
}

int sbr_cir_resolve_records(const int64_t* rec_row, int64_t n, const uint64_t* row_key,
                            const int32_t* row_vtx, int32_t* rec_vtx, int32_t* rec_target,
                            void* stream) {
  if (n <= 0) return SBR_OK;
  k_resolve_records<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(rec_row, row_key, row_vtx,
                                                                        n, rec_vtx, rec_target);
  return launch_status("k_resolve_records");
}

// Shard-local pre-selection for multi-GPU CIR: within one shard's rows keep
// every non-chain row and the first occurrence (ordinal order) of each
// (pr, pf) among chain rows.  The global first occurrence of a key is the
// minimum over the shards' local firsts, and every later selection step
// (truncation per depth, DedupTable registration) only looks at kept rows, so
// all-gathering the kept rows gives the same selection as gathering all of
// them; the dropped rows are duplicates (returned in *n_dup to be added to
// the global duplicates counter).  kept_idx: ascending row indices.
int sbr_cir_local_dedup(const SbrCirParams* P, const uint64_t* row_key, const uint64_t* row_pr,
                        const uint64_t* row_pf, const uint8_t* row_chain, int64_t n,
                        int64_t* kept_idx, int64_t* n_kept, uint64_t* n_dup, void* stream) {
  int rc = check_cir(nullptr, P);
  if (rc) return rc;
  if (!n_kept || !n_dup) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (n >= (1LL << 31)) return set_error(SBR_ERR_INVALID, "too many rows");
  *n_kept = 0;
  *n_dup = 0;
  if (n <= 0) return SBR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nt = P->n_targets;
  int tbits = 1, sbits = 1;
  while (tbits < kTargetBits && (1LL << tbits) < (int64_t)nt) ++tbits;
  while (sbits < kSampleBits && (1ULL << sbits) < P->num_samples) ++sbits;
  const bool dense = tbits + sbits + 4 <= 64;
  const int key_bits = dense ? tbits + sbits + 4 : 64;
  Arena A(st);
  uint64_t* dkey = A.get<uint64_t>(n);
  uint64_t* skey = A.get<uint64_t>(n);
  int32_t* idx0 = A.get<int32_t>(n);
  int32_t* sidx = A.get<int32_t>(n);
  uint8_t* chain_s = A.get<uint8_t>(n);
  int32_t* cpos = A.get<int32_t>(n);
  int32_t* cpos2 = A.get<int32_t>(n);
  uint64_t* ck = A.get<uint64_t>(n);
  uint64_t* ck2 = A.get<uint64_t>(n);
  uint8_t* keep_chain = A.get<uint8_t>(n);
  int32_t* kept = A.get<int32_t>(n);
  int64_t* kidx = A.get<int64_t>(n);
  int64_t* d_count = A.get<int64_t>(2);
  unsigned long long* cnt = A.get<unsigned long long>(SBR_CC_COUNT);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "local dedup scratch");
  size_t tmp_bytes = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, skey, skey, idx0, sidx, (int)n, 0, 64, st);
  cub::DeviceSelect::Flagged(nullptr, t2, idx0, chain_s, cpos, d_count, (int)n, st);
  tmp_bytes = std::max(tmp_bytes, t2);
  void* tmp = A.get<uint8_t>((int64_t)tmp_bytes);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "local dedup scratch");
  {
    int64_t n_chain = 0, nk = 0;
    unsigned long long dup = 0;
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * SBR_CC_COUNT, st));
    CK(cudaMemsetAsync(keep_chain, 0, n, st));
    k_iota<<<grid_for(n, 256), 256, 0, st>>>(idx0, n);
    LK("k_iota");
    const uint64_t* sort_in = row_key;
    if (dense && tbits + sbits < 60) {
      k_dense_keys<<<grid_for(n, 256), 256, 0, st>>>(row_key, n, tbits, sbits, dkey);
      LK("k_dense_keys");
      sort_in = dkey;
    }
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, sort_in, skey, idx0, sidx, (int)n, 0,
                                       key_bits, st));
    count_launch();
    // chain rows, as original indices, in ordinal order
    k_gather_u8<<<grid_for(n, 256), 256, 0, st>>>(row_chain, sidx, n, chain_s);
    LK("k_gather_u8");
    CK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, sidx, chain_s, cpos, d_count, (int)n, st));
    count_launch();
    CK(cudaMemcpyAsync(&n_chain, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n_chain > 0) {
      k_gather_u64<<<grid_for(n_chain, 256), 256, 0, st>>>(row_pr, cpos, n_chain, ck);
      LK("k_gather_u64");
      CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ck, ck2, cpos, cpos2, (int)n_chain, 32,
                                         64, st));
      count_launch();
      k_gather_u64<<<grid_for(n_chain, 256), 256, 0, st>>>(row_pf, cpos2, n_chain, ck);
      LK("k_gather_u64");
      k_first_flags_pr<<<grid_for(n_chain, 256), 256, 0, st>>>(ck2, ck, cpos2, n_chain,
                                                                keep_chain, cnt);
      LK("k_first_flags_pr");
    }
    k_kept<<<grid_for(n, 256), 256, 0, st>>>(row_chain, keep_chain, n, kept);
    LK("k_kept");
    k_iota64<<<grid_for(n, 256), 256, 0, st>>>(kidx, n);
    LK("k_iota64");
    CK(cub::DeviceSelect::Flagged(nullptr, t2, kidx, kept, kept_idx, d_count + 1, (int)n, st));
    if (t2 > tmp_bytes) {
      rc = set_error(SBR_ERR_NOMEM, "local dedup scratch");
      goto done;
    }
    CK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, kidx, kept, kept_idx, d_count + 1, (int)n, st));
    count_launch();
    CK(cudaMemcpyAsync(&nk, d_count + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&dup, cnt + SBR_CC_DUPLICATES, sizeof(dup), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *n_kept = nk;
    *n_dup = dup;
  }
done:
  return rc;
}

int sbr_cir_select(const SbrCirParams* P, const uint64_t* row_key, const uint64_t* row_pr,
                   const uint64_t* row_pf, const uint8_t* row_chain, int64_t n,
                   const uint8_t* los, uint64_t n_hash, int64_t n_buffer, int64_t* rec_row,
                   int64_t* n_records, uint64_t* counters_u64, void* stream) {
  int rc = check_cir(nullptr, P);
  if (rc) return rc;
  if (!n_records || !los) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (n_hash < 1 || n_buffer < 1) return set_error(SBR_ERR_INVALID, "capacity must be positive");
  if (n >= (1LL << 31)) return set_error(SBR_ERR_INVALID, "too many rows");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* counters = (unsigned long long*)counters_u64;
  const int nt = P->n_targets;
  Arena A(st);
  // dense ordinal key widths (k_dense_keys): target, sample, 4 depth bits
  int tbits = 1, sbits = 1;
  while (tbits < kTargetBits && (1LL << tbits) < (int64_t)nt) ++tbits;
  while (sbits < kSampleBits && (1ULL << sbits) < P->num_samples) ++sbits;
  const bool dense = tbits + sbits + 4 <= 64;
  const int depth_shift = dense ? tbits + sbits : 60;
  const int key_bits = dense ? tbits + sbits + 4 : 64;
  int64_t nreg = 0, n_los_keys = 0, n_chain = 0;
  int hflag[2];
  int64_t n_los_acc = 0, n_rows_buf = 0;
  *n_records = 0;
  {
    // ---- LoS key positions ----
    int32_t* los_pos = A.get<int32_t>(nt + 1);
    // ---- sorted rows ----
    uint64_t* skey = A.get<uint64_t>(n);
    int32_t* idx0 = A.get<int32_t>(n);
    int32_t* sidx = A.get<int32_t>(n);
    uint64_t* pr = A.get<uint64_t>(n);
    uint64_t* pf = A.get<uint64_t>(n);
    uint8_t* chain = A.get<uint8_t>(n);
    uint8_t* keep_chain = A.get<uint8_t>(n);
    int32_t* kept = A.get<int32_t>(n);
    int32_t* kept_pos = A.get<int32_t>(n + 1);
    int64_t* d_count = A.get<int64_t>(4);
    if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
    size_t tmp_bytes = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, skey, skey, idx0, sidx, (int)n, 0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, kept, kept_pos, (int)n + 1, st);
    tmp_bytes = std::max(tmp_bytes, t2);
    cub::DeviceSelect::Flagged(nullptr, t2, idx0, chain, sidx, d_count, (int)n, st);
    tmp_bytes = std::max(tmp_bytes, t2);
    void* tmp = A.get<uint8_t>((int64_t)tmp_bytes);
    if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");

    // LoS key positions: unoccluded targets in target order (generate_candidates 1036-1049)
    {
      std::vector<uint8_t> h(nt);
      std::vector<int32_t> h32(nt + 1, 0);
      CK(cudaMemcpyAsync(h.data(), los, nt, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      int32_t acc = 0;
      for (int k = 0; k < nt; ++k) {
        h32[k] = acc;
        acc += h[k] ? 1 : 0;
      }
      h32[nt] = acc;
      n_los_keys = acc;
      CK(cudaMemcpyAsync(los_pos, h32.data(), sizeof(int32_t) * (nt + 1), cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }

    if (n > 0) {
      k_iota<<<grid_for(n, 256), 256, 0, st>>>(idx0, n);
      LK("k_iota");
      const uint64_t* sort_in = row_key;
      if (depth_shift < 60) {
        k_dense_keys<<<grid_for(n, 256), 256, 0, st>>>(row_key, n, tbits, sbits, pr);
        LK("k_dense_keys");
        sort_in = pr;  // pr is free until the gathers below
      }
      CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, sort_in, skey, idx0, sidx, (int)n, 0,
                                         key_bits, st));
      count_launch();
      // pair hashes / chain flags into ordinal order
      k_gather_u64<<<grid_for(n, 256), 256, 0, st>>>(row_pr, sidx, n, pr);
      LK("k_gather_u64");
      k_gather_u64<<<grid_for(n, 256), 256, 0, st>>>(row_pf, sidx, n, pf);
      LK("k_gather_u64");
      k_gather_u8<<<grid_for(n, 256), 256, 0, st>>>(row_chain, sidx, n, chain);
      LK("k_gather_u8");
      // chain rows (positions in ordinal order)
      int32_t* cpos = A.get<int32_t>(n);
      int32_t* cpos2 = A.get<int32_t>(n);
      uint64_t* ck = A.get<uint64_t>(n);
      uint64_t* ck2 = A.get<uint64_t>(n);
      if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
      k_iota<<<grid_for(n, 256), 256, 0, st>>>(idx0, n);
      LK("k_iota");
      CK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, idx0, chain, cpos, d_count, (int)n, st));
      count_launch();
      CK(cudaMemcpyAsync(&n_chain, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaMemsetAsync(keep_chain, 0, n, st));
      if (n_chain > 0) {
        // one stable sort by the top 32 bits of pr keeps ordinal order inside
        // each run; k_first_flags_pr compares full (pr, pf) within a run
        k_gather_u64<<<grid_for(n_chain, 256), 256, 0, st>>>(pr, cpos, n_chain, ck);
        LK("k_gather_u64");
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ck, ck2, cpos, cpos2, (int)n_chain, 32, 64, st));
        count_launch();
        k_gather_u64<<<grid_for(n_chain, 256), 256, 0, st>>>(pf, cpos2, n_chain, ck);
        LK("k_gather_u64");
        k_first_flags_pr<<<grid_for(n_chain, 256), 256, 0, st>>>(ck2, ck, cpos2, n_chain, keep_chain,
                                                                  counters);
        LK("k_first_flags_pr");
      }
      k_kept<<<grid_for(n, 256), 256, 0, st>>>(chain, keep_chain, n, kept);
      LK("k_kept");
      CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, kept, kept_pos, (int)n, st));
      count_launch();
    }
    int64_t n_kept = 0;
    if (n > 0) {
      int32_t lastp = 0, lastk = 0;
      CK(cudaMemcpyAsync(&lastp, kept_pos + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&lastk, kept + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      n_kept = (int64_t)lastp + lastk;
    }
    if (n_kept > n_buffer) {
      // _emit_records: room = capacity - emitted_total per depth; a depth whose
      // rows are all cut (room == 0) returns no batch, so its truncation is not
      // counted -- only the depth that crosses the cap contributes.
      unsigned long long* per_depth = A.get<unsigned long long>(16);
      if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
      CK(cudaMemsetAsync(per_depth, 0, 16 * sizeof(unsigned long long), st));
      k_kept_per_depth<<<grid_for(n, 256), 256, 0, st>>>(skey, kept, n, depth_shift, per_depth);
      LK("k_kept_per_depth");
      unsigned long long hd[16];
      CK(cudaMemcpyAsync(hd, per_depth, sizeof hd, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      int64_t emitted = 0;
      unsigned long long truncated = 0;
      for (int d = 0; d < 16; ++d) {
        const int64_t rows = (int64_t)hd[d];
        if (rows == 0) continue;
        const int64_t room = n_buffer - emitted > 0 ? n_buffer - emitted : 0;
        if (rows > room) {
          if (room > 0) truncated += (unsigned long long)(rows - room);
          emitted += room;
        } else {
          emitted += rows;
        }
      }
      if (truncated) {
        k_add_counter<<<1, 1, 0, st>>>(counters, SBR_CC_CHUNK_TRUNCATED, truncated);
        LK("k_add_counter");
      }
    }

    // ---- registration keys ----
    int32_t* is_reg = A.get<int32_t>(n);
    int32_t* reg_pos = A.get<int32_t>(n + 1);
    int32_t* row_reg = A.get<int32_t>(n);
    if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
    int64_t n_row_keys = 0;
    if (n > 0) {
      k_reg_flags<<<grid_for(n, 256), 256, 0, st>>>(chain, kept, kept_pos, n, n_buffer, is_reg);
      LK("k_reg_flags");
      CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, is_reg, reg_pos, (int)n, st));
      count_launch();
      int32_t lastp = 0, lastk = 0;
      CK(cudaMemcpyAsync(&lastp, reg_pos + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&lastk, is_reg + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      n_row_keys = (int64_t)lastp + lastk;
    }
    nreg = n_los_keys + n_row_keys;
    uint64_t* rk1 = A.get<uint64_t>(nreg);
    uint64_t* rk2 = A.get<uint64_t>(nreg);
    int64_t* reg_src = A.get<int64_t>(nreg);
    uint8_t* state = A.get<uint8_t>(nreg);
    int32_t* pos1 = A.get<int32_t>(nreg);
    int32_t* pos2 = A.get<int32_t>(nreg);
    uint64_t* eslot = A.get<uint64_t>(2 * nreg);
    uint64_t* eslot2 = A.get<uint64_t>(2 * nreg);
    int32_t* eown = A.get<int32_t>(2 * nreg);
    int32_t* eown2 = A.get<int32_t>(2 * nreg);
    int* flags = A.get<int>(2);
    if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
    k_reg_keys_los<<<grid_for(nt, 256), 256, 0, st>>>(los, los_pos, nt, rk1, rk2, reg_src);
    LK("k_reg_keys_los");
    if (n > 0) {
      k_reg_keys_rows<<<grid_for(n, 256), 256, 0, st>>>(is_reg, reg_pos, pr, pf, n, n_los_keys, rk1,
                                                       rk2, reg_src, row_reg);
      LK("k_reg_keys_rows");
    }
    if (nreg > 0) {
      k_slot_entries<<<grid_for(nreg, 256), 256, 0, st>>>(rk1, rk2, nreg, n_hash, eslot, eown);
      LK("k_slot_entries");
      size_t sb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, sb, eslot, eslot2, eown, eown2, (int)(2 * nreg), 0, 64, st);
      void* stmp = A.get<uint8_t>((int64_t)sb);
      if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
      CK(cub::DeviceRadixSort::SortPairs(stmp, sb, eslot, eslot2, eown, eown2, (int)(2 * nreg), 0, 64, st));
      count_launch();
      CK(cudaMemsetAsync(pos1, 0xff, sizeof(int32_t) * nreg, st));
      CK(cudaMemsetAsync(pos2, 0xff, sizeof(int32_t) * nreg, st));
      k_entry_pos<<<grid_for(2 * nreg, 256), 256, 0, st>>>(eown2, eslot2, 2 * nreg, pos1, pos2);
      LK("k_entry_pos");
      CK(cudaMemsetAsync(state, 0, nreg, st));
      for (int round = 0; round < 1000000; ++round) {
        CK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
        k_greedy_round<<<grid_for(nreg, 256), 256, 0, st>>>(eslot2, eown2, pos1, pos2, nreg, state,
                                                           flags, flags + 1);
        LK("k_greedy_round");
        CK(cudaMemcpyAsync(hflag, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!hflag[1]) break;
        if (!hflag[0]) {
          rc = set_error(SBR_ERR_CUDA, "dedup registration did not converge");
          goto done;
        }
      }
      k_count_states<<<grid_for(nreg, 256), 256, 0, st>>>(state, nreg, counters);
      LK("k_count_states");
      k_claimed<<<grid_for(2 * nreg, 256), 256, 0, st>>>(eslot2, eown2, state, 2 * nreg, counters);
      LK("k_claimed");
    }

    // ---- buffer: accepted LoS, then rows ----
    std::vector<uint8_t> hstate(n_los_keys);
    if (n_los_keys) {
      CK(cudaMemcpyAsync(hstate.data(), state, n_los_keys, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    std::vector<int32_t> hlos_acc(n_los_keys + 1, 0);
    for (int64_t j = 0; j < n_los_keys; ++j) {
      hlos_acc[j] = (int32_t)n_los_acc;
      n_los_acc += hstate[j] == 1;
    }
    int32_t* los_acc_pos = A.get<int32_t>(n_los_keys + 1);
    int32_t* in_buf = A.get<int32_t>(n);
    int32_t* buf_pos = A.get<int32_t>(n + 1);
    if (!A.ok) return set_error(SBR_ERR_NOMEM, "select scratch");
    if (n_los_keys) {
      CK(cudaMemcpyAsync(los_acc_pos, hlos_acc.data(), sizeof(int32_t) * n_los_keys,
                         cudaMemcpyHostToDevice, st));
      k_los_buffer<<<grid_for(n_los_keys, 256), 256, 0, st>>>(reg_src, state, los_acc_pos,
                                                             (int)n_los_keys, n_buffer, rec_row);
      LK("k_los_buffer");
    }
    if (n > 0) {
      k_buffer_flags<<<grid_for(n, 256), 256, 0, st>>>(chain, kept, kept_pos, row_reg, state, n,
                                                      n_buffer, in_buf);
      LK("k_buffer_flags");
      CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in_buf, buf_pos, (int)n, st));
      count_launch();
      int32_t lastp = 0, lastk = 0;
      CK(cudaMemcpyAsync(&lastp, buf_pos + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&lastk, in_buf + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      n_rows_buf = (int64_t)lastp + lastk;
      k_row_buffer<<<grid_for(n, 256), 256, 0, st>>>(in_buf, buf_pos, sidx, n, n_los_acc,
                                                    n_buffer, rec_row);
      LK("k_row_buffer");
    }
    const int64_t total = n_los_acc + n_rows_buf;
    const int64_t nrec = total < n_buffer ? total : n_buffer;
    if (total > nrec) {
      k_add_counter<<<1, 1, 0, st>>>(counters, SBR_CC_BUFFER_OVERFLOW,
                                     (unsigned long long)(total - nrec));
      LK("k_add_counter");
    }
    k_add_counter<<<1, 1, 0, st>>>(counters, SBR_CC_CANDIDATES, (unsigned long long)nrec);
    LK("k_add_counter");
    CK(cudaStreamSynchronize(st));
    *n_records = nrec;
  }
done:
  return rc;
}

int sbr_cir_records(const SbrCirParams* P, const SbrVertexBuf* vb, const int32_t* rec_vtx,
                    const int32_t* rec_target, int64_t n, const SbrRecordBuf* out, void* stream) {
  if (!P || !vb || !out) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (out->max_depth < 1 || out->max_depth > 15) return set_error(SBR_ERR_INVALID, "bad max_depth");
  if (n <= 0) return SBR_OK;
  k_cir_records<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(*P, *vb, rec_vtx, rec_target, n,
                                                                   *out);
  return launch_status("k_cir_records");
}

int sbr_cir_refine(const SbrScene* scene, const SbrCirParams* P, const SbrRecordBuf* rec,
                   int64_t n, double* pv, int32_t* status, uint64_t* counters, void* stream) {
  int rc = check_cir(scene, P);
  if (rc) return rc;
  if (!scene || !rec) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (rec->max_depth < 1 || rec->max_depth > 15) return set_error(SBR_ERR_INVALID, "bad max_depth");
  if (n <= 0) return SBR_OK;
  k_cir_refine<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      dev_view(scene), *P, *rec, n, pv, status, (unsigned long long*)counters);
  return launch_status("k_cir_refine");
}

}  // extern "C"
