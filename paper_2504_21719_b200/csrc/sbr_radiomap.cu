// sbr_radiomap.cu -- radio-map SBR as a wavefront pipeline, plus the analytic direct term.
//
// Replaces emtrace radiomap.py:_map_chunk (347-563) and _direct_cells
// (566-583).  The reference loops over segments with every active ray of a
// chunk in lockstep (numpy rows); here each segment is two kernels over a
// compacted HBM ray queue:
//
//   k_map_trace   persistent, warp-batched closest-hit traversal in the
//                 while-while form (sbr_common.cuh trace_closest_ww): lean
//                 code, ~70 registers, so many warps hide the L1/L2 latency
//                 of node and triangle fetches.  Segment 0 generates its rays
//                 from global sample ids (Fibonacci lattice) on the fly.
//   k_map_shade   one thread per ray: plane crossing + deposit (float64 atomics
//                 into the L2-resident grid), escape / depth exit, threshold +
//                 Russian roulette, slab Fresnel energies, inverse-CDF draw,
//                 R / S / T field and direction update; survivors are appended
//                 to the next queue with warp-aggregated atomics (live-ray
//                 compaction between bounces).
//
// Queue counts live in device memory, so a whole map is a fixed sequence of
// launches with no host synchronisation.  Rays are keyed by their global
// sample id g; the RNG streams are (seed, g >> 19, seg, tag)[g & (2^19-1)],
// so queue order never affects the result.  Per ray-bounce HBM traffic is
// ~48 B (trace in) + 12 B (hit) + ~2 x 136 B (shade in/out) = ~330 B, i.e.
// ~2 ms per 1e7-ray map at HBM speed: the pipeline stays compute bound.
#include <cooperative_groups.h>

#include <atomic>
#include <string>

#include "sbr_utd.cuh"

namespace cg = cooperative_groups;

struct SbrScene;

namespace sbr {
DevScene dev_view(const SbrScene* s);
int set_error(int code, const std::string& msg);
}  // namespace sbr

using namespace sbr;

namespace {

// Exact cell accumulator (opt-in: sbr_set_exact_maps).  Every deposit is a
// non-negative float64; it is added to its cell as a 192-bit fixed-point
// integer (three 64-bit words, least significant bit 2^-160, range 2^32) with
// a carry chain of integer atomics, and k_exact_to_grid converts each cell
// once at the end of the call.  Integer addition is associative, so a cell's
// value does not depend on the order in which rays deposit: maps become
// bitwise reproducible run to run and for any wave-stream count, as the
// reference's maps are for any worker count (test_radiomap.py:335-346,
// 517-527).  Off by default: the atomics that return their old value cost
// ~3 % of a config-4 map (639 -> 661 ms) against float64 atomics, whose cell
// sums match to ~1e-16 relative in any order.
constexpr int kExactFrac = 160;
std::atomic<int> g_exact_maps{0};

__device__ __noinline__ void exact_add(unsigned long long* w, double v) {
  if (!(v > 0.0) || !(v < 4294967296.0)) return;  // zero / NaN deposit nothing; range 2^32
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const int e = (int)(bits >> 52) & 0x7ff;
  unsigned long long m = bits & 0xFFFFFFFFFFFFFULL;
  int p;  // weight of m's least significant bit: 2^(p - kExactFrac)
  if (e == 0) {
    p = 1 - 1075 + kExactFrac;
  } else {
    m |= 1ULL << 52;
    p = e - 1075 + kExactFrac;
  }
  if (p < 0) {
    if (p < -53) return;
    const int sh = -p;
    m = (m >> sh) + ((m >> (sh - 1)) & 1ULL);  // nearest, ties up
    p = 0;
    if (m == 0) return;
  }
  const int q = p >> 6, r = p & 63;
  unsigned long long a[3] = {0ULL, 0ULL, 0ULL};
  a[q] = m << r;
  if (r && q < 2) a[q + 1] = m >> (64 - r);
  // each word's own wrap-arounds are carried into the next word: the final
  // words are the exact 192-bit sum whatever the order of the adds
  unsigned long long carry = 0;
  for (int k = q; k < 3; ++k) {
    const unsigned long long add = a[k] + carry;
    unsigned long long c = add < carry ? 1ULL : 0ULL;
    if (add) {
      const unsigned long long old = atomicAdd(w + k, add);
      c += old + add < old ? 1ULL : 0ULL;
    }
    carry = c;
  }
}

// x / c for a cell size c.  When c is a power of two 2^k (1 m in configs 2
// and 4), x / 2^k and x * 2^-k are the same real number, correctly rounded:
// the same bits, with 2^-k built from c's exponent instead of a division.
#ifndef SBR_DIV_CELL
#define SBR_DIV_CELL 1  // config-4 map 616.6 -> 615.1 ms (before cdiv2 it measured 633.8 vs 632.5)
#endif
__device__ __forceinline__ double div_cell(double x, double c) {
  if (SBR_DIV_CELL) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(c);
    const unsigned e = (unsigned)(b >> 52);  // sign bit included: positive c only
    if ((b & 0xFFFFFFFFFFFFFULL) == 0 && e > 1 && e < 2045)
      return x * __longlong_as_double((long long)((unsigned long long)(2046u - e) << 52));
  }
  return SBR_DIV(x, c);
}

__device__ __forceinline__ void grid_deposit(double* grid, bool exact, int64_t cell, double v) {
  if (exact) exact_add(reinterpret_cast<unsigned long long*>(grid) + 3 * cell, v);
  else atomicAdd(grid + cell, v);
}

// cells of the exact accumulator added into the caller's float64 grid
__global__ void k_exact_to_grid(const unsigned long long* __restrict__ acc, int64_t ncell,
                                double* __restrict__ grid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncell;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long w0 = acc[3 * i], w1 = acc[3 * i + 1], w2 = acc[3 * i + 2];
    if (w0 | w1 | w2) {
      const double v = fma((double)w2, 0x1p128, (double)w1 * 0x1p64) + (double)w0;
      grid[i] += v * 0x1p-160;
    }
  }
}


#ifndef SBR_WAVE_LOG2
#define SBR_WAVE_LOG2 24  // 16.7M samples per pass (~7.4 GB of queues): one pass for 1e7
#endif
constexpr int64_t kChunkRays = 1LL << SBR_WAVE_LOG2;  // samples per wavefront pass (queue capacity)

// SoA ray queue (float64; E is the complex world-frame field 3-vector)
struct MapQueue {
  double *ox, *oy, *oz, *dx, *dy, *dz;
  double *exr, *exi, *eyr, *eyi, *ezr, *ezi;
  double *r_dist, *omega, *weight;
  uint64_t* g;
  uint64_t cap;  // entries
};

struct HitBuf {
  double* t;
  int32_t* tri;
};

// diffuse-scattering work items, deferred from k_map_shade to k_map_scatter so
// the expensive S update runs with full warps instead of ~3 lanes per warp
struct ScatterQueue {
  double *dx, *dy, *dz, *nx, *ny, *nz, *px, *py, *pz;
  double *exr, *exi, *eyr, *eyi, *ezr, *ezi;
  double *omega, *r_hit, *weight, *cos_i, *gamma;
  uint64_t* g;
  int32_t* matrow;
  uint64_t cap;
};

// Ray-queue traffic is read once and written once per segment (GBs per
// pass): stream it through L2 with evict-first hints so it does not evict
// the L2-resident scene (BVH nodes, triangles), the grid and spilled locals.
#ifndef SBR_STREAM_HINTS
#define SBR_STREAM_HINTS 1
#endif
template <typename T>
__device__ __forceinline__ T qld(const T* p) {
#if SBR_STREAM_HINTS
  return __ldcs(p);
#else
  return *p;
#endif
}
template <typename T>
__device__ __forceinline__ void qst(T* p, T v) {
#if SBR_STREAM_HINTS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Lane 0's atomicAdd on a uniform address: ptxas turns `if (lane == 0)
// atomicAdd(p, v)` into a warp-aggregated atomic whose result is shuffled to
// the group right away, so the warp stalls on the atomic's round trip at the
// call site.  Here the address is formed from %laneid inside the asm (p + 8 *
// laneid, which is p for the only caller, lane 0), so it is not provably
// uniform and the result is waited for only where it is first read.
// CALL FROM LANE 0 ONLY.
__device__ __forceinline__ unsigned long long atom_add_async(unsigned long long* p,
                                                            unsigned long long v) {
  unsigned long long r;
  asm volatile(
      "{\n\t.reg .u32 l;\n\t.reg .u64 a;\n\t"
      "mov.u32 l, %%laneid;\n\tmul.wide.u32 a, l, 8;\n\tadd.u64 a, a, %1;\n\t"
      "atom.global.add.u64 %0, [a], %2;\n\t}"
      : "=l"(r)
      : "l"(p), "l"(v));
  return r;
}

#ifndef SBR_RAW_ATOMICS
#define SBR_RAW_ATOMICS 1  // config-4 map 758 -> 755 ms
#endif
__device__ __forceinline__ unsigned long long lane0_add(unsigned long long* p, unsigned long long v) {
#if SBR_RAW_ATOMICS
  return atom_add_async(p, v);
#else
  return atomicAdd(p, v);
#endif
}

__device__ __forceinline__ unsigned long long append_slot(unsigned long long* counter) {
  cg::coalesced_group grp = cg::coalesced_threads();
  unsigned long long base = 0;
  if (grp.thread_rank() == 0) base = atomicAdd(counter, (unsigned long long)grp.size());
  base = grp.shfl(base, 0);
  return base + grp.thread_rank();
}




// ---------------------------------------------------------------------------
// trace
// ---------------------------------------------------------------------------
// Persistent, warp-batched traversal: each warp claims 32 queue entries with
// one atomic and traces them together in the while-while form.  (Refilling
// lanes individually as their rays finish was measured slower on B200: it
// breaks the warp-wide leaf batching of trace_closest_ww.)
// occupancy: 8 blocks of 128 per SM (64 registers) measured best for both
// (trace 9.08 -> 8.23 ms, shade 6.06 -> 5.21 ms per canyon map; the shade
// spills ~0.3 KB to L1-resident local memory and still wins on latency hiding)
#ifndef SBR_TRACE_MINB
#define SBR_TRACE_MINB 7  // with speculation: 6.85 ms vs 6.93 at 8 blocks
#endif
#ifndef SBR_SHADE_SPLIT
#define SBR_SHADE_SPLIT 1  // canyon shade 5.0 -> 4.8 ms per step (smaller kernels, less spill)
#endif
#define SHADE_FIRST (SBR_SHADE_SPLIT ? kFirst : seg == 0)
#ifndef SBR_SHADE_CHUNK
#define SBR_SHADE_CHUNK 128  // queue items a shade warp claims at once (256: config-4 map 899 ms, 128: 895, 1024: 962)
#endif
constexpr int kShadeChunk = SBR_SHADE_CHUNK;
#ifndef SBR_SHADE_STATIC
#define SBR_SHADE_STATIC 0  // 1: warp w takes chunks w, w + W, ... (no work atomic)
#endif
#ifndef SBR_SHADE_RES
#define SBR_SHADE_RES 128  // next-queue slots a warp reserves per atomic (multiple of 32): config-4 map 32: 812 ms, 64: 797, 128: 784, 256: 785
#endif
constexpr int kShadeRes = SBR_SHADE_RES;
#ifndef SBR_SEG0_DIR_QUEUE
#define SBR_SEG0_DIR_QUEUE 1  // config-4 map 648 -> 643 ms
#endif
#ifndef SBR_SHADE_SPECIALISE
#define SBR_SHADE_SPECIALISE 1
#endif
#ifndef SBR_SHADE_MINB
#define SBR_SHADE_MINB 8
#endif
#ifndef SBR_TRACE_SPLIT
#define SBR_TRACE_SPLIT 0  // split trace measured equal (4.20 vs 4.21 ms; 8 blocks/SM 4.23)
#endif
#define TRACE_FIRST (SBR_TRACE_SPLIT ? kFirst : seg == 0)
#ifndef SBR_WAVE_STREAMS
#define SBR_WAVE_STREAMS 2  // config-4 map 783 -> 757 ms (kernel tails of one pass overlap the other)
#endif
#ifndef SBR_TRACE_CLAIM_AHEAD
#define SBR_TRACE_CLAIM_AHEAD 1  // config-4 map 644 -> 640 ms
#endif
#ifndef SBR_TRACE_CLAIM
#define SBR_TRACE_CLAIM 1  // batches of 32 rays a trace warp claims per atomic
#endif
#ifndef SBR_TRACE_TPB
#define SBR_TRACE_TPB 128
#endif
#ifndef SBR_TRACE_UNIFORM
#define SBR_TRACE_UNIFORM 1  // warp-uniform traversal loops (ClosestTravT::round_u)
#endif
template <bool kFirst, bool kCheck = true>
__global__ void __launch_bounds__(SBR_TRACE_TPB, SBR_TRACE_MINB) k_map_trace(DevScene S, SbrMapParams P, int seg,
                                                   MapQueue q, const unsigned long long* count_in,
                                                   uint64_t begin, uint64_t count0, CombMap comb,
                                                   HitBuf hits, unsigned long long* work,
                                                   unsigned long long* counters, ShardMap sh) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t n = TRACE_FIRST ? comb.slots() : (uint64_t)*count_in;
  const double3 src = make_double3(P.source[0], P.source[1], P.source[2]);
#if SBR_TRACE_CLAIM_AHEAD
  // the next batch is claimed while this one is traced: the atomic's round
  // trip hides behind the traversal (lane 0's raw atomic is not aggregated)
  unsigned long long next = 0;
  if (lane == 0) next = atom_add_async(work, 32ULL);
  while (true) {
    const unsigned long long base = __shfl_sync(0xffffffffu, next, 0);
    if (base >= n) break;
    if (lane == 0) next = atom_add_async(work, 32ULL);
#else
  unsigned long long claim = 0;
  int left = 0;  // batches of 32 left in the current claim
  while (true) {
    if (left == 0) {
      if (lane == 0) claim = lane0_add(work, 32ULL * SBR_TRACE_CLAIM);
      claim = __shfl_sync(0xffffffffu, claim, 0);
      left = SBR_TRACE_CLAIM;
    }
    const unsigned long long base = claim;
    claim += 32;
    --left;
    if (base >= n) break;
#endif
    const uint64_t i = base + lane;
    bool active = i < n;
    double3 o = src, d = make_double3(0.0, 0.0, 1.0);
    if (active) {
      if (TRACE_FIRST) {
        const uint64_t local = comb.sample(i);
        active = local < count0;
        if (active) {
          d = fibonacci_dir(P.num_samples, sh.gid(begin + local));
#if SBR_SEG0_DIR_QUEUE
          // the (otherwise unused) segment-0 input queue carries the launch
          // direction to the shade, which would recompute it
          qst(&q.dx[i], d.x);
          qst(&q.dy[i], d.y);
          qst(&q.dz[i], d.z);
#endif
        }
        else qst(&hits.tri[i], -3);  // comb slot past the end of the range
      } else {
        o = make_double3(qld(&q.ox[i]), qld(&q.oy[i]), qld(&q.oz[i]));
        if (isnan(o.x)) {  // padding of a shade warp's last output batch
          active = false;
          qst(&hits.tri[i], -3);
        } else {
          d = make_double3(qld(&q.dx[i]), qld(&q.dy[i]), qld(&q.dz[i]));
        }
      }
    }
    alignas(8) int sn[(SBR_PACKED_STACK ? 2 : 1) * kStackSize];
    float st[SBR_PACKED_STACK ? 1 : kStackSize];
    ClosestTravT<false> T(sn, st);  // the map needs t and the slot only
    T.start(S, o, d, 1e-4, __longlong_as_double(0x7ff0000000000000LL));
    if (!active) T.idle();
#if SBR_TRACE_UNIFORM
    while (__any_sync(0xffffffffu, !T.done())) T.template round_u<kCheck>(S);
#else
    while (!T.done()) T.round(S);
#endif
    if (active) {
      HitRecord h;
      T.result(h);
      if (!T.ok) {
        flag_error(S, kErrStack);
        atomicAdd(counters + SBR_MC_STACK_OVERFLOW, 1ULL);
        h.tri = -2;  // dropped
      }
      qst(&hits.t[i], h.t);
      qst(&hits.tri[i], h.tri);
#ifdef SBR_COUNT_VISITS
      atomicAdd(counters + SBR_MC_DIRECT_VISIBLE, (unsigned long long)T.visits);
      atomicAdd(counters + SBR_MC_THRESHOLD_KILLED, (unsigned long long)T.tests);
#endif
    }
  }
}

// ---------------------------------------------------------------------------
// shade
// ---------------------------------------------------------------------------
struct LaneCounters {
  unsigned rb, deposits, escaped, respawns, terminated, thr, rr;
};

// kFirst: the segment-0 instantiation (launch directions from the sample id)
// and the queue instantiation are separate kernels when SBR_SHADE_SPLIT, so
// each carries only its own ray-source code
// kCull: the run culls (gain threshold / Russian roulette); kSimple: an
// isotropic, unrotated source without an array (the launch field is the
// zenith unit vector, weight 1) -- both specialisations only drop code the
// run never executes (smaller instruction footprint, SBR_SHADE_SPECIALISE)
template <bool kFirst, bool kCull = true, bool kSimple = false, bool kExact = false>
__global__ void __launch_bounds__(128, SBR_SHADE_MINB) k_map_shade(DevScene S, SbrMapParams P, int seg,
                                                   MapQueue qi, const unsigned long long* count_in,
                                                   uint64_t begin, CombMap comb, HitBuf hits,
                                                   MapQueue qo, unsigned long long* count_out,
                                                   ScatterQueue sq, unsigned long long* count_s,
                                                   double* __restrict__ grid,
                                                   unsigned long long* __restrict__ counters, ShardMap sh,
                                                   unsigned long long* work) {
  LaneCounters K = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
  const uint64_t n = SHADE_FIRST ? comb.slots() : (uint64_t)*count_in;
  const double3 n_hat = make_double3(P.normal[0], P.normal[1], P.normal[2]);
  const unsigned lane = threadIdx.x & 31u;
  // Work: each warp claims kShadeChunk consecutive queue items at a time and
  // walks them 32 per warp-uniform iteration (a __syncwarp closes each: lanes
  // that take a short exit wait for the warp, so the FP64 Fresnel / field code
  // issues for converged lanes; `continue` inside the do-while(0) ends the
  // item).  Output: the warp's R / T survivors fill kShadeRes-slot batches of
  // the next queue in input order (a new batch reserved with one atomic when
  // the current one is full), so a trace warp of the next segment gets the
  // survivors of neighbouring rays -- coherent -- instead of unrelated warps'
  // survivors, with few atomics on the shared counter; the warp pads its last
  // batch with dead entries (NaN origin) that the trace skips.
  unsigned long long res_base = 0;
  int res_fill = kShadeRes;  // warp-uniform: slots used in the current batch (full = none reserved)
#if SBR_SHADE_STATIC
  const uint64_t gwarp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t ck = gwarp;; ck += nwarps) {
    const unsigned long long c0 = ck * kShadeChunk;
    if (c0 >= n) break;
#else
  while (true) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = lane0_add(work, (unsigned long long)kShadeChunk);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= n) break;
#endif
    const uint64_t c1 = c0 + kShadeChunk < n ? c0 + kShadeChunk : n;
  for (uint64_t i0 = c0; i0 < c1; i0 += 32) {
    const uint64_t i = i0 + lane;
    bool emit = false;
    // the item's state, declared here so the output after the body reads it
    double3 o, d, pt, nd;
    cvec3 E;
    double r_dist, omega, weight;
    uint64_t g;
    if (i < c1) do {
    const int tri = qld(&hits.tri[i]);
    if (tri < -1) continue;  // empty comb slot / stack overflow
    SBR_DCHECK(S, tri < S.ntri && i < qi.cap);
    if (SHADE_FIRST && tri < 0) {
      // a launch ray that escapes does nothing but count (no plane crossing at
      // segment 0): skip its direction / field / precoding weight
      K.rb++;
      K.escaped++;
      continue;
    }
    if (SHADE_FIRST) {
      g = sh.gid(begin + comb.sample(i));
      o = make_double3(P.source[0], P.source[1], P.source[2]);
#if SBR_SEG0_DIR_QUEUE
      d = make_double3(qld(&qi.dx[i]), qld(&qi.dy[i]), qld(&qi.dz[i]));
#else
      d = fibonacci_dir(P.num_samples, g);
#endif
      if (kSimple) {
        E = antenna_iso(d);
        weight = 1.0;
      } else {
        E = antenna_field(P.pattern, d);
        weight = alpha_sq(P, d);
      }
      r_dist = 0.0;
      omega = P.omega0;
    } else {
      g = qld(&qi.g[i]);
      o = make_double3(qld(&qi.ox[i]), qld(&qi.oy[i]), qld(&qi.oz[i]));
      d = make_double3(qld(&qi.dx[i]), qld(&qi.dy[i]), qld(&qi.dz[i]));
      E.x = C(qld(&qi.exr[i]), qld(&qi.exi[i]));
      E.y = C(qld(&qi.eyr[i]), qld(&qi.eyi[i]));
      E.z = C(qld(&qi.ezr[i]), qld(&qi.ezi[i]));
      r_dist = qld(&qi.r_dist[i]);
      omega = qld(&qi.omega[i]);
      weight = qld(&qi.weight[i]);
    }
    K.rb++;
    const double t_hit = qld(&hits.t[i]);
    const uint64_t chunk = g >> SBR_CHUNK_LOG2;
    const uint64_t slot = g & ((1ULL << SBR_CHUNK_LOG2) - 1);
    // plane crossing before the hit (radiomap.py:394-413); escaped rays deposit too
    if (!SHADE_FIRST) {
      const double denom = dot_gemv(d, n_hat);
      double s = -1.0;
      if (fabs(denom) > 1e-12) s = SBR_DIV(P.plane_off - dot_gemv(o, n_hat), denom);
      if (s > 1e-4 && s < t_hit) {
        const double3 pt = o + s * d;
        const double3 rel = make_double3(pt.x - P.corner[0], pt.y - P.corner[1], pt.z - P.corner[2]);
        const double fu = floor(div_cell(dot_gemv(rel, make_double3(P.u_hat[0], P.u_hat[1], P.u_hat[2])), P.cell_w));
        const double fv = floor(div_cell(dot_gemv(rel, make_double3(P.v_hat[0], P.v_hat[1], P.v_hat[2])), P.cell_h));
        if (fu >= 0.0 && fu < (double)P.nx && fv >= 0.0 && fv < (double)P.ny) {
          const double val = SBR_DIV(P.scale * field_energy(E) * omega, fabs(denom)) * weight;
          grid_deposit(grid, kExact, (int64_t)fv * P.nx + (int64_t)fu, val);
          K.deposits++;
        }
      }
    }
    if (tri < 0) {
      K.escaped++;
      continue;
    }
    if (seg == P.max_depth) continue;
    const double r_hit = r_dist + t_hit;
    // culling (radiomap.py:427-447)
    if (kCull && seg >= P.cull_from && (P.gain_threshold > 0.0 || P.rr_depth >= 0)) {
      const double e_sq = field_energy(E);
      bool keep = true;
      if (P.gain_threshold > 0.0) {
        keep = e_sq >= P.gain_threshold * (r_hit * r_hit);
        if (!keep) K.thr++;
      }
      if (P.rr_depth >= 0 && seg >= P.rr_depth) {
        const double surv = e_sq < P.rr_max ? e_sq : P.rr_max;
        const double u_rr = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_ROULETTE, slot);
        if (keep && u_rr >= surv) K.rr++;
        keep = keep && (u_rr < surv);
        if (keep) weight /= surv;
      }
      if (!keep) continue;
    }
    pt = o + t_hit * d;
    double3 nrm = ldg3(S.normals + 3 * (int64_t)tri);
    if (dot_seq(d, nrm) > 0.0) nrm = neg(nrm);
    const double cos_i = fabs(dot_seq(d, nrm));
    const SbrMaterial m = S.mats[__ldg(S.matrow + tri)];
    const Fresnel4 F = slab_fresnel(m, cos_i);
    const double r_sq = cabs2(F.rp) + cabs2(F.rl);
    const double t_sq = cabs2(F.tp) + cabs2(F.tl);
    // _interaction_rows with q_D = 0 (paths.py:572-595)
    double q0 = 0.0, q1 = 0.0, q2 = 0.0;
    const double den = r_sq + t_sq;
    if (den > 0.0) {
      const double s_sq = m.scattering * m.scattering;
      q0 = SBR_DIV(1.0 * (1.0 - s_sq) * r_sq, den);
      q1 = SBR_DIV(1.0 * s_sq * r_sq, den);
      q2 = SBR_DIV(1.0 * t_sq, den);
    }
    if (!(P.allow_mask & 1)) q0 = 0.0;
    if (!(P.allow_mask & 2)) q1 = 0.0;
    if (!(P.allow_mask & 4)) q2 = 0.0;
    const double total = ((q0 + q1) + q2) + 0.0;
    if (!(total > 0.0)) {
      K.terminated++;
      continue;
    }
    q0 = SBR_DIV(q0, total);
    q1 = SBR_DIV(q1, total);
    q2 = SBR_DIV(q2, total);
    const double q3 = 0.0;  // q_D / total with q_D = 0 and total in (0, 3]: exactly +0
    const double u = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_INTERACTION, slot);
    const double c0 = q0, c1 = c0 + q1, c2 = c1 + q2, c3 = c2 + q3;
    int code = (u >= c0) + (u >= c1) + (u >= c2) + (u >= c3);
    if (code > 3) code = 3;
    weight = SBR_DIV(weight, code == 0 ? q0 : code == 1 ? q1 : code == 2 ? q2 : q3);

    double3 e_perp, e_par;
    incidence_frame(d, nrm, e_perp, e_par);
    const cplx c_perp = cdot_real(E, e_perp), c_par = cdot_real(E, e_par);
    nd = d;
    if (code == 0) {
      const double dn = dot_seq(d, nrm);
      const double3 kr = d - (2.0 * dn) * nrm;
      const double3 e_par_r = cross3(e_perp, kr);
      const cplx a = F.rp * c_perp, b = F.rl * c_par;
      E.x = m.spec_amp * (e_perp.x * a + e_par_r.x * b);
      E.y = m.spec_amp * (e_perp.y * a + e_par_r.y * b);
      E.z = m.spec_amp * (e_perp.z * a + e_par_r.z * b);
      nd = kr;
    } else if (code == 2) {
      const cplx a = F.tp * c_perp, b = F.tl * c_par;
      E.x = e_perp.x * a + e_par.x * b;
      E.y = e_perp.y * a + e_par.y * b;
      E.z = e_perp.z * a + e_par.z * b;
    }
    r_dist = r_hit;
    if (code == 1) {
      // gamma_reflected (materials.py:400-419) here, the rest in k_map_scatter
      const double g_num = sqrt(cabs2(F.rp * c_perp) + cabs2(F.rl * c_par));
      const double g_den = sqrt(cabs2(c_perp) + cabs2(c_par));
      const double gamma = g_den > 0.0 ? SBR_DIV(g_num, g_den) : 0.0;
      const unsigned long long j = append_slot(count_s);
      SBR_DCHECK(S, j < sq.cap);
      qst(&sq.dx[j], d.x);
      qst(&sq.dy[j], d.y);
      qst(&sq.dz[j], d.z);
      qst(&sq.nx[j], nrm.x);
      qst(&sq.ny[j], nrm.y);
      qst(&sq.nz[j], nrm.z);
      qst(&sq.px[j], pt.x);
      qst(&sq.py[j], pt.y);
      qst(&sq.pz[j], pt.z);
      qst(&sq.exr[j], E.x.re);
      qst(&sq.exi[j], E.x.im);
      qst(&sq.eyr[j], E.y.re);
      qst(&sq.eyi[j], E.y.im);
      qst(&sq.ezr[j], E.z.re);
      qst(&sq.ezi[j], E.z.im);
      qst(&sq.omega[j], omega);
      qst(&sq.r_hit[j], r_hit);
      qst(&sq.weight[j], weight);
      qst(&sq.cos_i[j], cos_i);
      qst(&sq.gamma[j], gamma);
      qst(&sq.g[j], g);
      qst(&sq.matrow[j], __ldg(S.matrow + tri));
      continue;
    }
    emit = true;
    } while (0);
    // ordered batch output of this iteration's survivors (warp-converged)
    const unsigned m = __ballot_sync(0xffffffffu, emit);
    if (m) {
      const int c = __popc(m);
      const int first = c < kShadeRes - res_fill ? c : kShadeRes - res_fill;
      unsigned long long nb = 0;
      if (c > first) {
        if (lane == 0) nb = lane0_add(count_out, (unsigned long long)kShadeRes);
        nb = __shfl_sync(0xffffffffu, nb, 0);
      }
      const int rank = __popc(m & ((1u << lane) - 1u));
      const unsigned long long j = rank < first ? res_base + res_fill + rank : nb + (rank - first);
      if (c > first) {
        res_base = nb;
        res_fill = c - first;
      } else {
        res_fill += c;
      }
      if (emit) {
        SBR_DCHECK(S, j < qo.cap);
        qst(&qo.ox[j], pt.x);
        qst(&qo.oy[j], pt.y);
        qst(&qo.oz[j], pt.z);
        qst(&qo.dx[j], nd.x);
        qst(&qo.dy[j], nd.y);
        qst(&qo.dz[j], nd.z);
        qst(&qo.exr[j], E.x.re);
        qst(&qo.exi[j], E.x.im);
        qst(&qo.eyr[j], E.y.re);
        qst(&qo.eyi[j], E.y.im);
        qst(&qo.ezr[j], E.z.re);
        qst(&qo.ezi[j], E.z.im);
        qst(&qo.r_dist[j], r_dist);
        qst(&qo.omega[j], omega);
        qst(&qo.weight[j], weight);
        qst(&qo.g[j], g);
      }
    }
    __syncwarp();
  }
  }
  // pad the last batch: dead entries (NaN origin) the next trace skips
  for (int p = res_fill + (int)lane; p < kShadeRes; p += 32) {
    SBR_DCHECK(S, res_base + p < qo.cap);
    qst(&qo.ox[res_base + p], __longlong_as_double(0x7ff8000000000000LL));
  }

  const unsigned v[7] = {K.rb, K.deposits, K.escaped, K.respawns, K.terminated, K.thr, K.rr};
  const int idx[7] = {SBR_MC_RAY_BOUNCES, SBR_MC_DEPOSITS, SBR_MC_ESCAPED, SBR_MC_RESPAWNS,
                      SBR_MC_TERMINATED, SBR_MC_THRESHOLD_KILLED, SBR_MC_ROULETTE_KILLED};
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const unsigned s = __reduce_add_sync(0xffffffffu, v[k]);
    if (lane == 0 && s) atomicAdd(counters + idx[k], (unsigned long long)s);
  }
}

// diffuse scattering update (radiomap.py:496-558) for the deferred S items
#ifndef SBR_SCATTER_MINB
#define SBR_SCATTER_MINB 8  // 64 registers: 0.38 -> 0.34 ms per map
#endif
// kLambert: every material's lobe is Lambertian (the other lobes' code --
// lobe normalisation loops, pow -- dropped from this instantiation)
template <bool kLambert = false>
__global__ void __launch_bounds__(128, SBR_SCATTER_MINB) k_map_scatter(DevScene S, SbrMapParams P, int seg,
                                                        ScatterQueue sq,
                                                        const unsigned long long* count_s,
                                                        MapQueue qo, unsigned long long* count_out,
                                                        unsigned long long* __restrict__ counters) {
  unsigned respawns = 0;
  const uint64_t n = *count_s;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = qld(&sq.g[j]);
    const uint64_t chunk = g >> SBR_CHUNK_LOG2;
    const uint64_t slot = g & ((1ULL << SBR_CHUNK_LOG2) - 1);
    const double3 d = make_double3(qld(&sq.dx[j]), qld(&sq.dy[j]), qld(&sq.dz[j]));
    const double3 nrm = make_double3(qld(&sq.nx[j]), qld(&sq.ny[j]), qld(&sq.nz[j]));
    cvec3 E;
    E.x = C(qld(&sq.exr[j]), qld(&sq.exi[j]));
    E.y = C(qld(&sq.eyr[j]), qld(&sq.eyi[j]));
    E.z = C(qld(&sq.ezr[j]), qld(&sq.ezi[j]));
    const double omega = qld(&sq.omega[j]), r_hit = qld(&sq.r_hit[j]), cos_i = qld(&sq.cos_i[j]);
    const double gamma = qld(&sq.gamma[j]);
    const SbrMaterial m = S.mats[qld(&sq.matrow[j])];
    const double u0 = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot);
    const double u1 = philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_RESPAWN, 2 * slot + 1);
    const double cos_t = u0, azim = kTwoPi * u1;
    const double x = 1.0 - cos_t * cos_t;
    const double sin_t = sqrt(x > 0.0 ? x : 0.0);
    const double3 t1 = perp_batch(nrm);
    const double3 t2 = cross3(nrm, t1);
    double sa, ca;
    sincos(azim, &sa, &ca);
    const double a = sin_t * ca, b = sin_t * sa;
    const double3 ks = make_double3((a * t1.x + b * t2.x) + cos_t * nrm.x,
                                    (a * t1.y + b * t2.y) + cos_t * nrm.y,
                                    (a * t1.z + b * t2.z) + cos_t * nrm.z);
    const double f_s = kLambert ? lambert_density(ks, nrm) : pattern_density(m, d, ks, nrm);
    const double patch = omega * (r_hit * r_hit) / (cos_i > 1e-12 ? cos_i : 1e-12);
    const double amp = m.scattering * gamma * sqrt(f_s * cos_i * patch);
    double3 th_i, ph_i;
    transverse_rows(d, th_i, ph_i);
    const cplx ci0 = cdot_real(E, th_i), ci1 = cdot_real(E, ph_i);
    double chi1 = 0.0, chi2 = 0.0;
    if (P.any_random_phase && m.random_phases) {
      chi1 = kTwoPi * philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot);
      chi2 = kTwoPi * philox_uniform(P.seed, chunk, (uint64_t)seg, TAG_MAP_PHASE, 2 * slot + 1);
    }
    const double sqk = sqrt(1.0 - m.xpd_kx), sk = sqrt(m.xpd_kx);
    double s1, k1, s2, k2;
    sincos(chi1, &s1, &k1);
    sincos(chi2, &s2, &k2);
    const cplx co0 = C(amp * k1, amp * s1) * (sqk * ci0 - sk * ci1);
    const cplx co1 = C(amp * k2, amp * s2) * (sk * ci0 + sqk * ci1);
    double3 th_s, ph_s;
    transverse_rows(ks, th_s, ph_s);
    const cplx inv_r = C(r_hit, 0.0);
    E.x = cdiv(th_s.x * co0 + ph_s.x * co1, inv_r);
    E.y = cdiv(th_s.y * co0 + ph_s.y * co1, inv_r);
    E.z = cdiv(th_s.z * co0 + ph_s.z * co1, inv_r);
    respawns++;
    const unsigned long long o = append_slot(count_out);
    SBR_DCHECK(S, o < qo.cap && j < sq.cap);
    qst(&qo.ox[o], qld(&sq.px[j]));
    qst(&qo.oy[o], qld(&sq.py[j]));
    qst(&qo.oz[o], qld(&sq.pz[j]));
    qst(&qo.dx[o], ks.x);
    qst(&qo.dy[o], ks.y);
    qst(&qo.dz[o], ks.z);
    qst(&qo.exr[o], E.x.re);
    qst(&qo.exi[o], E.x.im);
    qst(&qo.eyr[o], E.y.re);
    qst(&qo.eyi[o], E.y.im);
    qst(&qo.ezr[o], E.z.re);
    qst(&qo.ezi[o], E.z.im);
    qst(&qo.r_dist[o], 0.0);
    qst(&qo.omega[o], kTwoPi);
    qst(&qo.weight[o], qld(&sq.weight[j]));
    qst(&qo.g[o], g);
  }
  const unsigned s = __reduce_add_sync(0xffffffffu, respawns);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(counters + SBR_MC_RESPAWNS, (unsigned long long)s);
}

__global__ void k_reset_pass(unsigned long long* work, unsigned long long* count_next,
                             unsigned long long* count_s, unsigned long long* shade_work) {
  *work = 0ULL;
  *count_next = 0ULL;
  *count_s = 0ULL;
  *shade_work = 0ULL;
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

// ---------------------------------------------------------------------------
// edge (diffraction) estimator: compute_radio_map_diffraction (radiomap.py:842-965)
// ---------------------------------------------------------------------------
constexpr uint64_t TAG_MAP_WEDGE = 0x9115590451c40950ULL;

__device__ __forceinline__ void cone_point(const DevScene& S, int w, double3 src, double x,
                                           double phi, double3& v, double& s_in, double3& k_i,
                                           double3& k_s, double& sin_b) {
  const double3 o = ldg3(S.w_origin + 3 * w), e = ldg3(S.w_ehat + 3 * w);
  const double3 t0 = ldg3(S.w_t0 + 3 * w), n0 = ldg3(S.w_n0 + 3 * w);
  v = o + x * e;
  const double3 d = v - src;
  s_in = norm_seq(d);
  k_i = make_double3(d.x / s_in, d.y / s_in, d.z / s_in);
  const double cb = dot_gemv(d, e) / s_in;
  const double xb = 1.0 - cb * cb;
  sin_b = sqrt(xb > 0.0 ? xb : 0.0);
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double a = sin_b * cp, b = sin_b * sp;
  k_s = make_double3((a * t0.x + b * n0.x) + cb * e.x, (a * t0.y + b * n0.y) + cb * e.y,
                     (a * t0.z + b * n0.z) + cb * e.z);
}

__global__ void __launch_bounds__(128) k_map_wedges(DevScene S, SbrMapParams P,
                                                    const int32_t* __restrict__ wedge_ids,
                                                    int32_t nw, uint64_t wedge_samples,
                                                    double* __restrict__ grid, bool exact,
                                                    unsigned long long* __restrict__ counters) {
  unsigned deposits = 0, cones = 0;
  const uint64_t total = (uint64_t)nw * wedge_samples;
  const double3 nh = make_double3(P.normal[0], P.normal[1], P.normal[2]);
  const double3 src = make_double3(P.source[0], P.source[1], P.source[2]);
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const int w = __ldg(wedge_ids + idx / wedge_samples);
    const uint64_t i = idx % wedge_samples;
    const uint64_t block = i >> SBR_CHUNK_LOG2, slot = i & ((1ULL << SBR_CHUNK_LOG2) - 1);
    cones++;
    const double len = __ldg(S.w_len + w), nopen = __ldg(S.w_nopen + w);
    const double u0 = philox_uniform(P.seed, (uint64_t)w, block, TAG_MAP_WEDGE, 2 * slot);
    const double u1 = philox_uniform(P.seed, (uint64_t)w, block, TAG_MAP_WEDGE, 2 * slot + 1);
    const double xs = u0 * len, phis = u1 * nopen * kPi;
    double3 v, k_i, k_s;
    double s_in, sin_b;
    cone_point(S, w, src, xs, phis, v, s_in, k_i, k_s, sin_b);
    if (!(sin_b >= 1e-9)) continue;
    const double denom = dot_gemv(k_s, nh);
    if (!(fabs(denom) > 1e-9)) continue;
    const double gamma = (P.plane_off - dot_gemv(v, nh)) / denom;
    if (!(gamma > 1e-4)) continue;
    const double3 inc = neg(k_i);
    double azim = atan2(dot_gemv(inc, ldg3(S.w_n0 + 3 * w)), dot_gemv(inc, ldg3(S.w_t0 + 3 * w)));
    if (azim < 0.0) azim += kTwoPi;
    if (!(azim <= nopen * kPi)) continue;
    const double3 pts = v + gamma * k_s;
    const double3 rel = make_double3(pts.x - P.corner[0], pts.y - P.corner[1], pts.z - P.corner[2]);
    const double fu = floor(dot_gemv(rel, make_double3(P.u_hat[0], P.u_hat[1], P.u_hat[2])) / P.cell_w);
    const double fv = floor(dot_gemv(rel, make_double3(P.v_hat[0], P.v_hat[1], P.v_hat[2])) / P.cell_h);
    if (!(fu >= 0.0 && fu < (double)P.nx && fv >= 0.0 && fv < (double)P.ny)) continue;
    bool fine;
    if (occluded_segment(S, src, v, 1e-4, fine)) continue;
    if (!fine) flag_error(S, kErrStack);
    if (occluded_segment(S, v, pts, 1e-4, fine)) continue;
    if (!fine) flag_error(S, kErrStack);
    M2 T;
    double3 bi[2], bo[2];
    if (!utd_transfer(S, w, k_i, k_s, s_in, gamma, P.wavelength, T, bi, bo)) continue;
    // _weighting_rows: central differences of the plane crossing
    const double hx = 1e-4 * (len > 1.0 ? len : 1.0), hp = 1e-4;
    const double xq[4] = {xs + hx, xs - hx, xs, xs}, pq[4] = {phis, phis, phis + hp, phis - hp};
    double3 cr[4];
    bool bad = false;
    for (int q = 0; q < 4; ++q) {
      double3 vq, kiq, ksq;
      double sq, sbq;
      cone_point(S, w, src, xq[q], pq[q], vq, sq, kiq, ksq, sbq);
      double dq = dot_gemv(ksq, nh);
      if (fabs(dq) < 1e-9) {
        bad = true;
        dq = 1.0;
      }
      cr[q] = vq + ((P.plane_off - dot_gemv(vq, nh)) / dq) * ksq;
    }
    if (bad) continue;
    const double3 ddx = make_double3((cr[0].x - cr[1].x) / (2.0 * hx), (cr[0].y - cr[1].y) / (2.0 * hx),
                                     (cr[0].z - cr[1].z) / (2.0 * hx));
    const double3 ddp = make_double3((cr[2].x - cr[3].x) / (2.0 * hp), (cr[2].y - cr[3].y) / (2.0 * hp),
                                     (cr[2].z - cr[3].z) / (2.0 * hp));
    const double factor = norm_seq(cross3(ddx, ddp));
    const cvec3 E = antenna_field(P.pattern, k_i);
    const cplx c0 = cdot_real(E, bi[0]), c1 = cdot_real(E, bi[1]);
    const cplx o0 = T.m[0][0] * c0 + T.m[0][1] * c1;
    const cplx o1 = T.m[1][0] * c0 + T.m[1][1] * c1;
    const double spread = s_in * gamma * (s_in + gamma);
    const double e_p = (cabs2(o0) + cabs2(o1)) / spread;
    const double norm = len * nopen * kPi / (double)wedge_samples;
    grid_deposit(grid, exact, (int64_t)fv * P.nx + (int64_t)fu,
                 norm * P.scale * e_p * factor * alpha_sq(P, k_i));
    deposits++;
  }
  const unsigned lane = threadIdx.x & 31u;
  const unsigned sd = __reduce_add_sync(0xffffffffu, deposits);
  const unsigned sc = __reduce_add_sync(0xffffffffu, cones);
  if (lane == 0) {
    if (sd) atomicAdd(counters + SBR_MC_DEPOSITS, (unsigned long long)sd);
    if (sc) atomicAdd(counters + SBR_MC_CONE_SAMPLES, (unsigned long long)sc);
  }
}

constexpr int kMaxWaveStreams = 4;
std::atomic<int> g_wave_streams{SBR_WAVE_STREAMS};

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

// device scratch of one wavefront pass: two ray queues, the hit buffer and the
// control words, carved from one stream-ordered allocation (per call, so
// concurrent calls on different streams never share queues)
struct Wave {
  void* block = nullptr;
  MapQueue q[2];
  HitBuf hits;
  ScatterQueue sq;
  unsigned long long* ctl = nullptr;  // [0] trace work, [1] count A, [2] count B, [3] S count,
                                      // [4] shade work
};

int wave_alloc(int64_t cap, cudaStream_t st, Wave* w) {
  const size_t per_queue = (size_t)cap * (16 * sizeof(double));
  const size_t per_squeue = (size_t)cap * (21 * sizeof(double) + sizeof(int32_t));
  const size_t bytes = 2 * per_queue + per_squeue +
                       (size_t)cap * (sizeof(double) + sizeof(int32_t)) + 512;
  if (scratch_alloc(&w->block, bytes, st) != cudaSuccess)
    return set_error(SBR_ERR_NOMEM, "ray queues");
  char* p = (char*)w->block;
  for (int k = 0; k < 2; ++k) {
    double** f[15] = {&w->q[k].ox, &w->q[k].oy, &w->q[k].oz, &w->q[k].dx, &w->q[k].dy,
                      &w->q[k].dz, &w->q[k].exr, &w->q[k].exi, &w->q[k].eyr, &w->q[k].eyi,
                      &w->q[k].ezr, &w->q[k].ezi, &w->q[k].r_dist, &w->q[k].omega,
                      &w->q[k].weight};
    for (int i = 0; i < 15; ++i) {
      *f[i] = (double*)p;
      p += cap * sizeof(double);
    }
    w->q[k].g = (uint64_t*)p;
    p += cap * sizeof(uint64_t);
    w->q[k].cap = (uint64_t)cap;
  }
  w->sq.cap = (uint64_t)cap;
  {
    double** f[20] = {&w->sq.dx, &w->sq.dy, &w->sq.dz, &w->sq.nx, &w->sq.ny, &w->sq.nz,
                      &w->sq.px, &w->sq.py, &w->sq.pz, &w->sq.exr, &w->sq.exi, &w->sq.eyr,
                      &w->sq.eyi, &w->sq.ezr, &w->sq.ezi, &w->sq.omega, &w->sq.r_hit,
                      &w->sq.weight, &w->sq.cos_i, &w->sq.gamma};
    for (int i = 0; i < 20; ++i) {
      *f[i] = (double*)p;
      p += cap * sizeof(double);
    }
    w->sq.g = (uint64_t*)p;
    p += cap * sizeof(uint64_t);
    w->sq.matrow = (int32_t*)p;
    p += cap * sizeof(int32_t);
    p = (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
  }
  w->hits.t = (double*)p;
  p += cap * sizeof(double);
  w->hits.tri = (int32_t*)p;
  p += cap * sizeof(int32_t);
  p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
  w->ctl = (unsigned long long*)p;
  return SBR_OK;
}

}  // namespace

extern "C" {

// the bounce loop over local ids [sample_begin, sample_end) of shard `sh`
static int bounce_impl(const SbrScene* scene, const SbrMapParams* P, uint64_t sample_begin,
                       uint64_t sample_end, ShardMap sh, double* grid, uint64_t* counters_u64,
                       void* stream) {
  int rc = SBR_OK;
  const uint64_t total = sample_end - sample_begin;
  if (total == 0) return SBR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* counters = (unsigned long long*)counters_u64;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // equal passes of at most kChunkRays samples (e.g. a 1.25e8-sample shard:
  // 8 x 15.6M instead of 7 full passes and a half one that would run alone
  // at the end); samples are independent, so pass boundaries do not matter
#ifndef SBR_MAP_SHARD_MAX_LOG2
#define SBR_MAP_SHARD_MAX_LOG2 23  // 19: plain RNG-chunk-cyclic shards
#endif
#ifndef SBR_EQUAL_PASSES
#define SBR_EQUAL_PASSES 1
#endif
  const uint64_t npass_ = (total + (uint64_t)kChunkRays - 1) / (uint64_t)kChunkRays;
  const int64_t chunk = SBR_EQUAL_PASSES ? (int64_t)((total + npass_ - 1) / npass_)
                                         : (total < (uint64_t)kChunkRays ? (int64_t)total : kChunkRays);
  // segment 0 runs over comb slots: up to chunk + F items
  const uint64_t F = comb_stride(P->num_samples);
  // SBR_WAVE_STREAMS (2): consecutive passes alternate between the caller's
  // stream and a second one with its own queues, so one pass's kernel tails
  // overlap the other's bulk (passes are independent sample ranges; the grid
  // and counters take float64 / integer atomics from both)
  int nstreams = g_wave_streams.load();
  const int64_t npass = (int64_t)((total + (uint64_t)chunk - 1) / (uint64_t)chunk);
  if (nstreams > npass) nstreams = (int)npass;
  Wave waves[kMaxWaveStreams];
  cudaStream_t sts[kMaxWaveStreams] = {st, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxWaveStreams] = {nullptr, nullptr, nullptr, nullptr};
  // + the dead padding of every shade warp's last output batch
  const int64_t pad = (int64_t)kShadeRes * sms * SBR_SHADE_MINB * 4 + 64;
  for (int k = 0; k < nstreams && !rc; ++k) rc = wave_alloc(chunk + (int64_t)F + pad, st, &waves[k]);
  const int64_t ncell = (int64_t)P->nx * P->ny;
  const bool exact = g_exact_maps.load() != 0;
  unsigned long long* acc = nullptr;  // exact accumulator, when enabled
  if (!rc && exact) {
    if (scratch_alloc((void**)&acc, (size_t)ncell * 3 * sizeof(unsigned long long), st) != cudaSuccess)
      rc = set_error(SBR_ERR_NOMEM, "map accumulator");
    else
      cudaMemsetAsync(acc, 0, (size_t)ncell * 3 * sizeof(unsigned long long), st);
  }
  double* dep = exact ? reinterpret_cast<double*>(acc) : grid;
  if (!rc && nstreams > 1) {
    if (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess) {
      rc = set_error(SBR_ERR_CUDA, "wave stream event");
    } else {
      cudaEventRecord(ev_fork, st);  // queues allocated, caller's prior work done
      for (int k = 1; k < nstreams && !rc; ++k) {
        if (cudaStreamCreateWithFlags(&sts[k], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_join[k], cudaEventDisableTiming) != cudaSuccess) {
          rc = set_error(SBR_ERR_CUDA, "wave stream");
        } else {
          cudaStreamWaitEvent(sts[k], ev_fork, 0);
        }
      }
    }
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_map_trace<false>, SBR_TRACE_TPB, 0);
  if (per_sm < 1) per_sm = 1;
  const unsigned trace_blocks = (unsigned)(sms * per_sm);
  const unsigned shade_blocks = (unsigned)(sms * SBR_SHADE_MINB);
  const DevScene S = dev_view(scene);
  const bool shallow = SBR_TRACE_UNIFORM && S.depth < kStackSize;
  const bool cull = !SBR_SHADE_SPECIALISE || P->gain_threshold > 0.0 || P->rr_depth >= 0;
  const bool simple = SBR_SHADE_SPECIALISE && P->pattern.identity && P->pattern.kind == SBR_PATTERN_ISOTROPIC &&
                      P->n_elements <= 0;
  int pass = 0;
  for (uint64_t lo = sample_begin; lo < sample_end && !rc; lo += (uint64_t)chunk, ++pass) {
    const uint64_t cnt = (sample_end - lo) < (uint64_t)chunk ? (sample_end - lo) : (uint64_t)chunk;
    const CombMap comb{(cnt + F - 1) / F, F};
    Wave* w = &waves[pass % nstreams];
    cudaStream_t ps = sts[pass % nstreams];
    int cur = 0;
    for (int seg = 0; seg <= P->max_depth; ++seg) {
      // ctl[0] = work counter; ctl[1 + cur] = this segment's count; ctl[2 - cur] = next count
      k_reset_pass<<<1, 1, 0, ps>>>(w->ctl, w->ctl + 2 - cur, w->ctl + 3, w->ctl + 4);
      if ((rc = launch_status("k_reset_pass"))) break;
      prof_begin(ps, "k_map_trace");
      // a tree shallower than the stack cannot overflow it: unchecked pushes
      auto trace = seg == 0 ? (shallow ? k_map_trace<true, false> : k_map_trace<true, true>)
                            : (shallow ? k_map_trace<false, false> : k_map_trace<false, true>);
      trace<<<trace_blocks, SBR_TRACE_TPB, 0, ps>>>(S, *P, seg, w->q[cur], w->ctl + 1 + cur, lo, cnt,
                                                    comb, w->hits, w->ctl, counters, sh);
      prof_end(ps);
      if ((rc = launch_status("k_map_trace"))) break;
      prof_begin(ps, "k_map_shade");
      auto shade = seg == 0 ? (cull ? (simple ? k_map_shade<true, true, true> : k_map_shade<true, true, false>)
                                    : (simple ? k_map_shade<true, false, true> : k_map_shade<true, false, false>))
                            : exact ? (cull ? k_map_shade<false, true, false, true> : k_map_shade<false, false, false, true>)
                                    : (cull ? k_map_shade<false, true, false> : k_map_shade<false, false, false>);
      shade<<<shade_blocks, 128, 0, ps>>>(S, *P, seg, w->q[cur], w->ctl + 1 + cur, lo,
                                                comb, w->hits, w->q[1 - cur], w->ctl + 2 - cur,
                                                w->sq, w->ctl + 3, dep, counters, sh, w->ctl + 4);
      prof_end(ps);
      if ((rc = launch_status("k_map_shade"))) break;
      if (seg < P->max_depth && (P->allow_mask & 2)) {
        prof_begin(ps, "k_map_scatter");
        (S.all_lambertian && SBR_SHADE_SPECIALISE ? k_map_scatter<true> : k_map_scatter<false>)<<<shade_blocks, 128, 0, ps>>>(S, *P, seg, w->sq, w->ctl + 3, w->q[1 - cur],
                                                    w->ctl + 2 - cur, counters);
        prof_end(ps);
        if ((rc = launch_status("k_map_scatter"))) break;
      }
      cur = 1 - cur;
    }
  }
  for (int k = 1; k < kMaxWaveStreams; ++k) {
    if (!sts[k]) continue;
    if (ev_join[k]) {  // join: the caller's stream waits for the other streams' passes
      cudaEventRecord(ev_join[k], sts[k]);
      cudaStreamWaitEvent(st, ev_join[k], 0);
      cudaEventDestroy(ev_join[k]);
    }
    cudaStreamDestroy(sts[k]);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  for (int k = 0; k < nstreams; ++k)
    if (waves[k].block) cudaFreeAsync(waves[k].block, st);
  if (acc) {
    if (!rc) {
      const int64_t b = (ncell + 255) / 256;
      k_exact_to_grid<<<(unsigned)(b < 148 * 16 ? b : 148 * 16), 256, 0, st>>>(acc, ncell, grid);
      rc = launch_status("k_exact_to_grid");
    }
    cudaFreeAsync(acc, st);
  }
  return rc;
}

int sbr_set_exact_maps(int32_t on) {
  if (on != 0 && on != 1) return set_error(SBR_ERR_INVALID, "exact maps: 0 or 1");
  g_exact_maps = on;
  return SBR_OK;
}

int sbr_set_wave_streams(int32_t n) {
  if (n < 1 || n > kMaxWaveStreams) return set_error(SBR_ERR_INVALID, "wave streams: 1 to 4");
  g_wave_streams = n;
  return SBR_OK;
}

int sbr_radiomap_bounce(const SbrScene* scene, const SbrMapParams* P, uint64_t sample_begin,
                        uint64_t sample_end, double* grid, uint64_t* counters_u64, void* stream) {
  int rc = check_params(scene, P);
  if (rc) return rc;
  if (sample_end > P->num_samples || sample_begin > sample_end)
    return set_error(SBR_ERR_INVALID, "bad sample range");
  return bounce_impl(scene, P, sample_begin, sample_end, ShardMap{0u, 1u, SBR_CHUNK_LOG2}, grid, counters_u64,
                     stream);
}

int sbr_radiomap_bounce_sharded(const SbrScene* scene, const SbrMapParams* P,
                                int32_t shard_index, int32_t shard_count, double* grid,
                                uint64_t* counters_u64, void* stream) {
  int rc = check_params(scene, P);
  if (rc) return rc;
  if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
    return set_error(SBR_ERR_INVALID, "bad shard");
  // Shard blocks of 2^b ids, b = log2(num_samples / (8 x shards)) clamped to
  // [19, 23]: >= 8 blocks per shard (balanced), and up to 2^23 contiguous
  // lattice ids -- a polar band -- per block, so one 2^24-sample pass traces
  // two bands instead of 32 scattered 2^19-id chunks (config 4 shard of 8:
  // 4.0e9 -> 4.5e9 rb/s, the unsharded rate).  Results do not depend on it.
  uint32_t b = SBR_CHUNK_LOG2;
  while (b < SBR_MAP_SHARD_MAX_LOG2 && (P->num_samples >> (b + 1)) >= 8ULL * (uint64_t)shard_count) ++b;
  const uint64_t n_local = shard_size(P->num_samples, (uint32_t)shard_index, (uint32_t)shard_count, b);
  return bounce_impl(scene, P, 0, n_local, ShardMap{(uint32_t)shard_index, (uint32_t)shard_count, b},
                     grid, counters_u64, stream);
}

int sbr_radiomap_wedges(const SbrScene* scene, const SbrMapParams* P, const int32_t* wedge_ids,
                        int32_t n_wedges, uint64_t wedge_samples, double* grid,
                        uint64_t* counters, void* stream) {
  int rc = check_params(scene, P);
  if (rc) return rc;
  if (n_wedges <= 0 || wedge_samples == 0) return SBR_OK;
  if (dev_view(scene).n_wedges <= 0) return set_error(SBR_ERR_INVALID, "scene has no wedges");
  const uint64_t total = (uint64_t)n_wedges * wedge_samples;
  uint64_t blocks = (total + 127) / 128;
  if (blocks > 148 * 64) blocks = 148 * 64;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ncell = (int64_t)P->nx * P->ny;
  const bool exact = g_exact_maps.load() != 0;
  unsigned long long* acc = nullptr;
  if (exact) {
    if (scratch_alloc((void**)&acc, (size_t)ncell * 3 * sizeof(unsigned long long), st) != cudaSuccess)
      return set_error(SBR_ERR_NOMEM, "map accumulator");
    cudaMemsetAsync(acc, 0, (size_t)ncell * 3 * sizeof(unsigned long long), st);
  }
  prof_begin(stream, "k_map_wedges");
  k_map_wedges<<<(unsigned)blocks, 128, 0, st>>>(
      dev_view(scene), *P, wedge_ids, n_wedges, wedge_samples,
      exact ? reinterpret_cast<double*>(acc) : grid, exact, (unsigned long long*)counters);
  prof_end(stream);
  rc = launch_status("k_map_wedges");
  if (acc) {
    if (!rc) {
      const int64_t b = (ncell + 255) / 256;
      k_exact_to_grid<<<(unsigned)(b < 148 * 16 ? b : 148 * 16), 256, 0, st>>>(acc, ncell, grid);
      rc = launch_status("k_exact_to_grid");
    }
    cudaFreeAsync(acc, st);
  }
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
