// sbr_scene.cu -- device scene: LBVH build in HBM plus the scene C ABI.
//
// Replaces Accel.__init__ / _build_bvh (emtrace geometry.py:134-166, 244-349).
// Build pipeline (all on the GPU, stream-ordered):
//   1. per-triangle float64 AABB -> centroid; centroid bounds (atomics)
//   2. 63-bit Morton keys (21 bits per axis)              [kernel]
//   3. radix sort of (key, triangle) pairs                 [cub::DeviceRadixSort]
//   4. Karras 2012 binary radix tree over the sorted keys  [kernel]
//   5. bottom-up refit of conservative fp32 boxes          [kernel, atomics]
//   6. collapse subtrees of <= SBR_LEAF_MAX (2) triangles into leaves and
//      emit 64-B BVH2 nodes (both child boxes per node)    [scan + kernel]
// Triangles are stored in Morton (slot) order as float64 corners so the
// watertight test reproduces the reference's arithmetic exactly.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sbr_common.cuh"

namespace sbr {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

// The library's stream-ordered scratch (ray queues, sort buffers, CFR
// factors) comes from a private memory pool per device.  Freed blocks stay
// mapped between calls up to kScratchKeep bytes (a config-4 wavefront pass
// needs ~7.4 GB; remapping it at every synchronisation costs ~ms), anything
// above is returned to the driver at the next synchronisation, and
// sbr_release_scratch() trims the pool to zero.  The device's default pool
// (used by other libraries in the process) is never touched.
constexpr uint64_t kScratchKeep = 16ULL << 30;
constexpr int kMaxDevices = 64;
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[kMaxDevices] = {};

static cudaError_t scratch_pool(int device, cudaMemPool_t* out) {
  if (device < 0 || device >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool;
    const cudaError_t e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t keep = kScratchKeep;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pools[device] = pool;
  }
  *out = g_pools[device];
  return cudaSuccess;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  cudaMemPool_t pool;
  if (e == cudaSuccess) e = scratch_pool(device, &pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, st);
}

// cudaSetDevice for the duration of a scope, restoring the caller's device
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---- optional per-kernel CUDA-event timing (bench.py roofline evidence) ----
struct Span {
  std::string name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static std::atomic<bool> g_prof_on{false};
static std::vector<Span> g_spans;
static std::map<std::string, std::pair<double, uint64_t>> g_prof_acc;

void prof_begin(void* stream, const char* name) {
  if (!g_prof_on) return;
  Span s;
  s.name = name;
  cudaEventCreate(&s.a);
  cudaEventCreate(&s.b);
  cudaEventRecord(s.a, (cudaStream_t)stream);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_spans.push_back(s);
}

void prof_end(void* stream) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_spans.empty()) cudaEventRecord(g_spans.back().b, (cudaStream_t)stream);
}

static void prof_drain() {
  for (Span& s : g_spans) {
    cudaEventSynchronize(s.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s.a, s.b);
    auto& acc = g_prof_acc[s.name];
    acc.first += ms;
    acc.second += 1;
    cudaEventDestroy(s.a);
    cudaEventDestroy(s.b);
  }
  g_spans.clear();
}

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define SBR_CUDA(call)                                                             \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return ::sbr::set_error(SBR_ERR_CUDA, std::string(#call) + ": " +            \
                                                cudaGetErrorString(_e));           \
  } while (0)

}  // namespace sbr

struct SbrScene {
  int device = 0;
  int64_t ntri = 0;
  int32_t nnodes = 0;
  int32_t depth = 0;  // levels of the tree (a traversal stack needs < depth entries)
  sbr::BvhNode* nodes = nullptr;
  sbr::TriSlot* tris = nullptr;
  int32_t* tie_rank = nullptr;
  double* normals = nullptr;
  int32_t* matrow = nullptr;
  uint64_t* hash_r = nullptr;
  uint64_t* hash_f = nullptr;
  SbrMaterial* mats = nullptr;
  int32_t nmat = 0;
  int32_t all_lambertian = 0;  // every material's scattering lobe is Lambertian
  unsigned int* error_word = nullptr;
  float pad_base = 0.f;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  std::vector<int64_t> perm;
  // wedge tables (one allocation)
  void* wedge_block = nullptr;
  int64_t n_wedges = 0;
  const double *w_origin = nullptr, *w_ehat = nullptr, *w_t0 = nullptr, *w_n0 = nullptr,
               *w_nn = nullptr, *w_len = nullptr, *w_nopen = nullptr;
  const uint64_t *w_hr = nullptr, *w_hf = nullptr;
  const int32_t *w_mat0 = nullptr, *w_matn = nullptr, *slot_woff = nullptr, *slot_wids = nullptr;
};

namespace sbr {

DevScene dev_view(const SbrScene* s) {
  DevScene d;
  d.nodes = s->nodes;
  d.tris = s->tris;
  d.tie_rank = s->tie_rank;
  d.normals = s->normals;
  d.matrow = s->matrow;
  d.hash_r = s->hash_r;
  d.hash_f = s->hash_f;
  d.mats = s->mats;
  d.error_word = s->error_word;
  d.ntri = s->ntri;
  d.nnodes = s->nnodes;
  d.depth = s->depth;
  d.nmat = s->nmat;
  d.all_lambertian = s->all_lambertian;
  d.pad_base = s->pad_base;
  for (int k = 0; k < 3; ++k) {
    d.bounds_lo[k] = s->lo[k];
    d.bounds_hi[k] = s->hi[k];
  }
  d.n_wedges = s->n_wedges;
  d.w_origin = s->w_origin;
  d.w_ehat = s->w_ehat;
  d.w_t0 = s->w_t0;
  d.w_n0 = s->w_n0;
  d.w_nn = s->w_nn;
  d.w_len = s->w_len;
  d.w_nopen = s->w_nopen;
  d.w_hr = s->w_hr;
  d.w_hf = s->w_hf;
  d.w_mat0 = s->w_mat0;
  d.w_matn = s->w_matn;
  d.slot_woff = s->slot_woff;
  d.slot_wids = s->slot_wids;
  return d;
}

// ---------------------------------------------------------------------------
// build kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned int f2ord(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_centroids(const double* __restrict__ v0, const double* __restrict__ v1,
                            const double* __restrict__ v2, int64_t n, float3* cen,
                            unsigned int* cbounds /* 6: min xyz, max xyz (ordered) */) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float c[3] = {0.f, 0.f, 0.f};
  const bool live = i < n;
  if (live) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double a = v0[3 * i + k], b = v1[3 * i + k], d = v2[3 * i + k];
      const double lo = fmin(fmin(a, b), d), hi = fmax(fmax(a, b), d);
      c[k] = (float)((lo + hi) * 0.5);
    }
    cen[i] = make_float3(c[0], c[1], c[2]);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    unsigned int mn = live ? f2ord(c[k]) : 0xffffffffu;
    unsigned int mx = live ? f2ord(c[k]) : 0u;
    for (int off = 16; off; off >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(cbounds + k, mn);
      atomicMax(cbounds + 3 + k, mx);
    }
  }
}

__device__ __forceinline__ uint64_t spread21(uint64_t x) {
  x &= 0x1fffffULL;
  x = (x | (x << 32)) & 0x1f00000000ffffULL;
  x = (x | (x << 16)) & 0x1f0000ff0000ffULL;
  x = (x | (x << 8)) & 0x100f00f00f00f00fULL;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ULL;
  x = (x | (x << 2)) & 0x1249249249249249ULL;
  return x;
}

__global__ void k_morton(const float3* __restrict__ cen, int64_t n,
                         const unsigned int* __restrict__ cbounds, uint64_t* keys,
                         int32_t* ids) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float3 c = cen[i];
  const float lo[3] = {ord2f(cbounds[0]), ord2f(cbounds[1]), ord2f(cbounds[2])};
  const float hi[3] = {ord2f(cbounds[3]), ord2f(cbounds[4]), ord2f(cbounds[5])};
  const float v[3] = {c.x, c.y, c.z};
  uint64_t q[3];
  // one cubic grid over the centroid bounds (not each axis stretched to 21
  // bits): the curve then follows true distances in flat scenes (city
  // 1000 x 1000 x 60 m).  PLOC SAH cost city 74.6 -> 62.4 (reference binned
  // SAH: 63.3), canyon 40.8 -> 38.6; canyon map +8 %, config-3 visibility -14 %.
  const float cube = fmaxf(fmaxf(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float ext = cube;
    float f = ext > 0.f ? (v[k] - lo[k]) / ext : 0.5f;
    f = fminf(fmaxf(f, 0.f), 1.f);
    q[k] = (uint64_t)fminf(f * 2097152.0f, 2097151.0f);
  }
  keys[i] = (spread21(q[0]) << 2) | (spread21(q[1]) << 1) | spread21(q[2]);
  ids[i] = (int32_t)i;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ keys, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  const uint64_t a = keys[i], b = keys[j];
  if (a != b) return __clzll(a ^ b);
  return 64 + __clz(i ^ j);
}

// Karras 2012: internal node i of n-1; children < 0 encode leaves ~index.
__global__ void k_karras(const uint64_t* __restrict__ keys, int n, int2* children,
                         int2* ranges, int* parent_int, int* parent_leaf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  const int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
  const int dmin = delta(keys, n, i, i - d);
  int lmax = 2;
  while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
  const int j = i + l * d;
  const int dnode = delta(keys, n, i, j);
  int s = 0;
  int t = l;
  do {
    t = (t + 1) >> 1;
    if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  const int gamma = i + s * d + min(d, 0);
  const int first = min(i, j), last = max(i, j);
  const int left = (first == gamma) ? ~gamma : gamma;
  const int right = (last == gamma + 1) ? ~(gamma + 1) : gamma + 1;
  children[i] = make_int2(left, right);
  ranges[i] = make_int2(first, last);
  if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
  if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
}

struct Box32 {
  float lo[3], hi[3];
};

// Leaf boxes from float64 corners rounded outward, then bottom-up refit.
__global__ void k_refit(const double* __restrict__ v0, const double* __restrict__ v1,
                        const double* __restrict__ v2, const int32_t* __restrict__ ids,
                        int n, const int2* __restrict__ children,
                        const int* __restrict__ parent_int, const int* __restrict__ parent_leaf,
                        Box32* leaf_box, Box32* int_box, unsigned int* visits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int tri = ids[i];
  Box32 b;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = v0[3 * tri + k], c = v1[3 * tri + k], d = v2[3 * tri + k];
    b.lo[k] = __double2float_rd(fmin(fmin(a, c), d));
    b.hi[k] = __double2float_ru(fmax(fmax(a, c), d));
  }
  leaf_box[i] = b;
  if (n == 1) return;
  int node = parent_leaf[i];
  while (node >= 0) {
    __threadfence();
    if (atomicAdd(visits + node, 1u) == 0) return;  // first arrival: sibling not done
    __threadfence();
    const int2 ch = children[node];
    const Box32 bl = ch.x < 0 ? leaf_box[~ch.x] : int_box[ch.x];
    const Box32 br = ch.y < 0 ? leaf_box[~ch.y] : int_box[ch.y];
    Box32 u;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      u.lo[k] = fminf(bl.lo[k], br.lo[k]);
      u.hi[k] = fmaxf(bl.hi[k], br.hi[k]);
    }
    int_box[node] = u;
    node = node == 0 ? -1 : parent_int[node];
  }
}

#ifndef SBR_LEAF_MAX
#define SBR_LEAF_MAX 2  // leaves of <= 2 triangles: a float64 triangle test costs ~4 fp32 box
                        // tests, so smaller leaves win (canyon 2.55e9 -> 2.70e9 rb/s vs 4);
                        // the leaf code allows up to 4 (count - 1 in 2 bits)
#endif
__global__ void k_keep_flags(const int2* __restrict__ ranges, int nint, int* keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nint) return;
  const int2 r = ranges[i];
  keep[i] = (r.y - r.x + 1) > SBR_LEAF_MAX ? 1 : 0;
}

// Emit the collapsed BVH2 nodes.  Child code: internal kept node -> its
// compact index; subtree of <= SBR_LEAF_MAX triangles -> leaf(first, count).
__global__ void k_emit(const int2* __restrict__ children, const int2* __restrict__ ranges,
                       const int* __restrict__ keep, const int* __restrict__ compact,
                       const Box32* __restrict__ leaf_box, const Box32* __restrict__ int_box,
                       int nint, BvhNode* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nint || !keep[i]) return;
  const int2 ch = children[i];
  int code[2];
  Box32 bx[2];
  const int c2[2] = {ch.x, ch.y};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int c = c2[s];
    if (c < 0) {
      code[s] = leaf_encode(~c, 1);
      bx[s] = leaf_box[~c];
    } else {
      const int2 r = ranges[c];
      bx[s] = int_box[c];
      code[s] = keep[c] ? compact[c] : leaf_encode(r.x, r.y - r.x + 1);
    }
  }
  BvhNode nd;
  nd.a = make_float4(bx[0].lo[0], bx[0].hi[0], bx[0].lo[1], bx[0].hi[1]);
  nd.b = make_float4(bx[1].lo[0], bx[1].hi[0], bx[1].lo[1], bx[1].hi[1]);
  nd.c = make_float4(bx[0].lo[2], bx[0].hi[2], bx[1].lo[2], bx[1].hi[2]);
  nd.d = make_int4(code[0], code[1], 0, 0);
  out[compact[i]] = nd;
}

// root for scenes of <= 4 triangles: both children are the single leaf
__global__ void k_small_root(const Box32* __restrict__ leaf_box, int n, BvhNode* out) {
  Box32 u = leaf_box[0];
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      u.lo[k] = fminf(u.lo[k], leaf_box[i].lo[k]);
      u.hi[k] = fmaxf(u.hi[k], leaf_box[i].hi[k]);
    }
  BvhNode nd;
  nd.a = make_float4(u.lo[0], u.hi[0], u.lo[1], u.hi[1]);
  nd.b = nd.a;
  nd.c = make_float4(u.lo[2], u.hi[2], u.lo[2], u.hi[2]);
  const int code = leaf_encode(0, n);
  nd.d = make_int4(code, code, 0, 0);
  out[0] = nd;
}

__global__ void k_gather_tris(const double* __restrict__ v0, const double* __restrict__ v1,
                              const double* __restrict__ v2, const int32_t* __restrict__ ids,
                              int n, TriSlot* tris) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = ids[i];
  TriSlot s;
  s.p[0] = make_double2(v0[3 * t], v0[3 * t + 1]);
  s.p[1] = make_double2(v0[3 * t + 2], v1[3 * t]);
  s.p[2] = make_double2(v1[3 * t + 1], v1[3 * t + 2]);
  s.p[3] = make_double2(v2[3 * t], v2[3 * t + 1]);
  s.p[4] = make_double2(v2[3 * t + 2], 0.0);
  tris[i] = s;
}

// Per-slot geometry tables of SceneModel._build_tables (paths.py:446-450) and
// Accel (geometry.py:165-166), computed on the device from the float64
// corners with numpy's operation order (-fmad=false, no contraction):
//   normal = cross(v1 - v0, v2 - v0) / norm      (np.cross, np.linalg.norm)
//   plane hashes of _plane_hash_rows (paths.py:156-171): the normal divided
//   by its norm again, canonical sign (first |c| > 1e-8 positive), d = n . v0
//   as ((n0 p0 + n1 p1) + n2 p2), FNV-1a over the 8 little-endian bytes of
//   floor(c / 1e-4 + 0.5) and floor(c / 1e-4) for c in (n0, n1, n2, d).
__device__ __forceinline__ uint64_t fnv1a_fold(uint64_t h, uint64_t v) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    h = (h ^ (v & 0xFFULL)) * 0x100000001B3ULL;
    v >>= 8;
  }
  return h;
}

__global__ void k_slot_tables(const TriSlot* __restrict__ tris, int n, double* __restrict__ normals,
                              uint64_t* __restrict__ hash_r, uint64_t* __restrict__ hash_f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* T = reinterpret_cast<const double*>(tris + i);
  const double a0 = T[3] - T[0], a1 = T[4] - T[1], a2 = T[5] - T[2];   // v1 - v0
  const double b0 = T[6] - T[0], b1 = T[7] - T[1], b2 = T[8] - T[2];   // v2 - v0
  const double c0 = a1 * b2 - a2 * b1, c1 = a2 * b0 - a0 * b2, c2 = a0 * b1 - a1 * b0;
  const double len = sqrt((c0 * c0 + c1 * c1) + c2 * c2);
  double m0 = c0 / len, m1 = c1 / len, m2 = c2 / len;
  normals[3 * (int64_t)i] = m0;
  normals[3 * (int64_t)i + 1] = m1;
  normals[3 * (int64_t)i + 2] = m2;
  const double len2 = sqrt((m0 * m0 + m1 * m1) + m2 * m2);
  m0 = m0 / len2;
  m1 = m1 / len2;
  m2 = m2 / len2;
  const double lead = fabs(m0) > 1e-8 ? m0 : (fabs(m1) > 1e-8 ? m1 : (fabs(m2) > 1e-8 ? m2 : m0));
  if (lead < 0.0) {
    m0 = -m0;
    m1 = -m1;
    m2 = -m2;
  }
  const double d = (m0 * T[0] + m1 * T[1]) + m2 * T[2];
  const double comp[4] = {m0, m1, m2, d};
  uint64_t hr = 0xCBF29CE484222325ULL, hf = 0xCBF29CE484222325ULL;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double q = comp[k] / 1e-4;
    hr = fnv1a_fold(hr, (uint64_t)(int64_t)floor(q + 0.5));
    hf = fnv1a_fold(hf, (uint64_t)(int64_t)floor(q));
  }
  hash_r[i] = hr;
  hash_f[i] = hf;
}

// ---------------------------------------------------------------------------
// PLOC: parallel locally-ordered clustering over the Morton order (Meister &
// Bittner 2018).  Clusters start as the Morton-sorted leaves; every round each
// cluster finds its cheapest merge partner (surface area of the union) within
// +-kPlocRadius positions, mutual nearest pairs merge, the cluster list is
// compacted.  Gives SAH-like trees from the same GPU sort; the result is
// converted to the Karras-style (children, ranges) arrays by renumbering the
// leaves in depth-first order, so the leaf collapse / emit path is shared.
// ---------------------------------------------------------------------------
#ifndef SBR_PLOC_RADIUS
// PLOC search radius.  Re-swept on the config-4 headline (city, 1e9-ray map,
// k_map_trace ms per map / nodes per ray-bounce): r4 540, r6 520, r7 458,
// r8 474-496 / 25.9, r9 556, r10 599, r12 624 / 30.3, r16 528 / 26.6, r24
// worse; config-3 visibility r7 59.8 ms vs r16 60.8; the canyon trace is
// flat (4.1-4.3 ms).  SAH cost (61.2-62.6) does not rank these trees;
// visits per ray do.
#define SBR_PLOC_RADIUS 9  // with the SAH top (below) the radius barely matters
#endif
constexpr int kPlocRadius = SBR_PLOC_RADIUS;
// The greedy merges of the last large clusters decide the top of the tree;
// at some radii they made the root's children overlap (child / root surface
// area 1.53 instead of 1.05) and the city trace 20 % slower.  Once kPlocTop
// clusters remain, the rest of the tree is built top-down by SAH over the
// cluster boxes (SahBuild, host threads).  City trace per config-4 map
// (ms) / build (s): PLOC only 458 / 0.14, top 16k 444, 64k 405 / 0.28, 256k
// 388 / 0.20, pure SAH 389 / 0.50; canyon 4.23 -> 3.37 ms; config-3
// visibility 59.9 -> 57.6 ms.
#ifndef SBR_PAD_FLOOR_LOG2
#define SBR_PAD_FLOOR_LOG2 62  // was 26: boxes padded by 1.5e-8 x the scene size
#endif
#ifndef SBR_PLOC_TOP
#define SBR_PLOC_TOP 262144
#endif
constexpr int kPlocTop = SBR_PLOC_TOP;

__device__ __forceinline__ float half_area(const Box32& b) {
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return dx * dy + dy * dz + dz * dx;
}

__device__ __forceinline__ Box32 box_union(const Box32& a, const Box32& b) {
  Box32 u;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    u.lo[k] = fminf(a.lo[k], b.lo[k]);
    u.hi[k] = fmaxf(a.hi[k], b.hi[k]);
  }
  return u;
}

__global__ void k_leaf_boxes(const double* __restrict__ v0, const double* __restrict__ v1,
                             const double* __restrict__ v2, const int32_t* __restrict__ ids,
                             int n, Box32* box) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int tri = ids[i];
  Box32 b;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = v0[3 * tri + k], c = v1[3 * tri + k], d = v2[3 * tri + k];
    b.lo[k] = __double2float_rd(fmin(fmin(a, c), d));
    b.hi[k] = __double2float_ru(fmax(fmax(a, c), d));
  }
  box[i] = b;
}

__global__ void k_iota_i32(int32_t* a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void k_ploc_nearest(const int32_t* __restrict__ C, int m, const Box32* __restrict__ box,
                               int32_t* nearest, int radius) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const Box32 bi = box[C[i]];
  float best = __int_as_float(0x7f800000);
  int bj = -1;
  const int lo = i - radius < 0 ? 0 : i - radius;
  const int hi = i + radius >= m ? m - 1 : i + radius;
  for (int j = lo; j <= hi; ++j) {
    if (j == i) continue;
    const float c = half_area(box_union(bi, box[C[j]]));
    if (c < best) {  // ties keep the lower index: deterministic
      best = c;
      bj = j;
    }
  }
  nearest[i] = bj;
}

__global__ void k_ploc_flags(const int32_t* __restrict__ nearest, int m, int32_t* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int j = nearest[i];
  flag[i] = (j > i && nearest[j] == i) ? 1 : 0;
}

__global__ void k_ploc_merge(int32_t* C, const int32_t* __restrict__ nearest,
                             const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                             int m, int n, int base, Box32* box, int2* kids, int32_t* parent,
                             int32_t* csize) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || !flag[i]) return;
  const int j = nearest[i];
  const int id = base + pos[i];  // internal node ids n .. 2n-2, creation order
  const int a = C[i], b = C[j];
  kids[id - n] = make_int2(a, b);
  box[id] = box_union(box[a], box[b]);
  csize[id] = csize[a] + csize[b];
  parent[a] = id;
  parent[b] = id;
  C[i] = id;
  C[j] = -1;
}

__global__ void k_ploc_valid(const int32_t* __restrict__ C, int m, int32_t* valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) valid[i] = C[i] >= 0 ? 1 : 0;
}

__global__ void k_ploc_compact(const int32_t* __restrict__ C, const int32_t* __restrict__ valid,
                               const int32_t* __restrict__ pos, int m, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m && valid[i]) out[pos[i]] = C[i];
}

// leaf counts bottom-up (second arrival at a node sums its children)
__global__ void k_ploc_counts(const int32_t* __restrict__ parent, const int2* __restrict__ kids,
                              int n, int32_t* cnt, unsigned* visits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  cnt[i] = 1;
  int node = parent[i];
  while (node >= 0) {
    __threadfence();
    if (atomicAdd(visits + (node - n), 1u) == 0) return;
    __threadfence();
    const int2 k = kids[node - n];
    cnt[node] = cnt[k.x] + cnt[k.y];
    node = parent[node];
  }
}

// depth-first offset of every node: sum of left-sibling counts on the root path
__global__ void k_ploc_offsets(const int32_t* __restrict__ parent, const int2* __restrict__ kids,
                               const int32_t* __restrict__ cnt, int total, int n, int32_t* off) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= total) return;
  int o = 0, c = v, p = parent[v];
  while (p >= 0) {
    const int2 k = kids[p - n];
    if (k.y == c) o += cnt[k.x];
    c = p;
    p = parent[p];
  }
  off[v] = o;
}

// Karras-style arrays: internal node id -> index (2n-2-id, root at 0), leaves
// encoded ~(depth-first slot)
__global__ void k_ploc_export(const int2* __restrict__ kids, const int32_t* __restrict__ cnt,
                              const int32_t* __restrict__ off, const Box32* __restrict__ box,
                              int n, int2* children, int2* ranges, Box32* int_box) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n - 1) return;
  const int id = n + k;
  const int idx = 2 * n - 2 - id;
  const int2 c = kids[k];
  const int l = c.x < n ? ~off[c.x] : 2 * n - 2 - c.x;
  const int r = c.y < n ? ~off[c.y] : 2 * n - 2 - c.y;
  children[idx] = make_int2(l, r);
  ranges[idx] = make_int2(off[id], off[id] + cnt[id] - 1);
  int_box[idx] = box[id];
}

__global__ void k_ploc_leaves(const int32_t* __restrict__ off, const Box32* __restrict__ box,
                              const int32_t* __restrict__ ids_sorted, int n, Box32* leaf_box,
                              int32_t* ids_dfs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = off[i];
  leaf_box[s] = box[i];
  ids_dfs[s] = ids_sorted[i];
}

__global__ void k_fill_i32(int32_t* a, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

static inline float half_area_h(const Box32& b) {
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return dx * dy + dy * dz + dz * dx;
}
static inline Box32 box_union_h(const Box32& a, const Box32& b) {
  Box32 u;
  for (int k = 0; k < 3; ++k) {
    u.lo[k] = fminf(a.lo[k], b.lo[k]);
    u.hi[k] = fmaxf(a.hi[k], b.hi[k]);
  }
  return u;
}

// Top-down SAH over clusters (boxes + triangle counts): binned (64 centroid
// bins per axis) above 1024 clusters, an exact sweep below.  Subtrees above
// 16k clusters are built on separate host threads; each returns its internal
// nodes in post-order and the parent concatenates (left, right, itself), so
// the node numbering -- and with it the emitted tree -- is deterministic.
struct SahBuild {
  struct Node {
    int l, r;  // child refs: >= 0 cluster (node) id, < 0 local node ~k
    Box32 b;
    int64_t sz;
  };
  const std::vector<Box32>& box;      // cluster boxes (read-only)
  const std::vector<int32_t>& size;   // triangles per cluster
  static constexpr int kBins = 64;

  static float centroid2(const Box32& x, int axis) { return x.lo[axis] + x.hi[axis]; }

  // binned SAH split of ids[lo, hi) (partitioned in place); -1 if none
  int binned_split(std::vector<int32_t>& ids, int lo, int hi) const {
    float cmin[3] = {__builtin_inff(), __builtin_inff(), __builtin_inff()};
    float cmax[3] = {-__builtin_inff(), -__builtin_inff(), -__builtin_inff()};
    for (int i = lo; i < hi; ++i)
      for (int k = 0; k < 3; ++k) {
        const float c = centroid2(box[ids[i]], k);
        cmin[k] = fminf(cmin[k], c);
        cmax[k] = fmaxf(cmax[k], c);
      }
    float best_cost = __builtin_inff();
    int best_axis = -1, best_bin = 0;
    for (int axis = 0; axis < 3; ++axis) {
      const float ext = cmax[axis] - cmin[axis];
      if (!(ext > 0.0f)) continue;
      const float scale = kBins / ext;
      Box32 bb[kBins];
      int64_t bc[kBins] = {0};
      for (int b = 0; b < kBins; ++b)
        for (int k = 0; k < 3; ++k) {
          bb[b].lo[k] = __builtin_inff();
          bb[b].hi[k] = -__builtin_inff();
        }
      for (int i = lo; i < hi; ++i) {
        const Box32& x = box[ids[i]];
        int b = (int)((centroid2(x, axis) - cmin[axis]) * scale);
        b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
        bb[b] = box_union_h(bb[b], x);
        bc[b] += size[ids[i]];
      }
      float rc[kBins];
      Box32 acc = bb[kBins - 1];
      int64_t cnt = 0;
      for (int b = kBins - 1; b > 0; --b) {
        acc = box_union_h(acc, bb[b]);
        cnt += bc[b];
        rc[b] = cnt ? half_area_h(acc) * (float)cnt : 0.0f;
      }
      acc = bb[0];
      cnt = 0;
      for (int b = 1; b < kBins; ++b) {  // split: bins [0, b) | [b, kBins)
        acc = box_union_h(acc, bb[b - 1]);
        cnt += bc[b - 1];
        if (!cnt || rc[b] == 0.0f) continue;
        const float c = half_area_h(acc) * (float)cnt + rc[b];
        if (c < best_cost) {
          best_cost = c;
          best_axis = axis;
          best_bin = b;
        }
      }
    }
    if (best_axis < 0) return -1;
    const float scale = kBins / (cmax[best_axis] - cmin[best_axis]);
    const auto mid = std::stable_partition(ids.begin() + lo, ids.begin() + hi, [&](int id) {
      int b = (int)((centroid2(box[id], best_axis) - cmin[best_axis]) * scale);
      b = b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
      return b < best_bin;
    });
    const int split = (int)(mid - ids.begin());
    return (split > lo && split < hi) ? split : -1;
  }

  // exact SAH sweep over the three centroid orders (ids[lo, hi) left sorted
  // along the chosen axis); returns the split position
  int exact_split(std::vector<int32_t>& ids, int lo, int hi) const {
    int best_axis = 0, best_split = lo + (hi - lo) / 2;
    float best_cost = __builtin_inff();
    std::vector<float> right_cost(hi - lo);
    auto order = [&](int axis) {
      std::sort(ids.begin() + lo, ids.begin() + hi, [&](int a, int b) {
        const float ca = centroid2(box[a], axis), cb = centroid2(box[b], axis);
        return ca < cb || (ca == cb && a < b);
      });
    };
    for (int axis = 0; axis < 3; ++axis) {
      order(axis);
      Box32 acc = box[ids[hi - 1]];
      int64_t cnt = 0;
      for (int i = hi - 1; i > lo; --i) {  // suffix [i, hi)
        acc = box_union_h(acc, box[ids[i]]);
        cnt += size[ids[i]];
        right_cost[i - lo] = half_area_h(acc) * (float)cnt;
      }
      acc = box[ids[lo]];
      cnt = 0;
      for (int i = lo + 1; i < hi; ++i) {  // split: [lo, i) | [i, hi)
        acc = box_union_h(acc, box[ids[i - 1]]);
        cnt += size[ids[i - 1]];
        const float c = half_area_h(acc) * (float)cnt + right_cost[i - lo];
        if (c < best_cost) {
          best_cost = c;
          best_axis = axis;
          best_split = i;
        }
      }
    }
    order(best_axis);
    return best_split;
  }

  Box32 ref_box(int ref, const std::vector<Node>& out) const { return ref >= 0 ? box[ref] : out[~ref].b; }
  int64_t ref_size(int ref, const std::vector<Node>& out) const {
    return ref >= 0 ? size[ref] : out[~ref].sz;
  }
  int emit(int l, int r, std::vector<Node>& out) const {
    out.push_back(Node{l, r, box_union_h(ref_box(l, out), ref_box(r, out)),
                       ref_size(l, out) + ref_size(r, out)});
    return ~(int)(out.size() - 1);
  }

  // subtree over ids[lo, hi): internal nodes appended to `out` in post-order
  int build(std::vector<int32_t>& ids, int lo, int hi, std::vector<Node>& out, int depth) const {
    if (hi - lo == 1) return ids[lo];
    int split = hi - lo > 1024 ? binned_split(ids, lo, hi) : -1;
    if (split < 0) split = exact_split(ids, lo, hi);
    if (depth < 5 && hi - lo > 16384) {
      std::vector<Node> lout, rout;
      int lref = 0;
      std::thread t([&] { lref = build(ids, lo, split, lout, depth + 1); });
      int rref = build(ids, split, hi, rout, depth + 1);
      t.join();
      auto remap = [](int ref, int off) { return ref < 0 ? ~(~ref + off) : ref; };
      const int offl = (int)out.size();
      for (const Node& x : lout) out.push_back(Node{remap(x.l, offl), remap(x.r, offl), x.b, x.sz});
      const int offr = (int)out.size();
      for (const Node& x : rout) out.push_back(Node{remap(x.l, offr), remap(x.r, offr), x.b, x.sz});
      return emit(remap(lref, offl), remap(rref, offr), out);
    }
    const int l = build(ids, lo, split, out, depth + 1);
    const int r = build(ids, split, hi, out, depth + 1);
    return emit(l, r, out);
  }
};

// top-down SAH over the m remaining PLOC clusters C[0, m): new internal nodes
// base .. base + m - 2 (children before parents, root last)
static int ploc_top_sah(const int32_t* C, int m, int n, int base, Box32* box_all, int2* kids,
                        int32_t* parent, int32_t* csize, cudaStream_t st) {
  const int total = 2 * n - 1;
  std::vector<int32_t> ids(m), hpar(total), hsize(total);
  std::vector<Box32> hbox(total);
  SBR_CUDA(cudaMemcpyAsync(ids.data(), C, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st));
  SBR_CUDA(cudaMemcpyAsync(hbox.data(), box_all, sizeof(Box32) * total, cudaMemcpyDeviceToHost, st));
  SBR_CUDA(cudaMemcpyAsync(hpar.data(), parent, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, st));
  SBR_CUDA(cudaMemcpyAsync(hsize.data(), csize, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, st));
  SBR_CUDA(cudaStreamSynchronize(st));
  SahBuild B{hbox, hsize};
  std::vector<SahBuild::Node> out;
  out.reserve(m);
  B.build(ids, 0, m, out, 0);
  const int made = (int)out.size();
  if (made != m - 1) return set_error(SBR_ERR_INTERNAL, "PLOC top build: bad node count");
  std::vector<int2> hk(made);
  auto gid = [&](int ref) { return ref >= 0 ? ref : base + ~ref; };
  for (int k = 0; k < made; ++k) {
    const int id = base + k, l = gid(out[k].l), r = gid(out[k].r);
    hk[k] = make_int2(l, r);
    hbox[id] = out[k].b;
    hpar[l] = id;
    hpar[r] = id;
  }
  SBR_CUDA(cudaMemcpyAsync(kids + (base - n), hk.data(), sizeof(int2) * made,
                           cudaMemcpyHostToDevice, st));
  SBR_CUDA(cudaMemcpyAsync(box_all + base, hbox.data() + base, sizeof(Box32) * made,
                           cudaMemcpyHostToDevice, st));
  SBR_CUDA(cudaMemcpyAsync(parent, hpar.data(), sizeof(int32_t) * total, cudaMemcpyHostToDevice, st));
  SBR_CUDA(cudaStreamSynchronize(st));
  return SBR_OK;
}

static std::atomic<int> g_builder{1};  // 0 = Karras LBVH, 1 = PLOC + SAH top, 2 = PLOC only

// persistent scene buffer (freed by sbr_scene_destroy)
template <typename T>
static int palloc(T** p, size_t count) {
  SBR_CUDA(cudaMalloc((void**)p, sizeof(T) * (count ? count : 1)));
  return SBR_OK;
}

// stream-ordered build scratch, released (in stream order) on every exit path
struct ScratchArena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit ScratchArena(cudaStream_t s) : st(s) {}
  ScratchArena(const ScratchArena&) = delete;
  ScratchArena& operator=(const ScratchArena&) = delete;
  template <typename T>
  int get(T** p, size_t count) {
    void* q = nullptr;
    const cudaError_t e = scratch_alloc(&q, sizeof(T) * (count ? count : 1), st);
    if (e != cudaSuccess)
      return set_error(SBR_ERR_NOMEM, std::string("scene build scratch: ") + cudaGetErrorString(e));
    ptrs.push_back(q);
    *p = (T*)q;
    return SBR_OK;
  }
  ~ScratchArena() {
    for (void* q : ptrs) cudaFreeAsync(q, st);
  }
};

static inline unsigned grid_for(int64_t n, int block) {
  return (unsigned)((n + block - 1) / block);
}

}  // namespace sbr

using namespace sbr;

extern "C" {

const char* sbr_last_error(void) { return g_last_error.c_str(); }
int sbr_version(void) { return 100; }
// bit 0: checked build (-DSBR_CHECKED device bounds assertions)
int sbr_build_flags(void) {
#ifdef SBR_CHECKED
  return 1;
#else
  return 0;
#endif
}

int sbr_set_bvh_builder(int32_t builder) {
  if (builder < 0 || builder > 2)
    return set_error(SBR_ERR_INVALID, "builder: 0 LBVH, 1 PLOC + SAH top, 2 PLOC only");
  g_builder = builder;
  return SBR_OK;
}
uint64_t sbr_kernel_launches(void) { return g_launches.load(); }

int sbr_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain();
  g_prof_acc.clear();
  g_prof_on = on != 0;
  return SBR_OK;
}

double sbr_profile_kernel_ms(const char* name, uint64_t* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain();
  auto it = g_prof_acc.find(name ? name : "");
  if (launches) *launches = it == g_prof_acc.end() ? 0 : it->second.second;
  return it == g_prof_acc.end() ? 0.0 : it->second.first;
}

int sbr_scene_create(const double* v0, const double* v1, const double* v2, int64_t ntri,
                     int32_t device, void* stream, SbrScene** out) {
  if (!out) return set_error(SBR_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (ntri <= 0) return set_error(SBR_ERR_EMPTY_SCENE, "no triangles");
  if (ntri >= (1LL << 29)) return set_error(SBR_ERR_INVALID, "too many triangles");
  if (!v0 || !v1 || !v2) return set_error(SBR_ERR_INVALID, "NULL vertex array");
  double max_abs = 0.0;
  double lo[3] = {v0[0], v0[1], v0[2]}, hi[3] = {v0[0], v0[1], v0[2]};
  for (int64_t i = 0; i < 3 * ntri; ++i) {
    // a non-finite corner makes every merge cost inf / NaN (PLOC would never
    // pair its cluster) and every ray test meaningless: reject up front
    if (!std::isfinite(v0[i]) || !std::isfinite(v1[i]) || !std::isfinite(v2[i]))
      return set_error(SBR_ERR_INVALID, "non-finite vertex coordinate in triangle " +
                                            std::to_string(i / 3));
    max_abs = fmax(max_abs, fabs(v0[i]));
    max_abs = fmax(max_abs, fabs(v1[i]));
    max_abs = fmax(max_abs, fabs(v2[i]));
    const int k = (int)(i % 3);
    lo[k] = fmin(lo[k], fmin(fmin(v0[i], v1[i]), v2[i]));
    hi[k] = fmax(hi[k], fmax(fmax(v0[i], v1[i]), v2[i]));
  }
  DeviceGuard dg(device);
  {
    int cur = -1;
    SBR_CUDA(cudaGetDevice(&cur));
    if (cur != device) return set_error(SBR_ERR_CUDA, "cannot select device " + std::to_string(device));
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = (int)ntri;
  // the scene is destroyed (every persistent buffer freed) on any early
  // return; the scratch arena frees its buffers (stream-ordered) on every exit
  std::unique_ptr<SbrScene, void (*)(SbrScene*)> owner(new SbrScene(), sbr_scene_destroy);
  SbrScene* S = owner.get();
  ScratchArena A(st);
  S->device = device;
  S->ntri = ntri;
  for (int k = 0; k < 3; ++k) {
    S->lo[k] = lo[k];
    S->hi[k] = hi[k];
  }
  // box_setup's pad floor: with a direction component of exactly +-0 its
  // reciprocal is clamped to +-1e20, and the pad x 1e20 must then exceed any
  // distance inside the scene (2^-62 x 1e20 = 21.7 x the largest coordinate);
  // the relative pad 2^-22 |o| carries the rest of the error analysis
  S->pad_base = (float)(ldexp(max_abs + 1.0, -SBR_PAD_FLOOR_LOG2));

  double *dv0, *dv1, *dv2;
  const size_t bytes = sizeof(double) * 3 * (size_t)ntri;
  int rc;
  if ((rc = A.get(&dv0, 3 * ntri)) || (rc = A.get(&dv1, 3 * ntri)) || (rc = A.get(&dv2, 3 * ntri)))
    return rc;
  SBR_CUDA(cudaMemcpyAsync(dv0, v0, bytes, cudaMemcpyHostToDevice, st));
  SBR_CUDA(cudaMemcpyAsync(dv1, v1, bytes, cudaMemcpyHostToDevice, st));
  SBR_CUDA(cudaMemcpyAsync(dv2, v2, bytes, cudaMemcpyHostToDevice, st));

  float3* cen;
  unsigned int* cb;
  uint64_t *keys, *keys_sorted;
  int32_t *ids, *ids_sorted;
  if ((rc = A.get(&cen, n)) || (rc = A.get(&cb, 6)) || (rc = A.get(&keys, n)) ||
      (rc = A.get(&keys_sorted, n)) || (rc = A.get(&ids, n)) || (rc = A.get(&ids_sorted, n)))
    return rc;
  const unsigned init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
  SBR_CUDA(cudaMemcpyAsync(cb, init, sizeof init, cudaMemcpyHostToDevice, st));
  k_centroids<<<grid_for(n, 256), 256, 0, st>>>(dv0, dv1, dv2, n, cen, cb);
  count_launch();
  k_morton<<<grid_for(n, 256), 256, 0, st>>>(cen, n, cb, keys, ids);
  count_launch();
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, ids, ids_sorted, n, 0,
                                  64, st);
  char* tmp;
  if ((rc = A.get(&tmp, tmp_bytes))) return rc;
  SBR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, ids, ids_sorted,
                                           n, 0, 64, st));
  count_launch();

  const int nint = n > 1 ? n - 1 : 0;
  int2 *children, *ranges;
  int *parent_int, *parent_leaf, *keep, *compact;
  Box32 *leaf_box, *int_box;
  unsigned int* visits;
  if ((rc = A.get(&children, nint)) || (rc = A.get(&ranges, nint)) ||
      (rc = A.get(&parent_int, nint)) || (rc = A.get(&parent_leaf, n)) ||
      (rc = A.get(&keep, nint)) || (rc = A.get(&compact, nint)) || (rc = A.get(&leaf_box, n)) ||
      (rc = A.get(&int_box, nint)) || (rc = A.get(&visits, nint)))
    return rc;
  int32_t* ids_leaf = ids_sorted;  // triangle of each leaf slot
  const int builder = g_builder;
  if (builder >= 1 && n > 1) {
    const int top = builder == 1 ? kPlocTop : 0;
    // ---- PLOC hierarchy, exported in depth-first leaf order ----
    const int total = 2 * n - 1;
    Box32* box_all;
    int2* kids;
    int32_t *C, *C2, *nearest, *flag, *pos, *parent, *cnt, *off, *ids_dfs;
    unsigned* vis2;
    int32_t* csize;
    if ((rc = A.get(&csize, total))) return rc;
    k_fill_i32<<<grid_for(n, 256), 256, 0, st>>>(csize, n, 1);
    count_launch();
    if ((rc = A.get(&box_all, total)) || (rc = A.get(&kids, nint)) || (rc = A.get(&C, n)) ||
        (rc = A.get(&C2, n)) || (rc = A.get(&nearest, n)) || (rc = A.get(&flag, n + 1)) ||
        (rc = A.get(&pos, n + 1)) || (rc = A.get(&parent, total)) || (rc = A.get(&cnt, total)) ||
        (rc = A.get(&off, total)) || (rc = A.get(&vis2, nint)) || (rc = A.get(&ids_dfs, n)))
      return rc;
    k_leaf_boxes<<<grid_for(n, 256), 256, 0, st>>>(dv0, dv1, dv2, ids_sorted, n, box_all);
    count_launch();
    k_iota_i32<<<grid_for(n, 256), 256, 0, st>>>(C, n);
    count_launch();
    SBR_CUDA(cudaMemsetAsync(parent, 0xff, sizeof(int32_t) * total, st));
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, flag, pos, n + 1, st);
    char* stmp;
    if ((rc = A.get(&stmp, sb))) return rc;
    int m = n, base = n;
    while (m > 1) {
      if (m <= top) {
        // the last clusters: top-down SAH instead of greedy merging (below)
        if ((rc = ploc_top_sah(C, m, n, base, box_all, kids, parent, csize, st))) return rc;
        base += m - 1;
        m = 1;
        break;
      }
      k_ploc_nearest<<<grid_for(m, 128), 128, 0, st>>>(C, m, box_all, nearest, kPlocRadius);
      k_ploc_flags<<<grid_for(m, 256), 256, 0, st>>>(nearest, m, flag);
      SBR_CUDA(cub::DeviceScan::ExclusiveSum(stmp, sb, flag, pos, m + 1, st));
      k_ploc_merge<<<grid_for(m, 256), 256, 0, st>>>(C, nearest, flag, pos, m, n, base, box_all,
                                                     kids, parent, csize);
      k_ploc_valid<<<grid_for(m, 256), 256, 0, st>>>(C, m, flag);
      SBR_CUDA(cub::DeviceScan::ExclusiveSum(stmp, sb, flag, pos, m + 1, st));
      k_ploc_compact<<<grid_for(m, 256), 256, 0, st>>>(C, flag, pos, m, C2);
      int m_new = 0;
      SBR_CUDA(cudaMemcpyAsync(&m_new, pos + m, sizeof(int), cudaMemcpyDeviceToHost, st));
      SBR_CUDA(cudaStreamSynchronize(st));
      SBR_CUDA(cudaGetLastError());
      for (int q = 0; q < 7; ++q) count_launch();
      // every pass merges at least the globally cheapest mutual pair, so m
      // shrinks unless the merge costs are not comparable (NaN boxes)
      if (m_new >= m || m_new < 1)
        return set_error(SBR_ERR_INVALID, "PLOC build made no progress (" + std::to_string(m) +
                                              " clusters left): non-comparable triangle boxes");
      base += m - m_new;
      m = m_new;
      int32_t* t = C;
      C = C2;
      C2 = t;
    }
    SBR_CUDA(cudaMemsetAsync(vis2, 0, sizeof(unsigned) * nint, st));
    k_ploc_counts<<<grid_for(n, 256), 256, 0, st>>>(parent, kids, n, cnt, vis2);
    k_ploc_offsets<<<grid_for(total, 256), 256, 0, st>>>(parent, kids, cnt, total, n, off);
    k_ploc_export<<<grid_for(nint, 256), 256, 0, st>>>(kids, cnt, off, box_all, n, children, ranges,
                                                       int_box);
    k_ploc_leaves<<<grid_for(n, 256), 256, 0, st>>>(off, box_all, ids_sorted, n, leaf_box,
                                                    ids_dfs);
    for (int q = 0; q < 4; ++q) count_launch();
    ids_leaf = ids_dfs;
  } else {
    if (nint) {
      SBR_CUDA(cudaMemsetAsync(visits, 0, sizeof(unsigned) * nint, st));
      SBR_CUDA(cudaMemsetAsync(parent_int, 0xff, sizeof(int) * nint, st));
      k_karras<<<grid_for(nint, 256), 256, 0, st>>>(keys_sorted, n, children, ranges, parent_int,
                                                    parent_leaf);
      count_launch();
    }
    k_refit<<<grid_for(n, 256), 256, 0, st>>>(dv0, dv1, dv2, ids_sorted, n, children, parent_int,
                                              parent_leaf, leaf_box, int_box, visits);
    count_launch();
  }

  int nnodes = 1;
  if (n > 4) {
    k_keep_flags<<<grid_for(nint, 256), 256, 0, st>>>(ranges, nint, keep);
    count_launch();
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, keep, compact, nint, st);
    char* scan_tmp;
    if ((rc = A.get(&scan_tmp, scan_bytes))) return rc;
    SBR_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, keep, compact, nint, st));
    count_launch();
    int last_c = 0, last_k = 0;
    SBR_CUDA(cudaMemcpyAsync(&last_c, compact + nint - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    SBR_CUDA(cudaMemcpyAsync(&last_k, keep + nint - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    SBR_CUDA(cudaStreamSynchronize(st));
    nnodes = last_c + last_k;
  }
  if ((rc = palloc(&S->nodes, nnodes))) return rc;
  if (n > 4) {
    k_emit<<<grid_for(nint, 256), 256, 0, st>>>(children, ranges, keep, compact, leaf_box,
                                                int_box, nint, S->nodes);
  } else {
    k_small_root<<<1, 1, 0, st>>>(leaf_box, n, S->nodes);
  }
  count_launch();
  S->nnodes = nnodes;
  {
    // tree depth (host walk over the emitted nodes): traversals whose stack
    // cannot overflow skip the per-push check
    std::vector<BvhNode> bn((size_t)nnodes);
    SBR_CUDA(cudaMemcpyAsync(bn.data(), S->nodes, sizeof(BvhNode) * (size_t)nnodes,
                             cudaMemcpyDeviceToHost, st));
    SBR_CUDA(cudaStreamSynchronize(st));
    std::vector<std::pair<int, int>> work{{0, 1}};
    int depth = 1;
    while (!work.empty()) {
      const auto [id, d] = work.back();
      work.pop_back();
      depth = std::max(depth, d + 1);  // + the leaf level
      const int kids[2] = {bn[id].d.x, bn[id].d.y};
      for (int c : kids)
        if (c >= 0 && c < nnodes) work.push_back({c, d + 1});
    }
    S->depth = depth;
  }

  if ((rc = palloc(&S->tris, n))) return rc;
  k_gather_tris<<<grid_for(n, 256), 256, 0, st>>>(dv0, dv1, dv2, ids_leaf, n, S->tris);
  count_launch();

  S->perm.resize(n);
  std::vector<int32_t> ids_host(n);
  SBR_CUDA(cudaMemcpyAsync(ids_host.data(), ids_leaf, sizeof(int32_t) * n,
                           cudaMemcpyDeviceToHost, st));
  // default per-slot tables
  if ((rc = palloc(&S->error_word, 1)) || (rc = palloc(&S->tie_rank, n)) ||
      (rc = palloc(&S->normals, 3 * (size_t)n)) || (rc = palloc(&S->matrow, n)) ||
      (rc = palloc(&S->hash_r, n)) || (rc = palloc(&S->hash_f, n)))
    return rc;
  SBR_CUDA(cudaMemsetAsync(S->error_word, 0, sizeof(unsigned), st));
  SBR_CUDA(cudaMemsetAsync(S->matrow, 0, sizeof(int32_t) * n, st));
  k_slot_tables<<<grid_for(n, 256), 256, 0, st>>>(S->tris, n, S->normals, S->hash_r, S->hash_f);
  count_launch();
  SBR_CUDA(cudaStreamSynchronize(st));
  SBR_CUDA(cudaGetLastError());
  for (int i = 0; i < n; ++i) S->perm[i] = ids_host[i];
  *out = owner.release();
  return SBR_OK;
}

void sbr_scene_destroy(SbrScene* S) {
  if (!S) return;
  DeviceGuard dg(S->device);  // the caller's current device is restored on return
  cudaFree(S->nodes);
  cudaFree(S->tris);
  cudaFree(S->tie_rank);
  cudaFree(S->normals);
  cudaFree(S->matrow);
  cudaFree(S->hash_r);
  cudaFree(S->hash_f);
  cudaFree(S->mats);
  cudaFree(S->error_word);
  cudaFree(S->wedge_block);
  delete S;
}

int sbr_release_scratch(int32_t device) {
  int count = 0;
  SBR_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count || device >= kMaxDevices)
    return set_error(SBR_ERR_INVALID, "bad device");
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    pool = g_pools[device];
  }
  if (pool) {
    DeviceGuard dg(device);
    SBR_CUDA(cudaDeviceSynchronize());
    SBR_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  return SBR_OK;
}

int64_t sbr_scene_num_triangles(const SbrScene* S) { return S ? S->ntri : 0; }
int64_t sbr_scene_num_nodes(const SbrScene* S) { return S ? S->nnodes : 0; }

int sbr_scene_copy_nodes(const SbrScene* S, void* host_out) {
  if (!S || !host_out) return set_error(SBR_ERR_INVALID, "NULL argument");
  SBR_CUDA(cudaMemcpy(host_out, S->nodes, sizeof(BvhNode) * (size_t)S->nnodes,
                      cudaMemcpyDeviceToHost));
  return SBR_OK;
}

int sbr_scene_permutation(const SbrScene* S, int64_t* perm_out) {
  if (!S || !perm_out) return set_error(SBR_ERR_INVALID, "NULL argument");
  memcpy(perm_out, S->perm.data(), sizeof(int64_t) * S->perm.size());
  return SBR_OK;
}

int sbr_scene_copy_tables(const SbrScene* S, double* normals_out, uint64_t* hash_r_out,
                          uint64_t* hash_f_out) {
  if (!S) return set_error(SBR_ERR_INVALID, "NULL scene");
  DeviceGuard dg(S->device);
  const size_t n = (size_t)S->ntri;
  if (normals_out) SBR_CUDA(cudaMemcpy(normals_out, S->normals, 24 * n, cudaMemcpyDeviceToHost));
  if (hash_r_out) SBR_CUDA(cudaMemcpy(hash_r_out, S->hash_r, 8 * n, cudaMemcpyDeviceToHost));
  if (hash_f_out) SBR_CUDA(cudaMemcpy(hash_f_out, S->hash_f, 8 * n, cudaMemcpyDeviceToHost));
  return SBR_OK;
}

int sbr_scene_set_attributes(SbrScene* S, const int32_t* tie_rank, const double* normals,
                             const int32_t* matrow, const uint64_t* hash_r,
                             const uint64_t* hash_f) {
  if (!S) return set_error(SBR_ERR_INVALID, "NULL scene");
  DeviceGuard dg(S->device);  // restores the caller's device on return
  const size_t n = (size_t)S->ntri;
  if (tie_rank) SBR_CUDA(cudaMemcpy(S->tie_rank, tie_rank, 4 * n, cudaMemcpyHostToDevice));
  if (normals) SBR_CUDA(cudaMemcpy(S->normals, normals, 24 * n, cudaMemcpyHostToDevice));
  if (matrow) SBR_CUDA(cudaMemcpy(S->matrow, matrow, 4 * n, cudaMemcpyHostToDevice));
  if (hash_r) SBR_CUDA(cudaMemcpy(S->hash_r, hash_r, 8 * n, cudaMemcpyHostToDevice));
  if (hash_f) SBR_CUDA(cudaMemcpy(S->hash_f, hash_f, 8 * n, cudaMemcpyHostToDevice));
  return SBR_OK;
}

int sbr_scene_set_materials(SbrScene* S, const SbrMaterial* mats, int32_t n) {
  if (!S || !mats || n <= 0) return set_error(SBR_ERR_INVALID, "bad material table");
  DeviceGuard dg(S->device);  // restores the caller's device on return
  if (S->mats) SBR_CUDA(cudaFree(S->mats));
  SBR_CUDA(cudaMalloc(&S->mats, sizeof(SbrMaterial) * n));
  SBR_CUDA(cudaMemcpy(S->mats, mats, sizeof(SbrMaterial) * n, cudaMemcpyHostToDevice));
  S->nmat = n;
  S->all_lambertian = 1;
  for (int32_t k = 0; k < n; ++k)
    if (mats[k].pattern_kind != SBR_SCAT_LAMBERTIAN) S->all_lambertian = 0;
  return SBR_OK;
}

int sbr_scene_set_wedges(SbrScene* S, const SbrWedgeTable* W) {
  if (!S || !W) return set_error(SBR_ERR_INVALID, "NULL argument");
  if (W->n_wedges < 0) return set_error(SBR_ERR_INVALID, "bad wedge count");
  DeviceGuard dg(S->device);  // restores the caller's device on return
  if (S->wedge_block) {
    SBR_CUDA(cudaFree(S->wedge_block));
    S->wedge_block = nullptr;
  }
  S->n_wedges = 0;
  const int64_t nw = W->n_wedges, T = S->ntri;
  if (nw == 0) return SBR_OK;
  std::vector<int32_t> off(W->slot_offsets, W->slot_offsets + T + 1);
  const int64_t nids = off[T];
  const size_t b3 = sizeof(double) * 3 * nw, b1 = sizeof(double) * nw;
  const size_t bytes = 5 * b3 + 2 * b1 + 2 * sizeof(uint64_t) * nw + 2 * sizeof(int32_t) * nw +
                       sizeof(int32_t) * (T + 1) + sizeof(int32_t) * (nids > 0 ? nids : 1) + 256;
  SBR_CUDA(cudaMalloc(&S->wedge_block, bytes));
  char* p = (char*)S->wedge_block;
  auto put = [&](const void* src, size_t n) -> const void* {
    void* dst = p;
    if (n) cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    p += (n + 15) & ~(size_t)15;
    return dst;
  };
  S->w_origin = (const double*)put(W->origin, b3);
  S->w_ehat = (const double*)put(W->e_hat, b3);
  S->w_t0 = (const double*)put(W->t0_hat, b3);
  S->w_n0 = (const double*)put(W->n0_hat, b3);
  S->w_nn = (const double*)put(W->nn_hat, b3);
  S->w_len = (const double*)put(W->length, b1);
  S->w_nopen = (const double*)put(W->n_open, b1);
  S->w_hr = (const uint64_t*)put(W->hash_r, sizeof(uint64_t) * nw);
  S->w_hf = (const uint64_t*)put(W->hash_f, sizeof(uint64_t) * nw);
  S->w_mat0 = (const int32_t*)put(W->mat0, sizeof(int32_t) * nw);
  S->w_matn = (const int32_t*)put(W->matn, sizeof(int32_t) * nw);
  S->slot_woff = (const int32_t*)put(W->slot_offsets, sizeof(int32_t) * (T + 1));
  S->slot_wids = (const int32_t*)put(W->slot_ids, sizeof(int32_t) * nids);
  SBR_CUDA(cudaGetLastError());
  S->n_wedges = nw;
  return SBR_OK;
}

int sbr_scene_check(SbrScene* S, void* stream) {
  if (!S) return set_error(SBR_ERR_INVALID, "NULL scene");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned int w = 0;
  SBR_CUDA(cudaMemcpyAsync(&w, S->error_word, sizeof w, cudaMemcpyDeviceToHost, st));
  SBR_CUDA(cudaStreamSynchronize(st));
  SBR_CUDA(cudaGetLastError());
  if (w) {
    SBR_CUDA(cudaMemsetAsync(S->error_word, 0, sizeof(unsigned), st));
    if (w & kErrBounds)
      return set_error(SBR_ERR_INTERNAL, "device bounds check failed (checked build)");
    if (w & kErrStack) return set_error(SBR_ERR_STACK, "BVH traversal stack overflow");
  }
  return SBR_OK;
}

}  // extern "C"
