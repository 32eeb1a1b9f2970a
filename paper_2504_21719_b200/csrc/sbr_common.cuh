// sbr_common.cuh -- device-side building blocks shared by the sm_100a kernels.
//
//  * scene layout in HBM (BVH2 nodes with both child boxes, 64 B; float64
//    triangle corners, 80 B per slot)
//  * stateless Philox4x64-10 == numpy Philox + Generator.random
//    (emtrace sampling.py:49-78)
//  * float64 complex arithmetic with numpy's algorithms (division, |z|)
//  * the watertight float64 ray/triangle test of _core.pyx:26-112 and the
//    conservative fp32 child-box test
//
// The library is compiled with -fmad=false so float64 expressions round like
// the reference's numpy / Cython code; FMAs appear only where written
// explicitly (fp32 box tests, emulation of OpenBLAS products).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sbr.h"

namespace sbr {

// ---------------------------------------------------------------------------
// scene layout
// ---------------------------------------------------------------------------
// Internal node: 4 x float4 = 64 B
//   a = (l.lo.x, l.hi.x, l.lo.y, l.hi.y)
//   b = (r.lo.x, r.hi.x, r.lo.y, r.hi.y)
//   c = (l.lo.z, l.hi.z, r.lo.z, r.hi.z)
//   d = (int left, int right, 0, 0)    child >= 0: internal node index
//                                      child <  0: leaf ~((start << 2) | (count-1))
struct alignas(16) BvhNode {
  float4 a, b, c;
  int4 d;
};

__host__ __device__ inline int leaf_encode(int start, int count) {
  return ~((start << 2) | (count - 1));
}
__host__ __device__ inline int leaf_start(int code) { return (~code) >> 2; }
__host__ __device__ inline int leaf_count(int code) { return ((~code) & 3) + 1; }

// Triangle slot: v0.xyz v1.xyz v2.xyz + pad, as 5 double2 (80 B)
struct alignas(16) TriSlot {
  double2 p[5];
};

struct DevScene {
  const BvhNode* nodes;
  const TriSlot* tris;
  const int32_t* tie_rank;     // rank of (object_id, primitive_id)
  const double* normals;       // (T,3)
  const int32_t* matrow;       // material row per slot
  const uint64_t* hash_r;      // plane hash (round quantizer)
  const uint64_t* hash_f;      // plane hash (floor quantizer)
  const SbrMaterial* mats;
  unsigned int* error_word;    // bit0: traversal stack overflow
  int64_t ntri;
  int32_t nnodes;
  int32_t depth;               // levels of the binary tree (root = 1)
  int32_t all_lambertian;      // every material scatters with the Lambertian lobe
  int32_t nmat;
  float pad_base;              // box_setup's pad floor: 2^-62 * (max|coord| + 1)
  double bounds_lo[3], bounds_hi[3];  // scene AABB (float64)
  // diffraction wedges (n_wedges == 0: none)
  int64_t n_wedges;
  const double *w_origin, *w_ehat, *w_t0, *w_n0, *w_nn, *w_len, *w_nopen;
  const uint64_t *w_hr, *w_hf;
  const int32_t *w_mat0, *w_matn, *slot_woff, *slot_wids;
};

// Chunk-cyclic shards (sbr_radiomap_bounce_sharded, sbr_cir_sweep_sharded):
// a shard owns the id chunks (g >> log2) = index, index + count, ...; local
// id l walks them in order; count = 1 is the identity (contiguous ranges).
// Fibonacci ids run pole to pole, so contiguous shards would give one GPU the
// upward rays that escape at once and another the grazing ones.
struct ShardMap {
  uint32_t index, count, log2;
  __device__ __forceinline__ uint64_t gid(uint64_t l) const {
    if (count == 1) return l;
    const uint64_t mask = (1ULL << log2) - 1;
    return (((l >> log2) * count + index) << log2) | (l & mask);
  }
};
// number of ids [0, n) a cyclic shard owns
inline uint64_t shard_size(uint64_t n, uint32_t index, uint32_t count, uint32_t log2) {
  const uint64_t C = 1ULL << log2;
  const uint64_t chunks = (n + C - 1) / C;
  uint64_t m = 0;
  for (uint64_t c = index; c < chunks; c += count) m += (c + 1) * C <= n ? C : n - c * C;
  return m;
}

// Comb order of a launch over sample offsets [0, count): item w -> offset c + k*F (k = w % Q,
// c = w / Q) with F the Fibonacci number nearest sqrt(N): on the Fibonacci
// lattice ids i and i + F are neighbouring directions, so the 32 rays of a
// warp (and, through the queue order, their later bounces) stay coherent.
// Measured on the canyon (N = 1e7): F = 89 / 233 / 987 / 2584 / 4181 ->
// trace 5.9 / 5.2 / 4.5 / 4.2 / 4.2 ms per map.
struct CombMap {
  uint64_t q, stride;  // Q = ceil(count / F) columns, F
  __device__ __forceinline__ uint64_t sample(uint64_t w) const {
    return (w / q) + (w % q) * stride;
  }
  __device__ __forceinline__ uint64_t slots() const { return q * stride; }
};

inline uint64_t comb_stride(uint64_t num_samples) {
  uint64_t a = 1, b = 2, best = 1;
  const double target = sqrt((double)num_samples);
  while (b < (1ULL << 40)) {
    if (fabs((double)b - target) < fabs((double)best - target)) best = b;
    const uint64_t c = a + b;
    a = b;
    b = c;
  }
  return best;
}

// Traversal stack entries (pending far children).  The reference allows 256
// (_core.pyx:15, stack = 2 entries per split); a binary tree needs at most
// its depth, so 256 covers every tree the reference's own build can traverse.
#ifndef SBR_STACK_SIZE
#define SBR_STACK_SIZE 256
#endif
constexpr int kStackSize = SBR_STACK_SIZE;
constexpr unsigned kErrStack = 1u;
// Checked builds (-DSBR_CHECKED, libsbr_checked.so; compute-sanitizer is not
// available on the GPU pool) assert index ranges in the hot kernels: a failed
// check sets kErrBounds in the scene's error word, which sbr_scene_check
// reports as SBR_ERR_INTERNAL.  Release builds compile the checks away.
constexpr unsigned kErrBounds = 2u;
#ifdef SBR_CHECKED
#define SBR_DCHECK(S, cond)                                  \
  do {                                                       \
    if (!(cond)) atomicOr((S).error_word, ::sbr::kErrBounds); \
  } while (0)
#else
#define SBR_DCHECK(S, cond) \
  do {                      \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// Philox4x64-10 keyed stream
// ---------------------------------------------------------------------------
#ifndef SBR_PHILOX_UNROLL
#define SBR_PHILOX_UNROLL 10
#endif
constexpr int kPhiloxUnroll = SBR_PHILOX_UNROLL;
__device__ __forceinline__ double philox_uniform(uint64_t seed, uint64_t sample,
                                                 uint64_t depth, uint64_t tag,
                                                 uint64_t i) {
  uint64_t c0 = i / 4 + 1, c1 = 0, c2 = depth, c3 = tag;
  uint64_t k0 = seed, k1 = sample;
#pragma unroll kPhiloxUnroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  const uint64_t w = (i & 3) == 0 ? c0 : (i & 3) == 1 ? c1 : (i & 3) == 2 ? c2 : c3;
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

// FNV-1a tags of the radio-map streams (sampling.py:42-46)
constexpr uint64_t TAG_MAP_INTERACTION = 0xb89bb7c3608d55f4ULL;
constexpr uint64_t TAG_MAP_RESPAWN = 0x123e3e11a6151f88ULL;
constexpr uint64_t TAG_MAP_PHASE = 0xec7920a818db590bULL;
constexpr uint64_t TAG_MAP_ROULETTE = 0xba18862d049a6e7cULL;

constexpr double kTwoPi = 6.283185307179586;
constexpr double kFourPi = 12.566370614359172;
constexpr double kPi = 3.141592653589793;
constexpr double kGolden = 1.618033988749895;

// Fibonacci lattice direction of global sample g (sampling.py:81-95); the
// azimuth 2*pi*n/golden is formed and range-reduced in float64.
__device__ __forceinline__ double3 fibonacci_dir(uint64_t N, uint64_t g) {
  const double n = (double)((int64_t)g - (int64_t)(N / 2));
  const double cos_t = 2.0 * n / (double)N;
  const double x = 1.0 - cos_t * cos_t;
  const double sin_t = sqrt(x > 0.0 ? x : 0.0);
  const double phi = kTwoPi * n / kGolden;
  double s, c;
  sincos(phi, &s, &c);
  return make_double3(sin_t * c, sin_t * s, cos_t);
}

// ---------------------------------------------------------------------------
// vectors (numpy evaluation orders)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double3 operator+(double3 a, double3 b) {
  return make_double3(a.x + b.x, a.y + b.y, a.z + b.z);
}
__device__ __forceinline__ double3 operator-(double3 a, double3 b) {
  return make_double3(a.x - b.x, a.y - b.y, a.z - b.z);
}
__device__ __forceinline__ double3 operator*(double s, double3 a) {
  return make_double3(s * a.x, s * a.y, s * a.z);
}
__device__ __forceinline__ double3 neg(double3 a) { return make_double3(-a.x, -a.y, -a.z); }
// np.sum(a*b, axis=1): sequential
__device__ __forceinline__ double dot_seq(double3 a, double3 b) {
  return (a.x * b.x + a.y * b.y) + a.z * b.z;
}
// (n,3) @ (3,) through OpenBLAS dgemv (order measured)
__device__ __forceinline__ double dot_gemv(double3 a, double3 b) {
  return fma(a.z, b.z, fma(a.x, b.x, a.y * b.y));
}
// 1-D dot through ddot
__device__ __forceinline__ double dot_ddot(double3 a, double3 b) {
  return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x));
}
__device__ __forceinline__ double3 cross3(double3 a, double3 b) {
  return make_double3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double norm_seq(double3 a) {
  return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z);
}
__device__ __forceinline__ double3 ld3(const double* p) {
  return make_double3(p[0], p[1], p[2]);
}
__device__ __forceinline__ double3 ldg3(const double* p) {
  return make_double3(__ldg(p), __ldg(p + 1), __ldg(p + 2));
}

// ---------------------------------------------------------------------------
// complex128, numpy algorithms
// ---------------------------------------------------------------------------
struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx C(double r, double i) { return cplx{r, i}; }
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return C(a.re + b.re, a.im + b.im); }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return C(a.re - b.re, a.im - b.im); }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
  return C(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
__device__ __forceinline__ cplx operator*(double s, cplx a) { return C(s * a.re, s * a.im); }
// Code size of the complex helpers: every call site of an inlined float64
// division / square root / exp / sincos expands to a few hundred bytes of
// SASS, and the shade kernel called them ~40 times (85 KB of code, far past
// the ~32 KB instruction cache; ncu: "no instruction" was the largest stall).
// SBR_MATH_CALLS = 1 keeps one out-of-line copy of each (a call per use).
#ifndef SBR_MATH_CALLS
#define SBR_MATH_CALLS 1  // config-4 map 749 -> 727 ms; 2 (also cexp_, csqrt_): 742
#endif
#if SBR_MATH_CALLS >= 1
#define SBR_MATH_FN static __device__ __noinline__
#else
#define SBR_MATH_FN __device__ __forceinline__
#endif
#if SBR_MATH_CALLS >= 2
#define SBR_MATH_FN2 static __device__ __noinline__
#else
#define SBR_MATH_FN2 __device__ __forceinline__
#endif
// SBR_DIV_CALLS = 1: the shade kernel's real divisions go through one
// out-of-line copy (an inlined IEEE float64 division is ~20 instructions plus
// a slow-path call at every site)
#ifndef SBR_DIV_CALLS
#define SBR_DIV_CALLS 0
#endif
#if SBR_DIV_CALLS
static __device__ __noinline__ double ddiv_call(double a, double b) { return a / b; }
static __device__ __noinline__ double3 div3_call(double3 v, double s) {
  return make_double3(v.x / s, v.y / s, v.z / s);
}
#define SBR_DIV(a, b) ::sbr::ddiv_call((a), (b))
#define SBR_DIV3(v, s) ::sbr::div3_call((v), (s))
#else
#define SBR_DIV(a, b) ((a) / (b))
#define SBR_DIV3(v, s) make_double3((v).x / (s), (v).y / (s), (v).z / (s))
#endif
// numpy CDOUBLE_divide: Smith's method with a reciprocal
#ifndef SBR_CDIV_INLINE
#define SBR_CDIV_INLINE 0
#endif
#if SBR_CDIV_INLINE
__device__ __forceinline__
#else
SBR_MATH_FN
#endif
cplx cdiv(cplx a, cplx b) {
  const double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return C(a.re / br, a.im / br);
    const double rat = b.im / b.re;
    const double scl = 1.0 / (b.re + b.im * rat);
    return C((a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl);
  }
  const double rat = b.re / b.im;
  const double scl = 1.0 / (b.im + b.re * rat);
  return C((a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl);
}
// a1 / b and a2 / b with one Smith ratio and scale: cdiv's operations on the
// same b, so both results are cdiv's bits, for two of its divisions
struct cplx2 {
  cplx x, y;
};
#ifndef SBR_CDIV2
#define SBR_CDIV2 2  // inlined: config-4 map 632.5 -> 617.4 ms (out of line: 631.4)
#endif
#if SBR_CDIV2 == 2
__device__ __forceinline__
#else
static __device__ __noinline__
#endif
cplx2 cdiv2(cplx a1, cplx a2, cplx b) {
  const double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0)
      return cplx2{C(a1.re / br, a1.im / br), C(a2.re / br, a2.im / br)};
    const double rat = b.im / b.re;
    const double scl = 1.0 / (b.re + b.im * rat);
    return cplx2{C((a1.re + a1.im * rat) * scl, (a1.im - a1.re * rat) * scl),
                 C((a2.re + a2.im * rat) * scl, (a2.im - a2.re * rat) * scl)};
  }
  const double rat = b.re / b.im;
  const double scl = 1.0 / (b.im + b.re * rat);
  return cplx2{C((a1.re * rat + a1.im) * scl, (a1.im * rat - a1.re) * scl),
               C((a2.re * rat + a2.im) * scl, (a2.im * rat - a2.re) * scl)};
}
// np.abs(complex128) in numpy 2.x: max * sqrt(fma(r, r, 1)), r = min/max
#ifndef SBR_CABS_INLINE
#define SBR_CABS_INLINE 0
#endif
#if SBR_CABS_INLINE
__device__ __forceinline__
#else
SBR_MATH_FN
#endif
double cabs_np(cplx a) {
  const double x = fabs(a.re), y = fabs(a.im);
  const double m = fmax(x, y), k = fmin(x, y);
  if (m == 0.0 || isinf(m)) return m + k;
  const double r = k / m;
  return m * sqrt(fma(r, r, 1.0));
}
__device__ __forceinline__ double cabs2(cplx a) {
  const double m = cabs_np(a);
  return m * m;
}
#ifndef SBR_CEXP_CALL
#define SBR_CEXP_CALL 1  // out of line (2 call sites in the Fresnel): c2 shade 3.88 -> 3.83 ms; csqrt_ out of line too: 3.99
#endif
#if SBR_CEXP_CALL
static __device__ __noinline__ cplx cexp_(cplx a) {
#else
SBR_MATH_FN2 cplx cexp_(cplx a) {
#endif
  const double e = exp(a.re);
  double s, c;
  sincos(a.im, &s, &c);
  return C(e * c, e * s);
}
// principal sqrt, glibc csqrt finite branch (np.sqrt(complex) -> libm csqrt)
SBR_MATH_FN2 cplx csqrt_(cplx z) {
  const double x = z.re, y = z.im;
  if (y == 0.0) {
    if (x < 0.0) return C(0.0, copysign(sqrt(-x), y));
    return C(fabs(sqrt(x)), copysign(0.0, y));
  }
  if (x == 0.0) {
    const double r = sqrt(0.5 * fabs(y));
    return C(r, copysign(r, y));
  }
  const double d = hypot(x, y);
  double r, s;
  if (x > 0.0) {
    r = sqrt(0.5 * (d + x));
    s = 0.5 * (y / r);
  } else {
    s = sqrt(0.5 * (d - x));
    r = fabs(0.5 * (y / s));
  }
  return C(r, copysign(s, y));
}

struct cvec3 {
  cplx x, y, z;
};
// sum(field * e, axis=1) with complex field, real e: componentwise sequential
__device__ __forceinline__ cplx cdot_real(const cvec3& f, double3 e) {
  return C((f.x.re * e.x + f.y.re * e.y) + f.z.re * e.z,
           (f.x.im * e.x + f.y.im * e.y) + f.z.im * e.z);
}
__device__ __forceinline__ double field_energy(const cvec3& f) {
  return (cabs2(f.x) + cabs2(f.y)) + cabs2(f.z);
}

// ---------------------------------------------------------------------------
// ray / triangle (float64 watertight shear test, _core.pyx:26-112)
// ---------------------------------------------------------------------------
struct Ray64 {
  double3 o;
  int kx, ky, kz;
  double sx, sy, sz;
  double okx, oky, okz;  // origin components in shear order
};

__device__ __forceinline__ double comp(double3 v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : v.z);
}

__device__ __forceinline__ Ray64 ray_setup(double3 o, double3 d) {
  Ray64 r;
  r.o = o;
  int kz = 0;
  if (fabs(d.y) > fabs(d.x)) kz = 1;
  if (fabs(d.z) > fabs(comp(d, kz))) kz = 2;
  int kx = kz + 1 == 3 ? 0 : kz + 1;
  int ky = kx + 1 == 3 ? 0 : kx + 1;
  const double dkz = comp(d, kz);
  if (dkz < 0.0) {
    const int t = kx;
    kx = ky;
    ky = t;
  }
  r.kx = kx;
  r.ky = ky;
  r.kz = kz;
  r.sx = comp(d, kx) / dkz;
  r.sy = comp(d, ky) / dkz;
  r.sz = 1.0 / dkz;
  r.okx = comp(o, kx);
  r.oky = comp(o, ky);
  r.okz = comp(o, kz);
  return r;
}

// Same test as tri_hit, loading the corners' kx/ky/kz components by index
// (a TriSlot is 9 contiguous doubles v0 v1 v2) instead of selecting them from
// registers: identical arithmetic, ~40 fewer instructions per triangle.
template <bool kUV = true>
__device__ __forceinline__ bool tri_hit_idx(const Ray64& r, const TriSlot* __restrict__ tri,
                                            double t_min, double& t_out, double& u_out,
                                            double& v_out) {
  const double* T = reinterpret_cast<const double*>(tri);
  const double az = __ldg(T + r.kz) - r.okz;
  const double bz = __ldg(T + 3 + r.kz) - r.okz;
  const double cz = __ldg(T + 6 + r.kz) - r.okz;
  const double ax = (__ldg(T + r.kx) - r.okx) - r.sx * az;
  const double ay = (__ldg(T + r.ky) - r.oky) - r.sy * az;
  const double bx = (__ldg(T + 3 + r.kx) - r.okx) - r.sx * bz;
  const double by = (__ldg(T + 3 + r.ky) - r.oky) - r.sy * bz;
  const double cx = (__ldg(T + 6 + r.kx) - r.okx) - r.sx * cz;
  const double cy = (__ldg(T + 6 + r.ky) - r.oky) - r.sy * cz;
  const double u = cx * by - cy * bx;
  const double v = ax * cy - ay * cx;
  const double w = bx * ay - by * ax;
  if ((u < 0.0 || v < 0.0 || w < 0.0) && (u > 0.0 || v > 0.0 || w > 0.0)) return false;
  const double det = u + v + w;
  if (det == 0.0) return false;
  const double t_num = u * (r.sz * az) + v * (r.sz * bz) + w * (r.sz * cz);
  const double t = t_num / det;
  if (!(t > t_min)) return false;
  t_out = t;
  if (kUV) {
    u_out = v / det;
    v_out = w / det;
  }
  return true;
}

// Returns true on a hit with t > t_min; t, u, v as the reference computes them.
__device__ __forceinline__ bool tri_hit(const Ray64& r, const TriSlot* __restrict__ tri,
                                        double t_min, double& t_out, double& u_out,
                                        double& v_out) {
  const double2 q0 = __ldg(&tri->p[0]);
  const double2 q1 = __ldg(&tri->p[1]);
  const double2 q2 = __ldg(&tri->p[2]);
  const double2 q3 = __ldg(&tri->p[3]);
  const double2 q4 = __ldg(&tri->p[4]);
  const double3 a = make_double3(q0.x - r.o.x, q0.y - r.o.y, q1.x - r.o.z);
  const double3 b = make_double3(q1.y - r.o.x, q2.x - r.o.y, q2.y - r.o.z);
  const double3 c = make_double3(q3.x - r.o.x, q3.y - r.o.y, q4.x - r.o.z);
  const double az = comp(a, r.kz), bz = comp(b, r.kz), cz = comp(c, r.kz);
  const double ax = comp(a, r.kx) - r.sx * az, ay = comp(a, r.ky) - r.sy * az;
  const double bx = comp(b, r.kx) - r.sx * bz, by = comp(b, r.ky) - r.sy * bz;
  const double cx = comp(c, r.kx) - r.sx * cz, cy = comp(c, r.ky) - r.sy * cz;
  const double u = cx * by - cy * bx;
  const double v = ax * cy - ay * cx;
  const double w = bx * ay - by * ax;
  if ((u < 0.0 || v < 0.0 || w < 0.0) && (u > 0.0 || v > 0.0 || w > 0.0)) return false;
  const double det = u + v + w;
  if (det == 0.0) return false;
  const double t_num = u * (r.sz * az) + v * (r.sz * bz) + w * (r.sz * cz);
  const double t = t_num / det;
  if (!(t > t_min)) return false;
  t_out = t;
  u_out = v / det;
  v_out = w / det;
  return true;
}

// ---------------------------------------------------------------------------
// conservative fp32 box test
// ---------------------------------------------------------------------------
// Error analysis (d > 0, entry plane lo; the other cases are symmetric).
// ix = fl(1/fl(d)) = (1+a)/d, |a| <= 2^-23; oxp = fl32((o+p)*ix) computed in
// float64, so only its final rounding b (|b| <= 2^-24) is left;
// x0 = fma(lo, ix, -oxp) rounds once more (g, |g| <= 2^-24):
//     x0 = (1+a)(1+g)/d * [(lo - o) - p - (o+p) b].
// With p >= 2^-22 |o| the bracket is <= lo - o, hence x0 <= f(T) where T is
// the exact plane distance and f(t) = t + c|t|, c = 3*2^-24.  Symmetrically
// the exit planes satisfy x >= t - c|t|.  Both maps are monotonic, so the
// computed entry tn <= f(exact tn) and exit tf >= exact tf - c|exact tf|.
// The tests then only need:
//   * tn <= bound: bound_up() inflates by >= 31*2^-24 > c  (no slack on tn);
//   * tn <= tf and the t_min cull: compare against tf2 = tf + 2^-20 |tf|,
//     which is >= f(exact tf) (2^-20 = 16*2^-24 >= 2c plus one rounding).
// So a box holding an exact hit with t_min < t <= best_t is never culled,
// while the pad is 2^-22 |o| instead of a multiple of the scene size: a ray
// leaving a surface no longer re-enters the (flat) boxes around its origin.
// `pad_floor` (scene size * 2^-62) keeps the slab of a direction component of
// exactly +-0 (reciprocal clamped to +-1e20) unbounded across the scene.
struct RayBox {
  float ix, iy, iz;       // fl(1/fl(d)) (clamped to +-1e20)
  float oxp, oyp, ozp;    // fl((o + pad) * ix)  -> lo planes
  float oxm, oym, ozm;    // fl((o - pad) * ix)  -> hi planes
  float tlo;              // t_min rounded down: boxes exited before it hold no hit
};

__device__ __forceinline__ float safe_inv(double d) {
  const float f = (float)d;
  return fabsf(f) > 1e-20f ? 1.0f / f : copysignf(1e20f, f);
}

// `tlo` mirrors the reference's `tf > t_min` box cull (_core.pyx:69): a valid
// hit has t > t_min inside the box, and tf2 >= the exact exit, so culling
// tf2 < rd(t_min) is exact.
__device__ __forceinline__ RayBox box_setup(double3 o, double3 d, float pad_floor,
                                            double t_min) {
  RayBox b;
  // rd(t_min) without the rounding-mode intrinsic: constant-folds for the
  // usual constant t_min (the F2F.RM was re-issued in every node visit)
  float tl = (float)t_min;
  if ((double)tl > t_min) tl = __int_as_float(__float_as_int(tl) - 1);
  b.tlo = t_min > 0.0 ? tl : 0.0f;
  b.ix = safe_inv(d.x);
  b.iy = safe_inv(d.y);
  b.iz = safe_inv(d.z);
#ifdef SBR_PAD_EXPERIMENT  // diagnostics only: scales the (conservative) pad
  const double k = SBR_PAD_EXPERIMENT * 0x1p-22;
#else
  const double k = 0x1p-22;
#endif
  const double px = k * fabs(o.x) + pad_floor;
  const double py = k * fabs(o.y) + pad_floor;
  const double pz = k * fabs(o.z) + pad_floor;
  b.oxp = (float)((o.x + px) * (double)b.ix);
  b.oyp = (float)((o.y + py) * (double)b.iy);
  b.ozp = (float)((o.z + pz) * (double)b.iz);
  b.oxm = (float)((o.x - px) * (double)b.ix);
  b.oym = (float)((o.y - py) * (double)b.iy);
  b.ozm = (float)((o.z - pz) * (double)b.iz);
  return b;
}

// entry distance of [lo,hi] or +inf when missed / beyond `bound`
#ifndef SBR_BOX_FOLD
#define SBR_BOX_FOLD 1  // config-4 map 758 -> 752 ms, config-3 visibility 57.5 -> 56.9 ms
#endif
__device__ __forceinline__ float box_enter(const RayBox& rb, float lox, float hix, float loy,
                                           float hiy, float loz, float hiz, float bound) {
  const float x0 = fmaf(lox, rb.ix, -rb.oxp), x1 = fmaf(hix, rb.ix, -rb.oxm);
  const float y0 = fmaf(loy, rb.iy, -rb.oyp), y1 = fmaf(hiy, rb.iy, -rb.oym);
  const float z0 = fmaf(loz, rb.iz, -rb.ozp), z1 = fmaf(hiz, rb.iz, -rb.ozm);
#if SBR_BOX_FOLD
  // max(tn, tlo) <= min(tf2, bound) is the same test (tlo <= t_min < bound
  // always holds), with the entry clamped to tlo -- still a lower bound of
  // any valid hit in the box, so ordering and stack culling stay exact
  const float tn = fmaxf(fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1)), rb.tlo);
  const float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
  const float tf2 = fminf(fmaf(0x1p-20f, fabsf(tf), tf), bound);
  return tn <= tf2 ? tn : __int_as_float(0x7f800000);
#else
  const float tn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1));
  const float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
  const float tf2 = fmaf(0x1p-20f, fabsf(tf), tf);
  return (tn <= tf2 && tf2 >= rb.tlo && tn <= bound) ? tn : __int_as_float(0x7f800000);
#endif
}

// box_enter as (hit, entry) without the +inf select (the caller branches on
// the predicate directly; same test as SBR_BOX_FOLD box_enter)
__device__ __forceinline__ bool box_hit(const RayBox& rb, float lox, float hix, float loy,
                                        float hiy, float loz, float hiz, float bound,
                                        float& tn_out) {
  const float x0 = fmaf(lox, rb.ix, -rb.oxp), x1 = fmaf(hix, rb.ix, -rb.oxm);
  const float y0 = fmaf(loy, rb.iy, -rb.oyp), y1 = fmaf(hiy, rb.iy, -rb.oym);
  const float z0 = fmaf(loz, rb.iz, -rb.ozp), z1 = fmaf(hiz, rb.iz, -rb.ozm);
  const float tn = fmaxf(fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1)), rb.tlo);
  const float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
  const float tf2 = fminf(fmaf(0x1p-20f, fabsf(tf), tf), bound);
  tn_out = tn;
  return tn <= tf2;
}

// float upper bound of a float64 distance (for comparing fp32 entries)
__device__ __forceinline__ float bound_up(double t) {
  if (!(t < 3.0e38)) return __int_as_float(0x7f800000);
  return __double2float_ru(t) * 1.000002f + 1e-30f;
}

// ---------------------------------------------------------------------------
// closest hit / any hit over the device BVH
// ---------------------------------------------------------------------------
struct HitRecord {
  double t, u, v;
  int tri;  // slot, -1 = miss
};

// Exact reference semantics: minimum over hit triangles of (t, tie_rank) with
// t_min < t < t_max.  Returns false on stack overflow.
__device__ __forceinline__ bool trace_closest(const DevScene& S, double3 o, double3 d,
                                              double t_min, double t_max, HitRecord& h) {
  const Ray64 r = ray_setup(o, d);
  const RayBox rb = box_setup(o, d, S.pad_base, t_min);
  double best_t = t_max, bu = 0.0, bv = 0.0;
  int best = -1, best_rank = 0x7fffffff;
  float bound = bound_up(best_t);
  int stack_node[kStackSize];
  float stack_t[kStackSize];
  int sp = 0;
  int node = 0;
  bool ok = true;
  while (true) {
    if (node >= 0) {
      const BvhNode* nd = S.nodes + node;
      const float4 a = __ldg(&nd->a), b = __ldg(&nd->b), c = __ldg(&nd->c);
      const int4 ch = __ldg(&nd->d);
      const float tl = box_enter(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound);
      const float tr = box_enter(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound);
      const bool hl = tl < __int_as_float(0x7f800000);
      const bool hr = tr < __int_as_float(0x7f800000);
      if (hl && hr) {
        const bool lfirst = tl <= tr;
        const int near = lfirst ? ch.x : ch.y;
        const int far = lfirst ? ch.y : ch.x;
        if (sp >= kStackSize) {
          ok = false;
          break;
        }
        stack_node[sp] = far;
        stack_t[sp] = lfirst ? tr : tl;
        ++sp;
        node = near;
        continue;
      }
      if (hl) {
        node = ch.x;
        continue;
      }
      if (hr) {
        node = ch.y;
        continue;
      }
    } else {
      const int s = leaf_start(node), n = leaf_count(node);
      for (int j = s; j < s + n; ++j) {
        double t, u, v;
        if (tri_hit_idx(r, S.tris + j, t_min, t, u, v)) {
          const int rank = __ldg(S.tie_rank + j);
          if (t < best_t || (t == best_t && best >= 0 && rank < best_rank)) {
            best_t = t;
            best = j;
            best_rank = rank;
            bu = u;
            bv = v;
            bound = bound_up(best_t);
          }
        }
      }
    }
    // pop the next box still in front of the best hit
    bool found = false;
    while (sp > 0) {
      --sp;
      if (stack_t[sp] <= bound) {
        node = stack_node[sp];
        found = true;
        break;
      }
    }
    if (!found) break;
  }
  h.tri = best;
  h.t = best >= 0 ? best_t : __longlong_as_double(0x7ff0000000000000LL);
  h.u = best >= 0 ? bu : 0.0;
  h.v = best >= 0 ? bv : 0.0;
  return ok;
}

// Closest hit, "while-while" form with postponed leaves (Aila & Laine 2009):
// a lane that reaches a leaf parks it and keeps descending inner nodes
// (speculatively, with the bound of before the parked leaf) until every lane
// of the warp holds a leaf, then the warp tests its leaves
// together, so the expensive float64 triangle tests run with most lanes
// active instead of one or two.  Same result as trace_closest (the minimum of
// (t, tie_rank) over all triangles is independent of visiting order; box
// culling is conservative).  Lanes with active == false only vote.
constexpr int kDone = (int)0x80000000;  // never a node index or a leaf code
constexpr int kPending = (int)0x80000001;  // round_u: pop after the parked leaf's test
#ifndef SBR_DEFER_POP
#define SBR_DEFER_POP 1  // config-4 map 660 -> 647 ms, c2 trace 2.85 -> 2.67 ms
#endif

// SBR_PACKED_STACK: a stack entry is one 8-byte (node, entry distance) pair
// (one local load / store per pop / push instead of two); the caller's node
// array then holds 2 * kStackSize ints, 8-byte aligned
#ifndef SBR_PACKED_STACK
#define SBR_PACKED_STACK 1  // config-4 trace 497 -> 491 ms, canyon 4.29 -> 4.21 ms
#endif
__device__ __forceinline__ int ww_pop_t(const int* stack_node, const float* stack_t, int& sp,
                                        float bound, float& t_out) {
  while (sp > 0) {
    --sp;
#if SBR_PACKED_STACK
    const int2 e = reinterpret_cast<const int2*>(stack_node)[sp];
    if (__int_as_float(e.y) <= bound) {
      t_out = __int_as_float(e.y);
      return e.x;
    }
#else
    if (stack_t[sp] <= bound) {
      t_out = stack_t[sp];
      return stack_node[sp];
    }
#endif
  }
  return kDone;
}

#ifndef SBR_ANY_BOX_HIT
#define SBR_ANY_BOX_HIT 1  // config-3 visibility 56.5 -> 55.5 ms
#endif
#ifndef SBR_BOX_HIT
#define SBR_BOX_HIT 1  // (hit, entry) box test in the traversal loops: config-4 map 672 -> 660 ms
#endif
#ifndef SBR_UNI_NOSPEC
#define SBR_UNI_NOSPEC 1  // in the uniform loop speculation no longer pays: config-4 map 682.7 -> 678.7 ms
#endif
// Resumable per-lane closest-hit traversal state.  round() runs one
// inner-node phase + one leaf phase (while-while); done() reports completion.
// kUV = false skips the barycentric (u, v) divisions (radio map, CIR sweep).
template <bool kUV = true>
struct ClosestTravT {
  Ray64 r;
  RayBox rb;
  double t_min, best_t, bu, bv;
  int best, best_rank;
  float bound;
  // The stack lives in the caller's local arrays: a struct holding both the
  // arrays and the scalars stays in local memory as a whole (every sp / node /
  // ray-box access became an LDL/STL); with the arrays outside, the scalars
  // are promoted to registers.
  int* stack_node;
  float* stack_t;
  int sp, node, leaf;
  float node_t, leaf_t;  // entry distances of the current node / parked leaf
  bool ok;

  __device__ __forceinline__ ClosestTravT(int* sn, float* st) : stack_node(sn), stack_t(st) {}
#ifdef SBR_COUNT_VISITS
  unsigned visits, tests;
#endif

  __device__ __forceinline__ void start(const DevScene& S, double3 o, double3 d, double tmin,
                                        double tmax) {
    r = ray_setup(o, d);
    rb = box_setup(o, d, S.pad_base, tmin);
    t_min = tmin;
    best_t = tmax;
    bu = bv = 0.0;
    best = -1;
    best_rank = 0x7fffffff;
    bound = bound_up(best_t);
    sp = 0;
    node = 0;
    leaf = 0;
    node_t = leaf_t = 0.0f;
    ok = true;
#ifdef SBR_COUNT_VISITS
    visits = tests = 0;
#endif
  }
  __device__ __forceinline__ void idle() {
    node = kDone;
    leaf = 0;
  }
  __device__ __forceinline__ bool done() const { return node == kDone && leaf == 0; }

  __device__ __forceinline__ void round(const DevScene& S) {
    // ---- inner nodes (speculative: continue past a parked leaf)
    while (node >= 0) {
#ifdef SBR_COUNT_VISITS
      ++visits;
#endif
      SBR_DCHECK(S, node < S.nnodes);
      const BvhNode* nd = S.nodes + node;
      const float4 a = __ldg(&nd->a), b = __ldg(&nd->b), c = __ldg(&nd->c);
      const int4 ch = __ldg(&nd->d);
      const float tl = box_enter(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound);
      const float tr = box_enter(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound);
      const bool hl = tl < __int_as_float(0x7f800000);
      const bool hr = tr < __int_as_float(0x7f800000);
      if (hl && hr) {
        const bool lfirst = tl <= tr;
        if (sp >= kStackSize) {
          ok = false;
          node = kDone;
          leaf = 0;
          return;
        }
#if SBR_PACKED_STACK
        reinterpret_cast<int2*>(stack_node)[sp] =
            make_int2(lfirst ? ch.y : ch.x, __float_as_int(lfirst ? tr : tl));
#else
        stack_node[sp] = lfirst ? ch.y : ch.x;
        stack_t[sp] = lfirst ? tr : tl;
#endif
        ++sp;
        node = lfirst ? ch.x : ch.y;
        node_t = lfirst ? tl : tr;
      } else if (hl) {
        node = ch.x;
        node_t = tl;
      } else if (hr) {
        node = ch.y;
        node_t = tr;
      } else {
        node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
      }
      if (node < 0 && node != kDone && leaf == 0) {
        leaf = node;
        leaf_t = node_t;
        node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
#ifdef SBR_NO_SPECULATE
        break;  // A/B switch: with register-resident state speculation wins ~2 %
#endif
      }
      if (!__any_sync(__activemask(), leaf == 0)) break;
    }
    // ---- leaves
    while (leaf < 0) {
      const int s = leaf_start(leaf);
      // a parked leaf beyond the best hit found since parking is culled
      const int n = leaf_t <= bound ? leaf_count(leaf) : 0;
      SBR_DCHECK(S, s >= 0 && s + leaf_count(leaf) <= S.ntri);
#ifdef SBR_COUNT_VISITS
      tests += n;
#endif
      for (int j = s; j < s + n; ++j) {
        double t, u, v;
        u = v = 0.0;
        if (tri_hit_idx<kUV>(r, S.tris + j, t_min, t, u, v)) {
          const int rank = __ldg(S.tie_rank + j);
          if (t < best_t || (t == best_t && best >= 0 && rank < best_rank)) {
            best_t = t;
            best = j;
            best_rank = rank;
            bu = u;
            bv = v;
            bound = bound_up(best_t);
          }
        }
      }
      leaf = 0;
      if (node < 0 && node != kDone) {
        leaf = node;
        leaf_t = node_t;
        node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
      }
      if (!__any_sync(__activemask(), leaf < 0)) break;
    }
  }

  // Warp-uniform form of round(): EVERY lane of the warp calls it (finished
  // lanes idle inside, predicated off), so the loop votes use the full mask
  // (no active-mask / divergence bookkeeping per iteration).  kCheck = false
  // drops the per-push overflow test: valid when the tree is shallower than
  // the stack (a depth-first stack holds at most one entry per level).
  template <bool kCheck>
  __device__ __forceinline__ void round_u(const DevScene& S) {
    while (true) {
#if SBR_UNI_NOSPEC
      const bool act = node >= 0 && leaf == 0;  // no speculative descent past a parked leaf
#else
      const bool act = node >= 0;
#endif
      if (act) {
        SBR_DCHECK(S, node < S.nnodes);
        const BvhNode* nd = S.nodes + node;
        const float4 a = __ldg(&nd->a), b = __ldg(&nd->b), c = __ldg(&nd->c);
        const int4 ch = __ldg(&nd->d);
#if SBR_BOX_HIT && SBR_BOX_FOLD
        float tl, tr;
        const bool hl = box_hit(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound, tl);
        const bool hr = box_hit(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound, tr);
#else
        const float tl = box_enter(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound);
        const float tr = box_enter(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound);
        const bool hl = tl < __int_as_float(0x7f800000);
        const bool hr = tr < __int_as_float(0x7f800000);
#endif
        if (hl && hr) {
          const bool lfirst = tl <= tr;
          if (kCheck && sp >= kStackSize) {
            ok = false;
            node = kDone;
            leaf = 0;
          } else {
            SBR_DCHECK(S, sp < kStackSize);
#if SBR_PACKED_STACK
            reinterpret_cast<int2*>(stack_node)[sp] =
                make_int2(lfirst ? ch.y : ch.x, __float_as_int(lfirst ? tr : tl));
#else
            stack_node[sp] = lfirst ? ch.y : ch.x;
            stack_t[sp] = lfirst ? tr : tl;
#endif
            ++sp;
            node = lfirst ? ch.x : ch.y;
            node_t = lfirst ? tl : tr;
          }
        } else if (hl) {
          node = ch.x;
          node_t = tl;
        } else if (hr) {
          node = ch.y;
          node_t = tr;
        } else {
          node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
        }
        if (node < 0 && node != kDone && leaf == 0) {
          leaf = node;
          leaf_t = node_t;
#if SBR_DEFER_POP
          node = kPending;  // popped after the leaf test, with its tighter bound
#else
          node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
#endif
        }
      }
      if (!__any_sync(0xffffffffu, act && leaf == 0)) break;
    }
    while (true) {
      const bool has = leaf < 0;
      if (has) {
        const int s = leaf_start(leaf);
        const int n = leaf_t <= bound ? leaf_count(leaf) : 0;
        SBR_DCHECK(S, s >= 0 && s + leaf_count(leaf) <= S.ntri);
        for (int j = s; j < s + n; ++j) {
          double t, u, v;
          u = v = 0.0;
          if (tri_hit_idx<kUV>(r, S.tris + j, t_min, t, u, v)) {
            const int rank = __ldg(S.tie_rank + j);
            if (t < best_t || (t == best_t && best >= 0 && rank < best_rank)) {
              best_t = t;
              best = j;
              best_rank = rank;
              bu = u;
              bv = v;
              bound = bound_up(best_t);
            }
          }
        }
        leaf = 0;
#if SBR_DEFER_POP
        if (node == kPending) node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
#endif
        if (node < 0 && node != kDone) {
          leaf = node;
          leaf_t = node_t;
#if SBR_DEFER_POP
          node = kPending;
#else
          node = ww_pop_t(stack_node, stack_t, sp, bound, node_t);
#endif
        }
      }
      if (!__any_sync(0xffffffffu, has && leaf < 0)) break;
    }
  }

  __device__ __forceinline__ void result(HitRecord& h) const {
    h.tri = best;
    h.t = best >= 0 ? best_t : __longlong_as_double(0x7ff0000000000000LL);
    h.u = best >= 0 ? bu : 0.0;
    h.v = best >= 0 ? bv : 0.0;
  }
};

// Resumable per-lane any-hit traversal (occlusion), while-while with parked
// leaves like ClosestTrav; stops at the first triangle with t_min < t < limit.
#ifndef SBR_ANY_ORDER
#define SBR_ANY_ORDER 0
#endif
struct AnyTrav {
  Ray64 r;
  RayBox rb;
  double t_min, limit;
  float bound;
  int* stack_node;  // caller's local array (see ClosestTravT)
  int sp, node, leaf;
  int hit_tri;  // the occluding slot once found
  bool ok, found;

  __device__ __forceinline__ explicit AnyTrav(int* sn) : stack_node(sn) {}

  __device__ __forceinline__ void start(const DevScene& S, double3 o, double3 d, double tmin,
                                        double lim) {
    r = ray_setup(o, d);
    rb = box_setup(o, d, S.pad_base, tmin);
    t_min = tmin;
    limit = lim;
    bound = bound_up(lim);
    sp = 0;
    node = 0;
    leaf = 0;
    hit_tri = -1;
    ok = true;
    found = false;
  }
  // Test one candidate occluder (e.g. found by a neighbouring ray): the same
  // predicate the traversal applies, so the answer is unchanged -- any
  // triangle with t_min < t < limit occludes.
  __device__ __forceinline__ bool try_occluder(const DevScene& S, int j) {
    SBR_DCHECK(S, j >= 0 && j < S.ntri);
    double t, u, v;
    if (tri_hit_idx<false>(r, S.tris + j, t_min, t, u, v) && t < limit) {
      found = true;
      hit_tri = j;
      node = kDone;
      leaf = 0;
      return true;
    }
    return false;
  }
  __device__ __forceinline__ void idle() {
    node = kDone;
    leaf = 0;
  }
  __device__ __forceinline__ bool done() const { return node == kDone && leaf == 0; }
  __device__ __forceinline__ int pop() { return sp > 0 ? stack_node[--sp] : kDone; }

  __device__ __forceinline__ void round(const DevScene& S) {
    while (node >= 0) {
      SBR_DCHECK(S, node < S.nnodes);
      const BvhNode* nd = S.nodes + node;
      const float4 a = __ldg(&nd->a), b = __ldg(&nd->b), c = __ldg(&nd->c);
      const int4 ch = __ldg(&nd->d);
#if SBR_ANY_BOX_HIT && SBR_BOX_FOLD
      float tl, tr;
      const bool hl = box_hit(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound, tl);
      const bool hr = box_hit(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound, tr);
#else
      const float tl = box_enter(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound);
      const float tr = box_enter(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound);
      const bool hl = tl < __int_as_float(0x7f800000);
      const bool hr = tr < __int_as_float(0x7f800000);
#endif
      if (hl && hr) {
        if (sp >= kStackSize) {
          ok = false;
          node = kDone;
          leaf = 0;
          return;
        }
        // far child first: any hit ends the search and there is no bound to
        // shrink, so near-first only walks the crowded boxes around the ray's
        // origin (the surface a CIR vertex lies on) before reaching the
        // occluders.  Config-3 visibility: near-first 126 ms, fixed order
        // 107, nearest-to-midpoint 99, far-first 93 (identical results)
#if SBR_ANY_ORDER == 0
        const bool lfirst = tl > tr;   // far first
#elif SBR_ANY_ORDER == 1
        const bool lfirst = tl <= tr;  // near first
#else
        const bool lfirst = true;      // fixed
#endif
        stack_node[sp++] = lfirst ? ch.y : ch.x;
        node = lfirst ? ch.x : ch.y;
      } else if (hl) {
        node = ch.x;
      } else if (hr) {
        node = ch.y;
      } else {
        node = pop();
      }
      if (node < 0 && node != kDone && leaf == 0) {
        leaf = node;
        node = pop();
      }
      if (!__any_sync(__activemask(), leaf == 0)) break;
    }
    while (leaf < 0) {
      const int s = leaf_start(leaf), n = leaf_count(leaf);
      SBR_DCHECK(S, s >= 0 && s + n <= S.ntri);
      for (int j = s; j < s + n; ++j) {
        double t, u, v;
        if (tri_hit_idx<false>(r, S.tris + j, t_min, t, u, v) && t < limit) {
          found = true;
          hit_tri = j;
          node = kDone;
          leaf = 0;
          return;
        }
      }
      leaf = 0;
      if (node < 0 && node != kDone) {
        leaf = node;
        node = pop();
      }
      if (!__any_sync(__activemask(), leaf < 0)) break;
    }
  }
};

using ClosestTrav = ClosestTravT<true>;

// any hit with t_min < t < limit (_core.pyx:198-253); returns false on overflow
__device__ __forceinline__ bool trace_any(const DevScene& S, double3 o, double3 d,
                                          double t_min, double limit, bool& found) {
  const Ray64 r = ray_setup(o, d);
  const RayBox rb = box_setup(o, d, S.pad_base, t_min);
  const float bound = bound_up(limit);
  int stack_node[kStackSize];
  int sp = 0;
  int node = 0;
  found = false;
  while (true) {
    if (node >= 0) {
      const BvhNode* nd = S.nodes + node;
      const float4 a = __ldg(&nd->a), b = __ldg(&nd->b), c = __ldg(&nd->c);
      const int4 ch = __ldg(&nd->d);
      const float tl = box_enter(rb, a.x, a.y, a.z, a.w, c.x, c.y, bound);
      const float tr = box_enter(rb, b.x, b.y, b.z, b.w, c.z, c.w, bound);
      const bool hl = tl < __int_as_float(0x7f800000);
      const bool hr = tr < __int_as_float(0x7f800000);
      if (hl && hr) {
        if (sp >= kStackSize) return false;
        const bool lfirst = tl > tr;  // far child first, like AnyTrav
        stack_node[sp++] = lfirst ? ch.y : ch.x;
        node = lfirst ? ch.x : ch.y;
        continue;
      }
      if (hl) {
        node = ch.x;
        continue;
      }
      if (hr) {
        node = ch.y;
        continue;
      }
    } else {
      const int s = leaf_start(node), n = leaf_count(node);
      for (int j = s; j < s + n; ++j) {
        double t, u, v;
        if (tri_hit_idx(r, S.tris + j, t_min, t, u, v) && t < limit) {
          found = true;
          return true;
        }
      }
    }
    if (sp == 0) break;
    node = stack_node[--sp];
  }
  return true;
}

__device__ __forceinline__ void flag_error(const DevScene& S, unsigned bits) {
  atomicOr(S.error_word, bits);
}

// occluded_batch for one segment (geometry.py:187-201)
__device__ __forceinline__ bool occluded_segment(const DevScene& S, double3 a, double3 b,
                                                 double eps, bool& ok) {
  const double3 d = b - a;
  const double len = norm_seq(d);
  ok = true;
  if (!(len > 2.0 * eps)) return false;
  const double3 dn = make_double3(d.x / len, d.y / len, d.z / len);
  const double3 o = make_double3(a.x + eps * dn.x, a.y + eps * dn.y, a.z + eps * dn.z);
  bool found;
  ok = trace_any(S, o, dn, 0.0, len - 2.0 * eps, found);
  return found;
}

// kernel-launch evidence counter (host side, defined in sbr_scene.cu)
void count_launch();
// stream-ordered scratch from the library's own memory pool on the current
// device (sbr_scene.cu): never the device's default pool, so the process's
// other allocators are unaffected; freed blocks stay mapped up to a finite
// release threshold and sbr_release_scratch() trims the pool to zero
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
// optional CUDA-event timing of individual launches (sbr_profile_enable)
void prof_begin(void* stream, const char* name);
void prof_end(void* stream);

}  // namespace sbr
