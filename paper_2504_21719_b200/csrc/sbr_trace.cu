// sbr_trace.cu -- batched ray queries and sampling kernels behind the C ABI.
//
// sbr_trace_closest / sbr_trace_any / sbr_occluded replace the reference's
// Accel.trace_batch / occluded_batch -> _core.trace_closest / trace_any
// (geometry.py:178-201, _core.pyx:115-253); sbr_fibonacci and
// sbr_philox_uniform expose the launch lattice and RNG streams
// (sampling.py:49-95) for parity tests.
#include <string>

#include "sbr_common.cuh"

struct SbrScene;

namespace sbr {
DevScene dev_view(const SbrScene* s);
int set_error(int code, const std::string& msg);
}  // namespace sbr

using namespace sbr;

namespace {

// Batched queries: every warp takes 32 consecutive rays and traces them
// together with the while-while traversals of sbr_common.cuh (grid-stride
// over warp batches, so all lanes reach the warp votes together).
__global__ void __launch_bounds__(128) k_trace_closest(DevScene S, const double* __restrict__ o,
                                                       const double* __restrict__ d, double t_min,
                                                       const double* __restrict__ t_max, int64_t n,
                                                       double* t_out, int64_t* tri_out,
                                                       double* u_out, double* v_out) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  for (int64_t base = wid * 32; base < n; base += warps * 32) {
    const int64_t i = base + (threadIdx.x & 31);
    const bool active = i < n;
    alignas(8) int sn[(SBR_PACKED_STACK ? 2 : 1) * kStackSize];
    float st[SBR_PACKED_STACK ? 1 : kStackSize];
    ClosestTrav T(sn, st);
    if (active) T.start(S, ldg3(o + 3 * i), ldg3(d + 3 * i), t_min, __ldg(t_max + i));
    else T.idle();
    while (!T.done()) T.round(S);
    if (active) {
      if (!T.ok) flag_error(S, kErrStack);
      HitRecord h;
      T.result(h);
      t_out[i] = h.t;
      tri_out[i] = h.tri;
      u_out[i] = h.u;
      v_out[i] = h.v;
    }
  }
}

__global__ void __launch_bounds__(128) k_trace_any(DevScene S, const double* __restrict__ o,
                                                   const double* __restrict__ d, double t_min,
                                                   const double* __restrict__ t_max, int64_t n,
                                                   uint8_t* out) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  for (int64_t base = wid * 32; base < n; base += warps * 32) {
    const int64_t i = base + (threadIdx.x & 31);
    const bool active = i < n;
    int sn[kStackSize];
    AnyTrav T(sn);
    if (active) T.start(S, ldg3(o + 3 * i), ldg3(d + 3 * i), t_min, __ldg(t_max + i));
    else {
      T.idle();
      T.found = false;
      T.ok = true;
    }
    while (!T.done()) T.round(S);
    if (active) {
      if (!T.ok) flag_error(S, kErrStack);
      out[i] = T.found ? 1 : 0;
    }
  }
}

// occluded_batch (geometry.py:187-201): open segment a->b, endpoints offset by eps
__global__ void __launch_bounds__(128) k_occluded(DevScene S, const double* __restrict__ a,
                                                  const double* __restrict__ b, double eps,
                                                  int64_t n, uint8_t* out) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  for (int64_t base = wid * 32; base < n; base += warps * 32) {
    const int64_t i = base + (threadIdx.x & 31);
    bool cast = false;
    int sn[kStackSize];
    AnyTrav T(sn);
    if (i < n) {
      const double3 pa = ldg3(a + 3 * i), pb = ldg3(b + 3 * i);
      const double3 dd = pb - pa;
      const double len = norm_seq(dd);
      if (len > 2.0 * eps) {
        const double3 dn = make_double3(dd.x / len, dd.y / len, dd.z / len);
        T.start(S, make_double3(pa.x + eps * dn.x, pa.y + eps * dn.y, pa.z + eps * dn.z), dn,
                0.0, len - 2.0 * eps);
        cast = true;
      }
    }
    if (!cast) {
      T.idle();
      T.found = false;
      T.ok = true;
    }
    while (!T.done()) T.round(S);
    if (i < n) {
      if (!T.ok) flag_error(S, kErrStack);
      out[i] = T.found ? 1 : 0;
    }
  }
}

__global__ void k_fibonacci(uint64_t N, uint64_t begin, uint64_t end, double* out) {
  for (uint64_t g = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < end;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const double3 v = fibonacci_dir(N, g);
    double* p = out + 3 * (g - begin);
    p[0] = v.x;
    p[1] = v.y;
    p[2] = v.z;
  }
}

__global__ void k_philox(uint64_t seed, uint64_t sample, uint64_t depth, uint64_t tag,
                         uint64_t first, uint64_t count, double* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = philox_uniform(seed, sample, depth, tag, first + i);
}

unsigned grid_1d(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
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

int sbr_trace_closest(const SbrScene* scene, const double* o, const double* d, double t_min,
                      const double* t_max, int64_t n, double* t, int64_t* tri, double* u,
                      double* v, void* stream) {
  if (!scene) return set_error(SBR_ERR_INVALID, "NULL scene");
  if (n <= 0) return SBR_OK;
  k_trace_closest<<<grid_1d(n, 128), 128, 0, (cudaStream_t)stream>>>(dev_view(scene), o, d, t_min,
                                                                    t_max, n, t, tri, u, v);
  return launch_status("k_trace_closest");
}

int sbr_trace_any(const SbrScene* scene, const double* o, const double* d, double t_min,
                  const double* t_max, int64_t n, uint8_t* hit, void* stream) {
  if (!scene) return set_error(SBR_ERR_INVALID, "NULL scene");
  if (n <= 0) return SBR_OK;
  k_trace_any<<<grid_1d(n, 128), 128, 0, (cudaStream_t)stream>>>(dev_view(scene), o, d, t_min,
                                                                t_max, n, hit);
  return launch_status("k_trace_any");
}

int sbr_occluded(const SbrScene* scene, const double* a, const double* b, double eps, int64_t n,
                 uint8_t* out, void* stream) {
  if (!scene) return set_error(SBR_ERR_INVALID, "NULL scene");
  if (n <= 0) return SBR_OK;
  k_occluded<<<grid_1d(n, 128), 128, 0, (cudaStream_t)stream>>>(dev_view(scene), a, b, eps, n,
                                                               out);
  return launch_status("k_occluded");
}

int sbr_fibonacci(uint64_t N, uint64_t begin, uint64_t end, double* out, void* stream) {
  if (N < 1) return set_error(SBR_ERR_INVALID, "need at least one direction");
  if (end > N || begin > end) return set_error(SBR_ERR_INVALID, "bad sample range");
  if (end == begin) return SBR_OK;
  k_fibonacci<<<grid_1d((int64_t)(end - begin), 256), 256, 0, (cudaStream_t)stream>>>(N, begin,
                                                                                    end, out);
  return launch_status("k_fibonacci");
}

int sbr_philox_uniform(uint64_t seed, uint64_t sample, uint64_t depth, uint64_t tag,
                       uint64_t first, uint64_t count, double* out, void* stream) {
  if (count == 0) return SBR_OK;
  k_philox<<<grid_1d((int64_t)count, 256), 256, 0, (cudaStream_t)stream>>>(seed, sample, depth,
                                                                          tag, first, count, out);
  return launch_status("k_philox");
}

}  // extern "C"
