// sbr_wedges.cu -- diffraction wedge extraction on the GPU (scene ingestion).
//
// Replaces emtrace geometry.py:356-494 (extract_wedges, _edge_records,
// _merge_segments) and the per-wedge edge hashes of paths.py:111-125 /
// 457-475.  Same result as the reference:
//   * every triangle edge (mesh, prim, local) with endpoints quantised to
//     1e-9 (round half to even, like Python's round) and keyed by the sorted
//     endpoint pair; edges owned by one face become screens (n = 2), edges
//     owned by exactly two faces wedges when non-coplanar beyond the threshold
//     and convex on the material side (exterior angle n pi, n in (1, 2));
//     reflex edges and edges of > 2 faces are ignored;
//   * collinear segments with equal (sorted) face planes merge into one wedge
//     (line / plane keys quantised to 1e-6), the segment of the first owner
//     (o, m) is the reference for the frame, owner sides flip where the
//     planes are the reference's reversed, extents are the min / max of the
//     endpoint projections;
//   * wedges ordered by their first owner (o, m, local).
// Pipeline: per-edge keys -> stable LSD radix sort over the 6 int64 key
// columns (CUB) -> run boundaries -> per-run segment frames -> sort of the
// segments by their 14-column merge key and by (group, first owner) -> one
// thread per merged group (extents, sorted unique owner lists) -> sort of the
// wedges by first owner -> edge hashes.  The frame arithmetic follows the
// reference's numpy expressions in float64 (-fmad=false); arccos is CUDA's
// (the reference uses the platform libm), so n and the frames agree to ~1 ulp.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <array>
#include <climits>
#include <string>
#include <vector>

#include "sbr_common.cuh"

namespace sbr {
int set_error(int code, const std::string& msg);
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
}  // namespace sbr

using namespace sbr;

struct SbrWedgeSet {
  int64_t n_wedges = 0, n_owners0 = 0, n_ownersn = 0;
  std::vector<double> origin, e_hat, t0_hat, n0_hat, nn_hat, length, n_open;
  std::vector<uint64_t> hash_r, hash_f;
  std::vector<int64_t> off0, offn;          // (nw + 1) CSR offsets of the owner lists
  std::vector<int64_t> own0, ownn;          // triangle index (input order) * 3 + local
};

namespace {

constexpr int kKeyCols = 6;    // edge key: quantised endpoints (a, b), lexicographic
constexpr int kMergeCols = 14; // line key (6) + sorted plane keys (4 + 4)

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

__device__ __forceinline__ int64_t qkey(double x, double res) { return (int64_t)rint(x / res); }

__device__ __forceinline__ double3 ld3d(const double* p) { return make_double3(p[0], p[1], p[2]); }
__device__ __forceinline__ void st3(double* p, double3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
__device__ __forceinline__ double3 unit3(double3 v) {
  const double n = sqrt((v.x * v.x + v.y * v.y) + v.z * v.z);  // np.linalg.norm
  return make_double3(v.x / n, v.y / n, v.z / n);
}

// lexicographic comparison of int64 rows
__device__ __forceinline__ bool lex_less(const int64_t* a, const int64_t* b, int n) {
  for (int k = 0; k < n; ++k)
    if (a[k] != b[k]) return a[k] < b[k];
  return false;
}
__device__ __forceinline__ bool rows_equal(const int64_t* a, const int64_t* b, int n) {
  for (int k = 0; k < n; ++k)
    if (a[k] != b[k]) return false;
  return true;
}

// canonical sign: first component with |c| > eps positive (geometry.py _plane_key / _line_key)
__device__ __forceinline__ double3 canonical(double3 v) {
  const double c = fabs(v.x) > 1e-12 ? v.x : (fabs(v.y) > 1e-12 ? v.y : (fabs(v.z) > 1e-12 ? v.z : 0.0));
  return c < 0.0 ? make_double3(-v.x, -v.y, -v.z) : v;
}
__device__ __forceinline__ void plane_key(double3 n, double3 p, int64_t* out) {
  const double3 c = canonical(n);
  const double d = (c.x * p.x + c.y * p.y) + c.z * p.z;
  out[0] = qkey(c.x, 1e-6);
  out[1] = qkey(c.y, 1e-6);
  out[2] = qkey(c.z, 1e-6);
  out[3] = qkey(d, 1e-6);
}
__device__ __forceinline__ void line_key(double3 dir, double3 p, int64_t* out) {
  const double3 c = canonical(dir);
  const double pd = (p.x * c.x + p.y * c.y) + p.z * c.z;
  const double3 anchor = make_double3(p.x - pd * c.x, p.y - pd * c.y, p.z - pd * c.z);
  out[0] = qkey(c.x, 1e-6);
  out[1] = qkey(c.y, 1e-6);
  out[2] = qkey(c.z, 1e-6);
  out[3] = qkey(anchor.x, 1e-6);
  out[4] = qkey(anchor.y, 1e-6);
  out[5] = qkey(anchor.z, 1e-6);
}

// ---- stage 1: per-edge keys (edge e = 3 * triangle + local, insertion order)
__global__ void k_edge_keys(const double* __restrict__ v0, const double* __restrict__ v1,
                            const double* __restrict__ v2, int64_t ne, int64_t* __restrict__ key,
                            uint8_t* __restrict__ live) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / 3;
    const int l = (int)(e % 3);
    const double* c[3] = {v0 + 3 * t, v1 + 3 * t, v2 + 3 * t};
    const double* pa = c[l];
    const double* pb = c[(l + 1) % 3];
    int64_t ka[3], kb[3];
    for (int k = 0; k < 3; ++k) {
      ka[k] = qkey(pa[k], 1e-9);
      kb[k] = qkey(pb[k], 1e-9);
    }
    const bool same = ka[0] == kb[0] && ka[1] == kb[1] && ka[2] == kb[2];
    live[e] = same ? 0 : 1;
    const bool a_first = lex_less(ka, kb, 3);
    int64_t* out = key + kKeyCols * e;
    for (int k = 0; k < 3; ++k) {
      out[k] = a_first ? ka[k] : kb[k];
      out[3 + k] = a_first ? kb[k] : ka[k];
    }
  }
}

// column c of the rows in the current order, as order-preserving unsigned keys
__global__ void k_gather_col(const int64_t* __restrict__ rows, int ncols, int col,
                             const int32_t* __restrict__ perm, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint64_t)rows[(int64_t)perm[i] * ncols + col] ^ 0x8000000000000000ULL;
}

__global__ void k_iota32(int32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

// ---- stage 2: run boundaries of the sorted edge keys (live edges only)
// a run starts where the first `ncols` columns of consecutive sorted rows (row
// stride `stride`) differ; dead edges (live == 0, degenerate) form their own
// runs, which the segment stage skips
__global__ void k_run_flags(const int64_t* __restrict__ key, const int32_t* __restrict__ perm,
                            const uint8_t* __restrict__ live, int64_t n, int stride, int ncols,
                            int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = perm[i];
    flag[i] = i == 0 || (live && live[e] != live[perm[i - 1]]) ||
              !rows_equal(key + (int64_t)e * stride, key + (int64_t)perm[i - 1] * stride, ncols);
  }
}

struct EdgeIn {
  const double *v0, *v1, *v2;     // input-order corners (T, 3)
  const int64_t *obj, *prim;      // input-order ids
};

// Mesh.triangle_normals (geometry.py:66-69): normalize(cross(b - a, c - a))
__device__ __forceinline__ double3 face_normal(const EdgeIn& E, int64_t t) {
  const double3 a = ld3d(E.v0 + 3 * t), b = ld3d(E.v1 + 3 * t), c = ld3d(E.v2 + 3 * t);
  return unit3(cross3(b - a, c - a));
}

struct Segs {  // segment SoA, capacity = number of runs
  int64_t* line;   // (n, 6)
  int64_t* p0;     // (n, 4)
  int64_t* pn;     // (n, 4)
  double *pa, *pb, *e, *n0, *nn, *t0;  // (n, 3)
  double* nopen;
  int64_t *own0, *ownn;  // edge index 3 * t + local, -1 = none
  int64_t *o0, *m0;      // (o, m) of own0 (sort keys)
};

// kind of each run: 1 screen, 2 wedge, 0 nothing; segment data at the run's index
__global__ void k_run_segments(EdgeIn E, const int32_t* __restrict__ perm,
                               const uint8_t* __restrict__ live,
                               const int32_t* __restrict__ run_start, int64_t nruns, int64_t n,
                               double thresh, int8_t* __restrict__ kind, Segs S) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = run_start[r];
    const int64_t cnt = (r + 1 < nruns ? run_start[r + 1] : n) - s;
    kind[r] = 0;
    if (cnt > 2 || !live[perm[s]]) continue;  // > 2 faces, or a degenerate edge
    const int64_t ea = perm[s];
    const int64_t ta = ea / 3;
    const int la = (int)(ea % 3);
    const double* ca[3] = {E.v0 + 3 * ta, E.v1 + 3 * ta, E.v2 + 3 * ta};
    if (cnt == 1) {
      const double3 pa = ld3d(ca[la]), pb = ld3d(ca[(la + 1) % 3]);
      const double3 n = face_normal(E, ta);
      const double3 e = unit3(pb - pa);  // winding order: n0 x e points into the face
      line_key(e, pa, S.line + 6 * r);
      plane_key(n, pa, S.p0 + 4 * r);
      plane_key(n, pa, S.pn + 4 * r);
      st3(S.pa + 3 * r, pa);
      st3(S.pb + 3 * r, pb);
      st3(S.e + 3 * r, e);
      st3(S.n0 + 3 * r, n);
      st3(S.nn + 3 * r, neg(n));
      st3(S.t0 + 3 * r, cross3(n, e));
      S.nopen[r] = 2.0;
      S.own0[r] = ea;
      S.ownn[r] = -1;
      S.o0[r] = E.obj[ta];
      S.m0[r] = E.prim[ta];
      kind[r] = 1;
      continue;
    }
    int64_t eb = perm[s + 1];
    int64_t tb = eb / 3;
    // fa, fb = sorted(owners, key=(object_id, primitive_id)) (stable)
    int64_t fa = ea, fb = eb;
    if (E.obj[tb] < E.obj[ta] || (E.obj[tb] == E.obj[ta] && E.prim[tb] < E.prim[ta])) {
      fa = eb;
      fb = ea;
    }
    const int64_t tfa = fa / 3, tfb = fb / 3;
    const int lfa = (int)(fa % 3), lfb = (int)(fb % 3);
    const double* cfa[3] = {E.v0 + 3 * tfa, E.v1 + 3 * tfa, E.v2 + 3 * tfa};
    const double* cfb[3] = {E.v0 + 3 * tfb, E.v1 + 3 * tfb, E.v2 + 3 * tfb};
    const double3 na = face_normal(E, tfa), nb = face_normal(E, tfb);
    const double3 cn = cross3(na, nb);
    const double sn = sqrt((cn.x * cn.x + cn.y * cn.y) + cn.z * cn.z);
    double cosang = (na.x * nb.x + na.y * nb.y) + na.z * nb.z;
    cosang = cosang < -1.0 ? -1.0 : (cosang > 1.0 ? 1.0 : cosang);
    if (acos(cosang) <= thresh || sn < 1e-12) continue;
    const double3 pa = ld3d(cfa[lfa]), pb = ld3d(cfa[(lfa + 1) % 3]);
    const double3 eg = unit3(pb - pa);
    // _in_face_tangent(e_geo, pa, far)
    double3 ut[2];
    const double3 far[2] = {ld3d(cfa[(lfa + 2) % 3]), ld3d(cfb[(lfb + 2) % 3])};
    for (int q = 0; q < 2; ++q) {
      double3 u = far[q] - pa;
      const double ue = (u.x * eg.x + u.y * eg.y) + u.z * eg.z;
      u = make_double3(u.x - ue * eg.x, u.y - ue * eg.y, u.z - ue * eg.z);
      const double nu = sqrt((u.x * u.x + u.y * u.y) + u.z * u.z);
      ut[q] = nu > 0.0 ? make_double3(u.x / nu, u.y / nu, u.z / nu) : u;
    }
    if ((ut[1].x * na.x + ut[1].y * na.y) + ut[1].z * na.z > 0.0) continue;  // reflex
    double cu = (ut[0].x * ut[1].x + ut[0].y * ut[1].y) + ut[0].z * ut[1].z;
    cu = cu < -1.0 ? -1.0 : (cu > 1.0 ? 1.0 : cu);
    const double theta = acos(cu);
    const double nopen = 2.0 - theta / kPi;
    const double3 ch = make_double3(cn.x / sn, cn.y / sn, cn.z / sn);
    const bool fwd = (ch.x * eg.x + ch.y * eg.y) + ch.z * eg.z >= 0.0;
    const double3 e = fwd ? ch : neg(ch);
    const double3 n0 = fwd ? na : nb, nn = fwd ? nb : na;
    const int64_t f0 = fwd ? fa : fb, fn = fwd ? fb : fa;
    line_key(e, pa, S.line + 6 * r);
    plane_key(n0, pa, S.p0 + 4 * r);
    plane_key(nn, pa, S.pn + 4 * r);
    st3(S.pa + 3 * r, pa);
    st3(S.pb + 3 * r, pb);
    st3(S.e + 3 * r, e);
    st3(S.n0 + 3 * r, n0);
    st3(S.nn + 3 * r, nn);
    st3(S.t0 + 3 * r, cross3(n0, e));
    S.nopen[r] = nopen;
    S.own0[r] = f0;
    S.ownn[r] = fn;
    S.o0[r] = E.obj[f0 / 3];
    S.m0[r] = E.prim[f0 / 3];
    kind[r] = 2;
  }
}

// segment order: screens (run order) then wedges (run order), as the reference's
// numpy restatement concatenates them; pos = exclusive scans of the two flags
__global__ void k_seg_flags(const int8_t* __restrict__ kind, int64_t nruns, int32_t* fs,
                            int32_t* fw) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (int64_t)gridDim.x * blockDim.x) {
    fs[r] = kind[r] == 1;
    fw[r] = kind[r] == 2;
  }
}

__global__ void k_seg_order(const int8_t* __restrict__ kind, const int32_t* __restrict__ ps,
                            const int32_t* __restrict__ pw, int64_t nruns, int64_t n_screens,
                            int32_t* __restrict__ seg_run) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (kind[r] == 1) seg_run[ps[r]] = (int32_t)r;
    else if (kind[r] == 2) seg_run[n_screens + pw[r]] = (int32_t)r;
  }
}

// merge key of segment s (row-major (nseg, 14)) and its secondary sort columns
__global__ void k_merge_keys(Segs S, const int32_t* __restrict__ seg_run, int64_t nseg,
                             int64_t* __restrict__ mkey) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = seg_run[s];
    int64_t* out = mkey + kMergeCols * s;
    for (int k = 0; k < 6; ++k) out[k] = S.line[6 * r + k];
    const int64_t* p0 = S.p0 + 4 * r;
    const int64_t* pn = S.pn + 4 * r;
    const bool pn_first = lex_less(pn, p0, 4);   // tuple(sorted(planes))
    for (int k = 0; k < 4; ++k) {
      out[6 + k] = pn_first ? pn[k] : p0[k];
      out[10 + k] = pn_first ? p0[k] : pn[k];
    }
  }
}

// (group id, o, m, segment) rows for the within-group order
__global__ void k_group_rows(const int32_t* __restrict__ perm, const int32_t* __restrict__ gid_sorted,
                             Segs S, const int32_t* __restrict__ seg_run, int64_t nseg,
                             int64_t* __restrict__ rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = perm[i];
    const int64_t r = seg_run[s];
    int64_t* out = rows + 4 * s;
    out[0] = gid_sorted[i];
    out[1] = S.o0[r];
    out[2] = S.m0[r];
    out[3] = s;
  }
}

// group of every position of the (group, first owner)-sorted segment order
__global__ void k_pos_group(const int32_t* __restrict__ gstart, int64_t ngroups, int64_t nseg,
                            int32_t* __restrict__ pos_group) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g + 1 < ngroups ? gstart[g + 1] : nseg;
    for (int64_t i = gstart[g]; i < b; ++i) pos_group[i] = (int32_t)g;
  }
}

// per segment (sorted position i): owner sides relative to its group's
// reference segment (_merge_segments flip rule) as contribution rows
// (group, side, o, m, local, code), and the endpoint projections
// (p - p_ref) @ e_hat of the reference frame
__global__ void k_seg_contrib(Segs S, const int32_t* __restrict__ seg_run,
                              const int32_t* __restrict__ order, const int32_t* __restrict__ gstart,
                              const int32_t* __restrict__ pos_group, int64_t nseg, EdgeIn E,
                              int64_t* __restrict__ contrib, double* __restrict__ xlo,
                              double* __restrict__ xhi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int g = pos_group[i];
    const int64_t rr = seg_run[order[gstart[g]]];
    const int64_t r = seg_run[order[i]];
    const int64_t* p0 = S.p0 + 4 * r;
    const int64_t* pn = S.pn + 4 * r;
    const int64_t* p0r = S.p0 + 4 * rr;
    const int64_t* pnr = S.pn + 4 * rr;
    const bool same = rows_equal(p0, p0r, 4) && rows_equal(pn, pnr, 4);
    const bool rev = rows_equal(pn, p0r, 4) && rows_equal(p0, pnr, 4);
    const bool flip = !same && rev && !rows_equal(p0, pn, 4);
    const int64_t src[2] = {flip ? S.ownn[r] : S.own0[r], flip ? S.own0[r] : S.ownn[r]};
    for (int q = 0; q < 2; ++q) {
      int64_t* row = contrib + 6 * (2 * i + q);
      if (src[q] < 0) {
        row[0] = -1;  // no owner on this side: sorts first, dropped
        row[1] = row[2] = row[3] = row[4] = row[5] = -1;
        continue;
      }
      const int64_t t = src[q] / 3;
      row[0] = g;
      row[1] = q;
      row[2] = E.obj[t];
      row[3] = E.prim[t];
      row[4] = src[q] % 3;
      row[5] = src[q];
    }
    const double3 e = ld3d(S.e + 3 * rr), pref = ld3d(S.pa + 3 * rr);
    const double xa = dot_ddot(ld3d(S.pa + 3 * r) - pref, e);
    const double xb = dot_ddot(ld3d(S.pb + 3 * r) - pref, e);
    xlo[i] = fmin(xa, xb);
    xhi[i] = fmax(xa, xb);
  }
}

// per merged group: the reference segment's frame and the extents
struct WedgeOut {
  double *origin, *e, *t0, *n0, *nn, *len, *nopen;
};

__global__ void k_group_frames(Segs S, const int32_t* __restrict__ seg_run,
                               const int32_t* __restrict__ order, const int32_t* __restrict__ gstart,
                               int64_t ngroups, int64_t nseg, const double* __restrict__ xlo,
                               const double* __restrict__ xhi, WedgeOut W) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = gstart[g], b = g + 1 < ngroups ? gstart[g + 1] : nseg;
    const int64_t rr = seg_run[order[a]];
    double lo = xlo[a], hi = xhi[a];
    for (int64_t i = a + 1; i < b; ++i) {
      lo = fmin(lo, xlo[i]);
      hi = fmax(hi, xhi[i]);
    }
    const double3 e = ld3d(S.e + 3 * rr), pref = ld3d(S.pa + 3 * rr);
    st3(W.origin + 3 * g, make_double3(pref.x + lo * e.x, pref.y + lo * e.y, pref.z + lo * e.z));
    st3(W.e + 3 * g, e);
    st3(W.t0 + 3 * g, ld3d(S.t0 + 3 * rr));
    st3(W.n0 + 3 * g, ld3d(S.n0 + 3 * rr));
    st3(W.nn + 3 * g, ld3d(S.nn + 3 * rr));
    W.len[g] = hi - lo;
    W.nopen[g] = S.nopen[rr];
  }
}

// keep the first of each run of equal contribution rows (cols 0..4) that has an owner
__global__ void k_contrib_keep(const int64_t* __restrict__ rows, const int32_t* __restrict__ perm,
                               int64_t n, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* r = rows + 6 * (int64_t)perm[i];
    flag[i] = r[0] >= 0 && (i == 0 || !rows_equal(r, rows + 6 * (int64_t)perm[i - 1], 5));
  }
}

// hash_edge (paths.py:111-125) of every wedge
__global__ void k_edge_hashes(const double* __restrict__ origin, const double* __restrict__ e,
                              const double* __restrict__ len, int64_t nw, uint64_t* hr,
                              uint64_t* hf) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw;
       w += (int64_t)gridDim.x * blockDim.x) {
    double a[3], b[3];
    for (int k = 0; k < 3; ++k) {
      a[k] = origin[3 * w + k];
      b[k] = a[k] + len[w] * e[3 * w + k];
    }
    bool b_first = false;  // tuple(b) < tuple(a)
    for (int k = 0; k < 3; ++k)
      if (b[k] != a[k]) {
        b_first = b[k] < a[k];
        break;
      }
    const double* p = b_first ? b : a;
    const double* q = b_first ? a : b;
    uint64_t h1 = 0xCBF29CE484222325ULL, h2 = 0xCBF29CE484222325ULL;
    for (int k = 0; k < 6; ++k) {
      const double c = k < 3 ? p[k] : q[k - 3];
      const double x = c / 1e-4;
      uint64_t v1 = (uint64_t)(int64_t)floor(x + 0.5), v2 = (uint64_t)(int64_t)floor(x);
      for (int j = 0; j < 8; ++j) {
        h1 = (h1 ^ (v1 & 0xFFULL)) * 0x100000001B3ULL;
        h2 = (h2 ^ (v2 & 0xFFULL)) * 0x100000001B3ULL;
        v1 >>= 8;
        v2 >>= 8;
      }
    }
    hr[w] = h1;
    hf[w] = h2;
  }
}

unsigned grid_of(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)g;
}

// stable lexicographic sort of int64 rows (n, ncols): LSD radix passes over the
// columns, last first; perm = row indices in sorted order
int lexsort_rows(Arena& A, const int64_t* rows, int ncols, int64_t n, int32_t* perm,
                 cudaStream_t st) {
  if (n <= 0) return SBR_OK;
  uint64_t* k_in = A.get<uint64_t>(n);
  uint64_t* k_out = A.get<uint64_t>(n);
  int32_t* p_out = A.get<int32_t>(n);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "wedge sort scratch");
  k_iota32<<<grid_of(n), 256, 0, st>>>(perm, n);
  count_launch();
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, perm, p_out, (int)n, 0, 64, st);
  char* tmp = A.get<char>((int64_t)tmp_bytes);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "wedge sort scratch");
  for (int c = ncols - 1; c >= 0; --c) {
    k_gather_col<<<grid_of(n), 256, 0, st>>>(rows, ncols, c, perm, n, k_in);
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, perm, p_out, (int)n, 0, 64, st);
    cudaMemcpyAsync(perm, p_out, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
    count_launch();
    count_launch();
  }
  return SBR_OK;
}

// run starts of sorted rows: returns the run count, run_start filled
int run_starts(Arena& A, const int64_t* rows, int stride, int ncols, const int32_t* perm,
               const uint8_t* live, int64_t n, int32_t* run_start, int64_t* nruns,
               cudaStream_t st) {
  int32_t* flag = A.get<int32_t>(n + 1);
  int32_t* pos = A.get<int32_t>(n + 1);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "wedge run scratch");
  k_run_flags<<<grid_of(n), 256, 0, st>>>(rows, perm, live, n, stride, ncols, flag);
  count_launch();
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, thrust::counting_iterator<int32_t>(0), flag, run_start,
                             pos, (int)n, st);
  char* tmp = A.get<char>((int64_t)tb);
  if (!A.ok) return set_error(SBR_ERR_NOMEM, "wedge run scratch");
  cub::DeviceSelect::Flagged(tmp, tb, thrust::counting_iterator<int32_t>(0), flag, run_start, pos,
                             (int)n, st);
  count_launch();
  int32_t cnt = 0;
  cudaMemcpyAsync(&cnt, pos, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return set_error(SBR_ERR_CUDA, "wedge runs");
  *nruns = cnt;
  return SBR_OK;
}

template <typename T>
int to_host(std::vector<T>& v, const T* d, int64_t n, cudaStream_t st) {
  v.resize((size_t)(n > 0 ? n : 0));
  if (n > 0 && cudaMemcpyAsync(v.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return set_error(SBR_ERR_CUDA, "wedge copy-out");
  return SBR_OK;
}

}  // namespace

extern "C" {

int sbr_wedges_extract(const double* v0, const double* v1, const double* v2, const int64_t* obj,
                       const int64_t* prim, int64_t ntri,
                       double dihedral_threshold_deg, int32_t device, void* stream,
                       SbrWedgeSet** out) {
  if (!out || !v0 || !v1 || !v2 || !obj || !prim)
    return set_error(SBR_ERR_INVALID, "NULL argument");
  *out = nullptr;
  if (ntri < 0 || ntri >= (1LL << 29)) return set_error(SBR_ERR_INVALID, "bad triangle count");
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return set_error(SBR_ERR_CUDA, "bad device");
  cudaStream_t st = (cudaStream_t)stream;
  SbrWedgeSet* W = new SbrWedgeSet();
  int rc = SBR_OK;
  {
    Arena A(st);
    const int64_t ne = 3 * ntri;
    double *dv0 = A.get<double>(3 * ntri), *dv1 = A.get<double>(3 * ntri),
           *dv2 = A.get<double>(3 * ntri);
    int64_t *dobj = A.get<int64_t>(ntri), *dprim = A.get<int64_t>(ntri);
    int64_t* key = A.get<int64_t>(kKeyCols * ne);
    uint8_t* live = A.get<uint8_t>(ne);
    int32_t* perm = A.get<int32_t>(ne);
    int32_t* run_start = A.get<int32_t>(ne + 1);
    if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge scratch");
    const size_t b3 = sizeof(double) * 3 * (size_t)ntri;
    if (!rc && ntri > 0) {
      cudaMemcpyAsync(dv0, v0, b3, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dv1, v1, b3, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dv2, v2, b3, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dobj, obj, sizeof(int64_t) * ntri, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dprim, prim, sizeof(int64_t) * ntri, cudaMemcpyHostToDevice, st);
      k_edge_keys<<<grid_of(ne), 256, 0, st>>>(dv0, dv1, dv2, ne, key, live);
      count_launch();
      rc = lexsort_rows(A, key, kKeyCols, ne, perm, st);
    }
    int64_t nruns = 0;
    if (!rc && ntri > 0) rc = run_starts(A, key, kKeyCols, kKeyCols, perm, live, ne, run_start, &nruns, st);
    int64_t nseg = 0, n_screens = 0;
    Segs S;
    int32_t* seg_run = nullptr;
    EdgeIn E{dv0, dv1, dv2, dobj, dprim};
    if (!rc && nruns > 0) {
      S.line = A.get<int64_t>(6 * nruns);
      S.p0 = A.get<int64_t>(4 * nruns);
      S.pn = A.get<int64_t>(4 * nruns);
      S.pa = A.get<double>(3 * nruns);
      S.pb = A.get<double>(3 * nruns);
      S.e = A.get<double>(3 * nruns);
      S.n0 = A.get<double>(3 * nruns);
      S.nn = A.get<double>(3 * nruns);
      S.t0 = A.get<double>(3 * nruns);
      S.nopen = A.get<double>(nruns);
      S.own0 = A.get<int64_t>(nruns);
      S.ownn = A.get<int64_t>(nruns);
      S.o0 = A.get<int64_t>(nruns);
      S.m0 = A.get<int64_t>(nruns);
      int8_t* kind = A.get<int8_t>(nruns);
      int32_t *fs = A.get<int32_t>(nruns + 1), *fw = A.get<int32_t>(nruns + 1);
      int32_t *ps = A.get<int32_t>(nruns + 1), *pw = A.get<int32_t>(nruns + 1);
      seg_run = A.get<int32_t>(nruns);
      if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge segment scratch");
      if (!rc) {
        const double thresh = dihedral_threshold_deg * (kPi / 180.0);  // np.deg2rad
        k_run_segments<<<grid_of(nruns, 128), 128, 0, st>>>(E, perm, live, run_start, nruns, ne,
                                                            thresh, kind, S);
        k_seg_flags<<<grid_of(nruns), 256, 0, st>>>(kind, nruns, fs, fw);
        count_launch();
        count_launch();
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, fs, ps, (int)nruns + 1, st);
        char* tmp = A.get<char>((int64_t)tb);
        if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge scan scratch");
        if (!rc) {
          cudaMemsetAsync(fs + nruns, 0, sizeof(int32_t), st);
          cudaMemsetAsync(fw + nruns, 0, sizeof(int32_t), st);
          cub::DeviceScan::ExclusiveSum(tmp, tb, fs, ps, (int)nruns + 1, st);
          cub::DeviceScan::ExclusiveSum(tmp, tb, fw, pw, (int)nruns + 1, st);
          int32_t cs = 0, cw = 0;
          cudaMemcpyAsync(&cs, ps + nruns, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
          cudaMemcpyAsync(&cw, pw + nruns, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
          if (cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(SBR_ERR_CUDA, "wedge scan");
          n_screens = cs;
          nseg = (int64_t)cs + cw;
          if (!rc && nseg > 0) {
            k_seg_order<<<grid_of(nruns), 256, 0, st>>>(kind, ps, pw, nruns, n_screens, seg_run);
            count_launch();
          }
        }
      }
    }
    int64_t ngroups = 0;
    int32_t *gorder = nullptr, *gstart = nullptr;
    if (!rc && nseg > 0) {
      int64_t* mkey = A.get<int64_t>(kMergeCols * nseg);
      int32_t* mperm = A.get<int32_t>(nseg);
      int32_t* gflag_start = A.get<int32_t>(nseg + 1);
      int64_t* grows = A.get<int64_t>(4 * nseg);
      gorder = A.get<int32_t>(nseg);
      gstart = A.get<int32_t>(nseg + 1);
      int32_t* gid_sorted = A.get<int32_t>(nseg + 1);
      if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge merge scratch");
      if (!rc) {
        k_merge_keys<<<grid_of(nseg), 256, 0, st>>>(S, seg_run, nseg, mkey);
        count_launch();
        rc = lexsort_rows(A, mkey, kMergeCols, nseg, mperm, st);
      }
      int64_t nmg = 0;
      if (!rc) rc = run_starts(A, mkey, kMergeCols, kMergeCols, mperm, nullptr, nseg, gflag_start, &nmg, st);
      if (!rc) {
        // group id of each sorted position: inclusive scan of the run flags - 1
        int32_t* flag = A.get<int32_t>(nseg);
        if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge merge scratch");
        if (!rc) {
          k_run_flags<<<grid_of(nseg), 256, 0, st>>>(mkey, mperm, nullptr, nseg, kMergeCols,
                                                     kMergeCols, flag);
          size_t tb = 0;
          cub::DeviceScan::InclusiveSum(nullptr, tb, flag, gid_sorted, (int)nseg, st);
          char* tmp = A.get<char>((int64_t)tb);
          if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge merge scratch");
          if (!rc) {
            cub::DeviceScan::InclusiveSum(tmp, tb, flag, gid_sorted, (int)nseg, st);
            count_launch();
            count_launch();
            // rows (gid + 1, o, m, s): lexsort -> segments grouped, first owner first
            k_group_rows<<<grid_of(nseg), 256, 0, st>>>(mperm, gid_sorted, S, seg_run, nseg, grows);
            count_launch();
            rc = lexsort_rows(A, grows, 4, nseg, gorder, st);
          }
        }
      }
      if (!rc) {
        // group starts in gorder: the positions where the gid changes
        int64_t ng = 0;
        rc = run_starts(A, grows, 4, 1, gorder, nullptr, nseg, gstart, &ng, st);
        ngroups = ng;
      }
    }
    if (!rc && ngroups > 0) {
      WedgeOut O;
      O.origin = A.get<double>(3 * ngroups);
      O.e = A.get<double>(3 * ngroups);
      O.t0 = A.get<double>(3 * ngroups);
      O.n0 = A.get<double>(3 * ngroups);
      O.nn = A.get<double>(3 * ngroups);
      O.len = A.get<double>(ngroups);
      O.nopen = A.get<double>(ngroups);
      int32_t* pos_group = A.get<int32_t>(nseg);
      int64_t* contrib = A.get<int64_t>(12 * nseg);
      double *xlo = A.get<double>(nseg), *xhi = A.get<double>(nseg);
      int32_t* cperm = A.get<int32_t>(2 * nseg);
      int32_t* cflag = A.get<int32_t>(2 * nseg);
      int32_t* ckeep = A.get<int32_t>(2 * nseg);
      int32_t* ckcnt = A.get<int32_t>(1);
      uint64_t *hr = A.get<uint64_t>(ngroups), *hf = A.get<uint64_t>(ngroups);
      if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge output scratch");
      if (!rc) {
        k_pos_group<<<grid_of(ngroups, 128), 128, 0, st>>>(gstart, ngroups, nseg, pos_group);
        k_seg_contrib<<<grid_of(nseg, 128), 128, 0, st>>>(S, seg_run, gorder, gstart, pos_group,
                                                         nseg, E, contrib, xlo, xhi);
        k_group_frames<<<grid_of(ngroups, 128), 128, 0, st>>>(S, seg_run, gorder, gstart, ngroups,
                                                             nseg, xlo, xhi, O);
        k_edge_hashes<<<grid_of(ngroups), 256, 0, st>>>(O.origin, O.e, O.len, ngroups, hr, hf);
        for (int q = 0; q < 4; ++q) count_launch();
        // sorted(set(...)) per (group, side): lexsort of the rows, first of each run
        // rows (group, side, o, m, local, code): every column, so equal rows are
        // adjacent and the code (= (m, local) of one owner) breaks no tie
        rc = lexsort_rows(A, contrib, 6, 2 * nseg, cperm, st);
      }
      if (!rc) {
        k_contrib_keep<<<grid_of(2 * nseg), 256, 0, st>>>(contrib, cperm, 2 * nseg, cflag);
        count_launch();
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, cperm, cflag, ckeep, ckcnt, (int)(2 * nseg), st);
        char* tmp = A.get<char>((int64_t)tb);
        if (!A.ok) rc = set_error(SBR_ERR_NOMEM, "wedge owner scratch");
        if (!rc) {
          cub::DeviceSelect::Flagged(tmp, tb, cperm, cflag, ckeep, ckcnt, (int)(2 * nseg), st);
          count_launch();
        }
      }
      // host: owner lists per wedge, the final order by first owner, copy-out
      std::vector<int32_t> keep_idx, kc;
      std::vector<int64_t> crows;
      std::vector<double> origin, e, t0, n0, nn, len, nopen;
      std::vector<uint64_t> vhr, vhf;
      if (!rc) rc = to_host(kc, ckcnt, 1, st);
      if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(SBR_ERR_CUDA, "wedge owners");
      if (!rc) rc = to_host(keep_idx, ckeep, kc[0], st);
      if (!rc) rc = to_host(crows, contrib, 12 * nseg, st);
      if (!rc) rc = to_host(origin, O.origin, 3 * ngroups, st);
      if (!rc) rc = to_host(e, O.e, 3 * ngroups, st);
      if (!rc) rc = to_host(t0, O.t0, 3 * ngroups, st);
      if (!rc) rc = to_host(n0, O.n0, 3 * ngroups, st);
      if (!rc) rc = to_host(nn, O.nn, 3 * ngroups, st);
      if (!rc) rc = to_host(len, O.len, ngroups, st);
      if (!rc) rc = to_host(nopen, O.nopen, ngroups, st);
      if (!rc) rc = to_host(vhr, hr, ngroups, st);
      if (!rc) rc = to_host(vhf, hf, ngroups, st);
      if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(SBR_ERR_CUDA, "wedge copy-out");
      if (!rc) {
        // CSR of the unique sorted contributions per (group, side)
        std::vector<std::vector<int64_t>> side0((size_t)ngroups), siden((size_t)ngroups);
        std::vector<std::array<int64_t, 3>> first((size_t)ngroups,
                                                 std::array<int64_t, 3>{INT64_MAX, INT64_MAX, INT64_MAX});
        std::vector<char> has0((size_t)ngroups, 0);
        for (int32_t k : keep_idx) {
          const int64_t* row = crows.data() + 6 * (int64_t)k;
          const int64_t g = row[0];
          (row[1] == 0 ? side0 : siden)[g].push_back(row[5]);
          // (face0 + facen)[0]: face0's first (sorted) owner, else facen's
          if (row[1] == 0 && !has0[g]) {
            has0[g] = 1;
            first[g] = {row[2], row[3], row[4]};
          } else if (row[1] == 1 && !has0[g] && siden[g].size() == 1) {
            first[g] = {row[2], row[3], row[4]};
          }
        }
        std::vector<int64_t> order((size_t)ngroups);
        for (int64_t g = 0; g < ngroups; ++g) order[g] = g;
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t x, int64_t y) { return first[x] < first[y]; });
        const int64_t nw = ngroups;
        W->n_wedges = nw;
        W->origin.resize(3 * nw);
        W->e_hat.resize(3 * nw);
        W->t0_hat.resize(3 * nw);
        W->n0_hat.resize(3 * nw);
        W->nn_hat.resize(3 * nw);
        W->length.resize(nw);
        W->n_open.resize(nw);
        W->hash_r.resize(nw);
        W->hash_f.resize(nw);
        W->off0.assign(1, 0);
        W->offn.assign(1, 0);
        for (int64_t i = 0; i < nw; ++i) {
          const int64_t g = order[i];
          for (int k = 0; k < 3; ++k) {
            W->origin[3 * i + k] = origin[3 * g + k];
            W->e_hat[3 * i + k] = e[3 * g + k];
            W->t0_hat[3 * i + k] = t0[3 * g + k];
            W->n0_hat[3 * i + k] = n0[3 * g + k];
            W->nn_hat[3 * i + k] = nn[3 * g + k];
          }
          W->length[i] = len[g];
          W->n_open[i] = nopen[g];
          W->hash_r[i] = vhr[g];
          W->hash_f[i] = vhf[g];
          W->own0.insert(W->own0.end(), side0[g].begin(), side0[g].end());
          W->ownn.insert(W->ownn.end(), siden[g].begin(), siden[g].end());
          W->off0.push_back((int64_t)W->own0.size());
          W->offn.push_back((int64_t)W->ownn.size());
        }
        W->n_owners0 = (int64_t)W->own0.size();
        W->n_ownersn = (int64_t)W->ownn.size();
      }
    }
    if (!rc && cudaGetLastError() != cudaSuccess) rc = set_error(SBR_ERR_CUDA, "wedge kernels");
  }
  if (prev >= 0) cudaSetDevice(prev);
  if (rc) {
    delete W;
    return rc;
  }
  if (W->off0.empty()) {
    W->off0.assign(1, 0);
    W->offn.assign(1, 0);
  }
  *out = W;
  return SBR_OK;
}

int sbr_wedges_count(const SbrWedgeSet* W, int64_t* n_wedges, int64_t* n_owners0,
                     int64_t* n_ownersn) {
  if (!W) return set_error(SBR_ERR_INVALID, "NULL wedge set");
  if (n_wedges) *n_wedges = W->n_wedges;
  if (n_owners0) *n_owners0 = W->n_owners0;
  if (n_ownersn) *n_ownersn = W->n_ownersn;
  return SBR_OK;
}

int sbr_wedges_copy(const SbrWedgeSet* W, double* origin, double* e_hat, double* t0_hat,
                    double* n0_hat, double* nn_hat, double* length, double* n_open,
                    uint64_t* hash_r, uint64_t* hash_f, int64_t* off0, int64_t* own0,
                    int64_t* offn, int64_t* ownn) {
  if (!W) return set_error(SBR_ERR_INVALID, "NULL wedge set");
  const size_t n = (size_t)W->n_wedges;
  auto cp = [](void* dst, const void* src, size_t bytes) {
    if (dst && bytes) memcpy(dst, src, bytes);
  };
  cp(origin, W->origin.data(), 24 * n);
  cp(e_hat, W->e_hat.data(), 24 * n);
  cp(t0_hat, W->t0_hat.data(), 24 * n);
  cp(n0_hat, W->n0_hat.data(), 24 * n);
  cp(nn_hat, W->nn_hat.data(), 24 * n);
  cp(length, W->length.data(), 8 * n);
  cp(n_open, W->n_open.data(), 8 * n);
  cp(hash_r, W->hash_r.data(), 8 * n);
  cp(hash_f, W->hash_f.data(), 8 * n);
  cp(off0, W->off0.data(), 8 * (n + 1));
  cp(offn, W->offn.data(), 8 * (n + 1));
  cp(own0, W->own0.data(), 8 * W->own0.size());
  cp(ownn, W->ownn.data(), 8 * W->ownn.size());
  return SBR_OK;
}

void sbr_wedges_free(SbrWedgeSet* W) { delete W; }

}  // extern "C"
