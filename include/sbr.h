/*
 * sbr.h -- C ABI of the B200-native shooting-and-bouncing-rays (SBR) core.
 *
 * This is the drop-in boundary for the emtrace hot path.  The
 * reference binds its native code one level lower, at
 *   emtrace._kernels.active().trace_closest / trace_any
 *   (pkg/src/emtrace/_kernels.py:21-24, pkg/src/emtrace/_core.pyx:115-253),
 * but those entry points take the reference's own host SAH BVH arrays.  Here
 * the BVH is built on the GPU, so the boundary sits at the level of
 *   Accel.__init__ / trace_batch / occluded_batch   (geometry.py:131-201)
 *   compute_radio_map_sbr / _map_chunk / _direct_cells (radiomap.py:347-633)
 *   generate_candidates / refine_candidate / compute_path_fields /
 *   frequency_response                                (paths.py:1019-1547)
 * Each function below cites the reference interface it replaces.
 *
 * Conventions
 *  - Every function returns an int status (SBR_OK = 0).  sbr_last_error()
 *    returns a thread-local message for the last failure.  Status codes map
 *    onto the reference's exceptions (see SBR_ERR_*).
 *  - Array arguments named *_dev are DEVICE pointers owned by the caller
 *    (torch allocates them); everything else is host memory.  `stream` is a
 *    cudaStream_t (NULL = legacy default stream).  Calls are asynchronous on
 *    `stream` unless stated otherwise.
 *  - All geometry and field arithmetic is IEEE float64 with the reference's
 *    operation order (no FMA contraction); BVH boxes are conservative fp32.
 *  - Triangle indices returned by the library are SLOTS of the library's own
 *    (Morton) order; sbr_scene_permutation() maps them to input order.
 */
#ifndef SBR_H
#define SBR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (-> Python exceptions) ------------------------------ */
#define SBR_OK 0
#define SBR_ERR_INVALID 1        /* ValueError                                */
#define SBR_ERR_EMPTY_SCENE 2    /* errors.EmptyScene (geometry.py:136-137)  */
#define SBR_ERR_STACK 3          /* RuntimeError("BVH traversal stack overflow"),
                                    _core.pyx:190-191                         */
#define SBR_ERR_CUDA 4           /* RuntimeError (CUDA failure)               */
#define SBR_ERR_UNSUPPORTED 5    /* NotImplementedError (out-of-scope feature) */
#define SBR_ERR_NOMEM 6          /* MemoryError                               */

/* Radio-map RNG chunking: part of the reference's RNG contract
 * (radiomap.py:53-55, CHUNK_SAMPLES = 1 << 19). */
#define SBR_CHUNK_LOG2 19

/* ---- material / antenna parameter blocks -------------------------------- */
enum { SBR_SCAT_LAMBERTIAN = 0, SBR_SCAT_DIRECTIVE = 1, SBR_SCAT_BACKSCATTERING = 2 };
enum { SBR_PATTERN_ISOTROPIC = 0, SBR_PATTERN_TR38901 = 1 };

/* One row per object id in sorted order (paths.py:491-499: the reference keeps
 * one material row per object, tri_material_row = searchsorted(object_ids)). */
typedef struct SbrMaterial {
  double eta_re, eta_im;          /* complex_permittivity(f)  materials.py:130   */
  double sqrt_eta_re, sqrt_eta_im;/* np.sqrt(eta) (principal), host-computed     */
  double kd;                      /* 2*pi*thickness/wavelength, materials.py:232 */
  double thickness;
  double scattering;              /* S                                           */
  double spec_amp;                /* sqrt(max(0, 1-S^2))   materials.py:123      */
  double xpd_kx;
  double lambda_mix;
  int32_t pattern_kind;           /* SBR_SCAT_*                                  */
  int32_t alpha_r, alpha_i;
  int32_t random_phases;
} SbrMaterial;

/* Transmit / receive antenna pattern (em.py:258-308). */
typedef struct SbrAntenna {
  int32_t kind;                   /* SBR_PATTERN_*                               */
  int32_t identity;               /* rot == I (exact fast path)                  */
  double scale;                   /* tr38901 amplitude normalisation (em.py:281) */
  double rot[9];                  /* row-major rotation_ypr(orientation)         */
} SbrAntenna;

/* Radio-map run parameters (RadioMapConfig radiomap.py:169-215,
 * MeasurementGrid radiomap.py:65-152, source / pattern / array / precoder). */
typedef struct SbrMapParams {
  double source[3];
  double corner[3];
  double u_hat[3];
  double v_hat[3];
  double normal[3];               /* cross(u_hat, v_hat)                         */
  double plane_off;               /* normal . center (np 1-D dot)                */
  double cell_w, cell_h;
  double scale;                   /* (lambda/4pi)^2 / cell_area                  */
  double wavelength;
  double omega0;                  /* 4*pi / num_samples                          */
  double rr_max;
  double gain_threshold;
  uint64_t num_samples;
  uint64_t seed;
  int32_t nx, ny;
  int32_t max_depth;
  int32_t allow_mask;             /* bit0 R, bit1 S, bit2 T (D never in the loop)*/
  int32_t rr_depth;               /* -1 = off                                    */
  int32_t cull_from;
  int32_t any_random_phase;
  int32_t n_elements;             /* 0 = no array: weight0 = 1                   */
  SbrAntenna pattern;
  const double* elem_offsets_dev; /* (n_elements, 3)                             */
  const double* precoder_dev;     /* (n_elements, 2) complex (re, im)            */
} SbrMapParams;

/* Radio-map diagnostics counters (radiomap.py:413-631). */
enum {
  SBR_MC_DEPOSITS = 0,
  SBR_MC_ESCAPED,
  SBR_MC_TERMINATED,
  SBR_MC_RESPAWNS,
  SBR_MC_THRESHOLD_KILLED,
  SBR_MC_ROULETTE_KILLED,
  SBR_MC_RAY_BOUNCES,      /* sum of rows traced (the rb metric) */
  SBR_MC_DIRECT_VISIBLE,
  SBR_MC_STACK_OVERFLOW,
  SBR_MC_COUNT
};

/* ---- scene -------------------------------------------------------------- */
typedef struct SbrScene SbrScene;

/* Replaces Accel.__init__ / _build_bvh (geometry.py:134-166, 244-349).
 * v0, v1, v2: host (ntri, 3) float64 corners in input order.  Builds an LBVH
 * (Morton codes, radix sort, Karras hierarchy, bottom-up refit, leaves <= 4)
 * on `device`.  Fails with SBR_ERR_EMPTY_SCENE when ntri == 0. */
int sbr_scene_create(const double* v0, const double* v1, const double* v2,
                     int64_t ntri, int32_t device, void* stream, SbrScene** out);
void sbr_scene_destroy(SbrScene* scene);
int64_t sbr_scene_num_triangles(const SbrScene* scene);
int64_t sbr_scene_num_nodes(const SbrScene* scene);
/* Host copy of slot -> input triangle index (the reference's Accel.perm). */
int sbr_scene_permutation(const SbrScene* scene, int64_t* perm_out);
/* Per-slot attributes, host arrays in SLOT order:
 *   tie_rank  : rank of (object_id, primitive_id) -- closest-hit tie rule
 *               (_core.pyx:158-161)
 *   normals   : (T,3) float64 geometric normals (geometry.py:165-166)
 *   matrow    : material row (paths.py:497-499)
 *   hash_r/f  : plane hashes (paths.py:449-450), may be NULL                 */
int sbr_scene_set_attributes(SbrScene* scene, const int32_t* tie_rank,
                             const double* normals, const int32_t* matrow,
                             const uint64_t* hash_r, const uint64_t* hash_f);
int sbr_scene_set_materials(SbrScene* scene, const SbrMaterial* mats, int32_t n);
/* Reads and clears the device error word (stack overflow).  Synchronises
 * `stream`.  Returns SBR_ERR_STACK if any traversal overflowed. */
int sbr_scene_check(SbrScene* scene, void* stream);

/* ---- ray queries ---------------------------------------------------------- */
/* Replaces Accel.trace_batch -> trace_closest (geometry.py:178-185,
 * _core.pyx:115-195).  Outputs: t (inf = miss), tri (slot, -1 = miss), u, v. */
int sbr_trace_closest(const SbrScene* scene, const double* origins_dev,
                      const double* dirs_dev, double t_min,
                      const double* t_max_dev, int64_t n, double* t_dev,
                      int64_t* tri_dev, double* u_dev, double* v_dev, void* stream);
/* Replaces trace_any (_core.pyx:198-253). hit_dev: uint8 per ray. */
int sbr_trace_any(const SbrScene* scene, const double* origins_dev,
                  const double* dirs_dev, double t_min, const double* t_max_dev,
                  int64_t n, uint8_t* hit_dev, void* stream);
/* Replaces Accel.occluded_batch (geometry.py:187-201): open segments a->b
 * with endpoints offset by eps. */
int sbr_occluded(const SbrScene* scene, const double* a_dev, const double* b_dev,
                 double eps, int64_t n, uint8_t* occluded_dev, void* stream);

/* ---- sampling ------------------------------------------------------------- */
/* fibonacci_directions(num_samples)[begin:end] (sampling.py:81-95). */
int sbr_fibonacci(uint64_t num_samples, uint64_t begin, uint64_t end,
                  double* dirs_dev, void* stream);
/* RngStream(seed, sample, depth, purpose).generator().random(count)
 * (sampling.py:49-78) for purposes identified by their FNV-1a tag hash. */
int sbr_philox_uniform(uint64_t seed, uint64_t sample, uint64_t depth,
                       uint64_t tag_hash, uint64_t first, uint64_t count,
                       double* out_dev, void* stream);

/* ---- radio map ------------------------------------------------------------ */
/* Replaces the _map_chunk bounce loop over global sample ids
 * [sample_begin, sample_end) (radiomap.py:347-563, 586-628).  Deposits are
 * accumulated (float64 atomics) into grid_dev (ny, nx); counters_dev holds
 * SBR_MC_COUNT uint64 and is accumulated into.  sample_begin/end may be any
 * sub-range: the RNG is keyed by (seed, g >> 19, depth, tag)[g & (2^19-1)],
 * so shards are bitwise-independent of how samples are split. */
int sbr_radiomap_bounce(const SbrScene* scene, const SbrMapParams* params,
                        uint64_t sample_begin, uint64_t sample_end,
                        double* grid_dev, uint64_t* counters_dev, void* stream);
/* Replaces _direct_cells (radiomap.py:566-583): analytic LoS term per cell
 * centre into direct_dev (ny, nx) (overwritten), counts visible cells. */
int sbr_radiomap_direct(const SbrScene* scene, const SbrMapParams* params,
                        double* direct_dev, uint64_t* counters_dev, void* stream);

/* ---- misc ----------------------------------------------------------------- */
const char* sbr_last_error(void);
int sbr_version(void);
/* Number of CUDA kernels this library launched since load (evidence counter). */
uint64_t sbr_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SBR_H */
