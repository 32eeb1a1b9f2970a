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
#define SBR_ERR_INTERNAL 7       /* RuntimeError (checked build: device bounds check) */

/* Radio-map RNG chunking: part of the reference's RNG contract
 * (radiomap.py:53-55, CHUNK_SAMPLES = 1 << 19). */
#define SBR_CHUNK_LOG2 19
/* id-chunk size of the chunk-cyclic CIR shards (sbr_cir_sweep_sharded) */
#define SBR_CIR_SHARD_LOG2 12

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
  SBR_MC_CONE_SAMPLES,     /* edge-estimator samples drawn (radiomap.py:889) */
  SBR_MC_COUNT
};

/* Build flags of the loaded library: bit 0 = checked build (SBR_CHECKED). */
int sbr_build_flags(void);

/* ---- scene -------------------------------------------------------------- */
typedef struct SbrScene SbrScene;

/* Replaces Accel.__init__ / _build_bvh (geometry.py:134-166, 244-349).
 * v0, v1, v2: host (ntri, 3) float64 corners in input order.  Builds the BVH
 * on `device` (Morton codes, radix sort, PLOC or Karras hierarchy, bottom-up
 * refit, leaves of <= 2 triangles).  Fails with SBR_ERR_EMPTY_SCENE when
 * ntri == 0 and SBR_ERR_INVALID for a non-finite coordinate (the reference
 * accepts those and produces NaN geometry).  On failure nothing is leaked. */
int sbr_scene_create(const double* v0, const double* v1, const double* v2,
                     int64_t ntri, int32_t device, void* stream, SbrScene** out);
/* Frees the scene; the calling thread's current CUDA device is unchanged. */
void sbr_scene_destroy(SbrScene* scene);
/* Returns every freed block of the library's private scratch pool on `device`
 * (ray queues, sort buffers; kept mapped between calls up to 16 GiB) to the
 * driver.  Synchronises the device.  No reference counterpart. */
int sbr_release_scratch(int32_t device);
/* Hierarchy of subsequently created scenes over the same GPU Morton sort:
 * 0 = Karras 2012 LBVH; 1 = PLOC (parallel locally-ordered clustering) down
 * to 262,144 clusters, then a top-down SAH over the clusters (default); 2 =
 * PLOC all the way.  All collapse to <= 2-triangle leaves. */
int sbr_set_bvh_builder(int32_t builder);
int64_t sbr_scene_num_triangles(const SbrScene* scene);
int64_t sbr_scene_num_nodes(const SbrScene* scene);
/* Host copy of the BVH2 node array (sbr_scene_num_nodes() x 64 B: child boxes
 * as float4 (l.lo.x, l.hi.x, l.lo.y, l.hi.y), (r...), (l.lo.z, l.hi.z, r.lo.z,
 * r.hi.z) and int4 child codes (>= 0 node, < 0 leaf ~(start << 2 | count-1))),
 * for structural tests and tree-quality diagnostics. */
int sbr_scene_copy_nodes(const SbrScene* scene, void* host_out);
/* Host copy of slot -> input triangle index (the reference's Accel.perm). */
int sbr_scene_permutation(const SbrScene* scene, int64_t* perm_out);
/* Host copies of the per-slot tables sbr_scene_create derives on the device
 * from the float64 corners with numpy's operation order: geometric normals
 * normalize((v1-v0) x (v2-v0)) (geometry.py:165-166, (T,3) f64) and the
 * (round, floor) plane hashes of _plane_hash_rows (paths.py:156-171, (T,)
 * u64).  Any output may be NULL. */
int sbr_scene_copy_tables(const SbrScene* scene, double* normals_out, uint64_t* hash_r_out,
                          uint64_t* hash_f_out);
/* Per-slot attributes, host arrays in SLOT order (override the derived ones):
 *   tie_rank  : rank of (object_id, primitive_id) -- closest-hit tie rule
 *               (_core.pyx:158-161)
 *   normals   : (T,3) float64 geometric normals (geometry.py:165-166)
 *   matrow    : material row (paths.py:497-499)
 *   hash_r/f  : plane hashes (paths.py:449-450), may be NULL                 */
int sbr_scene_set_attributes(SbrScene* scene, const int32_t* tie_rank,
                             const double* normals, const int32_t* matrow,
                             const uint64_t* hash_r, const uint64_t* hash_f);
int sbr_scene_set_materials(SbrScene* scene, const SbrMaterial* mats, int32_t n);

/* Diffraction wedges (geometry.py:356-494 extract_wedges; paths.py:452-475
 * tables), host arrays uploaded once: per-wedge frame, length, exterior
 * angle n, edge hashes (hash_edge, paths.py:111-125), material rows of the
 * 0- and n-faces, and per SLOT the sorted ids of the wedges it owns (CSR). */
typedef struct SbrWedgeTable {
  int64_t n_wedges;
  const double* origin;           /* (nw, 3) */
  const double* e_hat;            /* (nw, 3) */
  const double* t0_hat;           /* (nw, 3) */
  const double* n0_hat;           /* (nw, 3) */
  const double* nn_hat;           /* (nw, 3) */
  const double* length;           /* (nw) */
  const double* n_open;           /* (nw) */
  const uint64_t* hash_r;         /* (nw) */
  const uint64_t* hash_f;         /* (nw) */
  const int32_t* mat0;            /* (nw) material row of face0[0] */
  const int32_t* matn;            /* (nw) material row of (facen or face0)[0] */
  const int32_t* slot_offsets;    /* (T + 1) */
  const int32_t* slot_ids;        /* (slot_offsets[T]) */
} SbrWedgeTable;
int sbr_scene_set_wedges(SbrScene* scene, const SbrWedgeTable* table);
/* Replaces extract_wedges (geometry.py:356-494) and hash_edge
 * (paths.py:111-125): diffraction wedge extraction on `device` from the
 * flattened host triangles in input order (corners (T,3) f64, object and
 * primitive ids).  The result lives in an opaque SbrWedgeSet: per wedge
 * origin, e_hat, t0_hat, n0_hat, nn_hat (3 f64 each), length, n (exterior
 * angle / pi), the (round, floor) edge hashes, and the owner lists face0 /
 * facen as CSR over owner codes 3 * input_triangle + local_edge, sorted like
 * the reference's sorted(set(...)); wedges in the reference's order. */
typedef struct SbrWedgeSet SbrWedgeSet;
int sbr_wedges_extract(const double* v0, const double* v1, const double* v2, const int64_t* obj,
                       const int64_t* prim, int64_t ntri, double dihedral_threshold_deg,
                       int32_t device, void* stream, SbrWedgeSet** out);
int sbr_wedges_count(const SbrWedgeSet* set, int64_t* n_wedges, int64_t* n_owners0,
                     int64_t* n_ownersn);
/* Host copies (any pointer may be NULL); off0 / offn hold n_wedges + 1 entries. */
int sbr_wedges_copy(const SbrWedgeSet* set, double* origin, double* e_hat, double* t0_hat,
                    double* n0_hat, double* nn_hat, double* length, double* n_open,
                    uint64_t* hash_r, uint64_t* hash_f, int64_t* off0, int64_t* own0,
                    int64_t* offn, int64_t* ownn);
void sbr_wedges_free(SbrWedgeSet* set);

/* ---- scene files (host code, no device needed) ------------------------- */
/* Replaces _read_obj_arrays / _obj_corner_index (E/sceneio.py:129-175): ASCII
 * OBJ text -> vertices (nv, 3) f64 and fan-triangulated 0-based triangles
 * (nt, 3) i64; `v` / `f` lines only, 1-based or negative indices, v/vt/vn
 * tokens, '#' comments; numbers in Python float()/int() syntax.  Parsed on
 * host threads in two passes (counts, then blocks at known offsets).  On a
 * syntax error returns SBR_ERR_INVALID with the 1-based line, the error kind
 * (1 vertex needs 3 coordinates, 2 bad vertex, 3 face needs at least 3
 * vertices, 4 bad face index, 5 index 0, 6 index out of range) and its detail
 * text (the stripped line body / the face token / str(index)) in err_detail.
 * Degenerate-triangle removal stays with the caller (reference semantics). */
typedef struct SbrObjMesh SbrObjMesh;
int sbr_obj_parse(const char* text, int64_t len, SbrObjMesh** out, int64_t* err_line,
                  int32_t* err_kind, char* err_detail, int64_t detail_cap);
int sbr_obj_sizes(const SbrObjMesh* mesh, int64_t* n_vertices, int64_t* n_triangles);
int sbr_obj_copy(const SbrObjMesh* mesh, double* vertices, int64_t* triangles);
void sbr_obj_free(SbrObjMesh* mesh);
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
/* The bounce loop over a block-cyclic shard of the global sample ids
 * [0, num_samples): blocks of 2^b ids (g >> b) = shard_index, shard_index +
 * shard_count, ..., b = log2(num_samples / (8 * shard_count)) clamped to
 * [SBR_CHUNK_LOG2, 23] (whole RNG chunks; >= 8 blocks per shard).  The shards
 * of one call partition the ids, so summing their grids / counters gives
 * sbr_radiomap_bounce(0, num_samples); unlike contiguous ranges every shard
 * sees the whole sphere of directions (balanced work per GPU), while each
 * block is a contiguous polar band (coherent passes).  No reference
 * counterpart (multi-GPU only). */
int sbr_radiomap_bounce_sharded(const SbrScene* scene, const SbrMapParams* params,
                                int32_t shard_index, int32_t shard_count, double* grid_dev,
                                uint64_t* counters_dev, void* stream);
/* Wavefront passes of a multi-pass map in flight at once (1..4): 2 (default)
 * runs consecutive passes on the caller's stream and a second one with their
 * own queues (~7.4 GB each) so kernel tails overlap; 1 serialises them
 * (per-kernel timing).  No reference counterpart. */
int sbr_set_wave_streams(int32_t n);
/* Exact map cells (0 = off, default; 1 = on): deposits accumulate as 192-bit
 * fixed-point integers (LSB 2^-160, range 2^32) and are converted once per
 * call, so maps are bitwise reproducible whatever the deposit order -- the
 * reference's worker-count determinism (radiomap.py chunk sums;
 * tests/test_radiomap.py:335-346).  Off: float64 atomics, last-bit order
 * dependence, ~3 % faster on config 4.  Applies to sbr_radiomap_bounce*,
 * sbr_radiomap_wedges. */
int sbr_set_exact_maps(int32_t on);
/* Replaces _direct_cells (radiomap.py:566-583): analytic LoS term per cell
 * centre into direct_dev (ny, nx) (overwritten), counts visible cells. */
int sbr_radiomap_direct(const SbrScene* scene, const SbrMapParams* params,
                        double* direct_dev, uint64_t* counters_dev, void* stream);

/* Replaces compute_radio_map_diffraction (radiomap.py:842-965): the edge
 * estimator over the listed wedges (collect_wedges_near_source, 645-671):
 * wedge_samples (offset, cone azimuth) draws per wedge from the `map-wedge`
 * Philox stream keyed (seed, wedge, block), plane crossing, exterior-region
 * and occlusion tests, UTD transfer, finite-difference area weighting, float64
 * atomic deposit into grid_dev (accumulated).  Requires sbr_scene_set_wedges. */
int sbr_radiomap_wedges(const SbrScene* scene, const SbrMapParams* params,
                        const int32_t* wedge_ids_dev, int32_t n_wedges, uint64_t wedge_samples,
                        double* grid_dev, uint64_t* counters_dev, void* stream);

/* ---- path solver (CIR) ---------------------------------------------------- */
/* Counters of the path-solver pipeline (paths.py:1098-1103, 1509-1512). */
enum {
  SBR_CC_SAMPLES_ESCAPED = 0,
  SBR_CC_SAMPLES_TERMINATED,
  SBR_CC_RAY_BOUNCES,        /* closest-hit rows traced in the sweep          */
  SBR_CC_VERTICES,           /* interaction vertices written                  */
  SBR_CC_VIS_RAYS,           /* (vertex, target) occlusion rays cast          */
  SBR_CC_ROWS,               /* visible (vertex, target) rows emitted         */
  SBR_CC_DUPLICATES,
  SBR_CC_CHUNK_TRUNCATED,
  SBR_CC_BUFFER_OVERFLOW,
  SBR_CC_CANDIDATES,
  SBR_CC_HASH_REGISTERED,
  SBR_CC_HASH_SLOTS,         /* distinct DedupTable slots claimed             */
  SBR_CC_REJ_COPLANAR,
  SBR_CC_REJ_OCCLUDED,
  SBR_CC_REJ_DEGENERATE,
  SBR_CC_STACK_OVERFLOW,
  SBR_CC_VERTEX_OVERFLOW,
  SBR_CC_ROW_OVERFLOW,
  SBR_CC_REJ_OFF_EDGE,
  SBR_CC_COUNT
};

/* Refinement outcome per record (paths.py:1123-1245 Rejection reasons). */
enum { SBR_REFINE_OK = 0, SBR_REFINE_COPLANAR_MISS = 1, SBR_REFINE_OCCLUDED = 2,
       SBR_REFINE_DEGENERATE = 3, SBR_REFINE_OFF_EDGE = 4 };

/* Generation parameters of one source (PathConfig paths.py:356-395). */
typedef struct SbrCirParams {
  double source[3];
  double q_diffraction;
  uint64_t num_samples;
  uint64_t seed;
  int32_t max_depth;
  int32_t allow_mask;             /* R=1 S=2 T=4 D=8                            */
  int32_t n_targets;
  int32_t pad_;
  const double* targets_dev;      /* (n_targets, 3)                             */
} SbrCirParams;

/* Interaction vertices of the sweep (the reference's per-depth `history`,
 * paths.py:774-781), one entry per closest hit that chose an interaction.
 * Device SoA, `capacity` entries; `parent` links a vertex to the previous
 * interaction of the same sample, so a row's whole history is a chain. */
typedef struct SbrVertexBuf {
  double* point;                  /* (cap, 3) o + t d                           */
  double* normal;                 /* (cap, 3) geometric normal facing the ray   */
  double* run_prob;               /* product of chosen interaction probabilities*/
  int64_t* sample;                /* global sample id                           */
  uint64_t* hash_r;               /* chain hash after this step (round / floor) */
  uint64_t* hash_f;
  int32_t* parent;                /* previous vertex of the sample, -1 = none   */
  int32_t* tri;                   /* scene slot                                 */
  uint8_t* code;                  /* 0 R, 1 S, 2 T, 3 D                         */
  uint8_t* depth;                 /* 1-based                                    */
  uint8_t* suffix_start;          /* depth of the last S step, 0 = none         */
  int32_t* wedge;                 /* wedge of a D step, -1                      */
  int64_t capacity;
} SbrVertexBuf;

/* Materialised candidate records (CandidateRecord paths.py:249-273), SoA with
 * `max_depth` step slots per record.  LoS records have depth 0. */
typedef struct SbrRecordBuf {
  int32_t* target;                /* (n)                                        */
  int64_t* sample;                /* (n) -1 = LoS                               */
  int32_t* depth;                 /* (n)                                        */
  int32_t* suffix_start;          /* (n)                                        */
  uint8_t* diffuse;               /* (n) diffuse-terminal                       */
  uint64_t* chain_hash;           /* (n) round-quantizer chain hash             */
  double* prefix_prob;            /* (n)                                        */
  double* anchor;                 /* (n, 3)                                     */
  int8_t* kind;                   /* (n, L) 0 R 1 S 2 T, -1 unused              */
  int32_t* tri;                   /* (n, L) scene slot                          */
  double* vertex;                 /* (n, L, 3)                                  */
  double* normal;                 /* (n, L, 3)                                  */
  int32_t max_depth;              /* L                                          */
  int32_t pad_;
  int32_t* wedge;                 /* (n, L) wedge index, -1                     */
} SbrRecordBuf;

/* Field-replay parameters of one source (compute_path_fields, paths.py:1302). */
typedef struct SbrFieldParams {
  double wavelength;
  double q_diffraction;
  double tx_velocity[3];
  uint64_t num_samples;
  uint64_t seed;
  int32_t allow_mask;
  int32_t n_objects;              /* rows of obj_velocity_dev (may be 0)        */
  SbrAntenna tx_pattern;
  const SbrAntenna* rx_pattern_dev;   /* (n_targets) per-target rx pattern      */
  const double* rx_velocity_dev;      /* (n_targets, 3)                         */
  const double* obj_velocity_dev;     /* (n_objects, 3) per material row        */
} SbrFieldParams;

/* Sweep of global sample ids [sample_begin, sample_end) through the bounce
 * loop of _sweep_chunk (paths.py:704-828, _continue_rays 855-900): closest
 * hit, slab energies, interaction draw (Philox `interaction` stream keyed by
 * global id), rolling plane hash, mirror / hemisphere respawn.  Appends one
 * vertex per interaction at index counters_dev[SBR_CC_VERTICES]. */
int sbr_cir_sweep(const SbrScene* scene, const SbrCirParams* params, uint64_t sample_begin,
                  uint64_t sample_end, const SbrVertexBuf* vb, uint64_t* counters_dev,
                  void* stream);
/* Spatial (Morton) order of the first nv vertices, for coherent occlusion
 * rays in sbr_cir_visibility: order_dev (nv) int32 vertex indices. */
/* sbr_cir_sweep over a chunk-cyclic shard of [0, num_samples): id chunks of
 * 2^SBR_CIR_SHARD_LOG2 dealt round-robin (balanced work per GPU; contiguous
 * shards of the pole-to-pole Fibonacci order differ 2x in visibility work).
 * vb needs (shard size) * max_depth vertices.  No reference counterpart. */
int sbr_cir_sweep_sharded(const SbrScene* scene, const SbrCirParams* params,
                          int32_t shard_index, int32_t shard_count, const SbrVertexBuf* vb,
                          uint64_t* counters_dev, void* stream);
int sbr_cir_vertex_order(const SbrScene* scene, const SbrVertexBuf* vb, int64_t nv,
                         int32_t* order_dev, void* stream);
/* _visible_pairs (paths.py:657-683): half-space side test + occlusion ray for
 * every (vertex, target) pair over positions [v_begin, v_end) of order_dev
 * (NULL = identity order); appends visible rows (ordinal key
 * (depth << 60 | sample << 20 | target), vertex index) at
 * counters_dev[SBR_CC_ROWS].  Rows beyond row_capacity are counted, not
 * written.  Row order is irrelevant: sbr_cir_select sorts by ordinal. */
int sbr_cir_visibility(const SbrScene* scene, const SbrCirParams* params,
                       const SbrVertexBuf* vb, int64_t v_begin, int64_t v_end,
                       const int32_t* order_dev, uint64_t* row_key_dev, int32_t* row_vtx_dev,
                       int64_t row_capacity, uint64_t* counters_dev, void* stream);
/* Per-row dedup keys (_emit_records paths.py:919-924): pair hashes
 * fnv1a(chain_hash_{round,floor}, seed=target) and the chain flag (no diffuse
 * step anywhere in the prefix and the row itself not diffuse). */
int sbr_cir_row_pairs(const SbrVertexBuf* vb, const uint64_t* row_key_dev,
                      const int32_t* row_vtx_dev, int64_t n, uint64_t* pr_dev, uint64_t* pf_dev,
                      uint8_t* chain_dev, void* stream);
/* Candidate selection with the reference's exact semantics
 * (_emit_records paths.py:903-987, DedupTable / PathBuffer 174-226,
 * generate_candidates 1019-1103 at workers=1) over rows given by ordinal key,
 * pair hashes and chain flag -- local rows, or rows all-gathered from every
 * rank (multi-GPU): ordinal sort, first occurrence of each (pair_r, pair_f)
 * among chain rows, per-depth truncation to n_buffer, LoS pre-claims, greedy
 * both-slot registration in a table of n_hash slots, buffer cap.
 * los_visible_dev: (n_targets) uint8, 1 = unoccluded.  Output rec_row_dev
 * (capacity n_buffer) in buffer order: index into the row arrays, or ~target
 * (< 0) for a LoS record; *n_records (host) receives the count.
 * Synchronises `stream`. */
int sbr_cir_select(const SbrCirParams* params, const uint64_t* row_key_dev,
                   const uint64_t* row_pr_dev, const uint64_t* row_pf_dev,
                   const uint8_t* row_chain_dev, int64_t n_rows, const uint8_t* los_visible_dev,
                   uint64_t n_hash, int64_t n_buffer, int64_t* rec_row_dev, int64_t* n_records,
                   uint64_t* counters_dev, void* stream);
/* Shard-local pre-selection for multi-GPU CIR (no reference counterpart: it
 * only shrinks the all-gather of compute_paths_sharded).  Keeps every
 * non-chain row and the first occurrence, in ordinal order, of each
 * (pr, pf) among this shard's chain rows; kept_idx_dev (n_rows) receives the
 * kept row indices ascending, *n_kept / *n_dup (host) the kept and dropped
 * counts.  Gathering only kept rows leaves sbr_cir_select's result unchanged;
 * add the dropped rows to SBR_CC_DUPLICATES.  Synchronises `stream`. */
int sbr_cir_local_dedup(const SbrCirParams* params, const uint64_t* row_key_dev,
                        const uint64_t* row_pr_dev, const uint64_t* row_pf_dev,
                        const uint8_t* row_chain_dev, int64_t n_rows, int64_t* kept_idx_dev,
                        int64_t* n_kept, uint64_t* n_dup, void* stream);
/* rec_row -> (vertex index, target) for sbr_cir_records (vertex -1 = LoS). */
int sbr_cir_resolve_records(const int64_t* rec_row_dev, int64_t n, const uint64_t* row_key_dev,
                            const int32_t* row_vtx_dev, int32_t* rec_vtx_dev,
                            int32_t* rec_target_dev, void* stream);
/* Walks vertex parent chains into CandidateRecord arrays
 * (_record_from_batch paths.py:990-1016). */
int sbr_cir_records(const SbrCirParams* params, const SbrVertexBuf* vb,
                    const int32_t* rec_vtx_dev, const int32_t* rec_target_dev, int64_t n,
                    const SbrRecordBuf* out, void* stream);
/* Image-method refinement (refine_candidate paths.py:1123-1252, D branch
 * out of scope): path_vertices_dev (n, L+2, 3) = [source, steps..., target],
 * status_dev (n) SBR_REFINE_*; rejection counters accumulated. */
int sbr_cir_refine(const SbrScene* scene, const SbrCirParams* params, const SbrRecordBuf* rec,
                   int64_t n, double* path_vertices_dev, int32_t* status_dev,
                   uint64_t* counters_dev, void* stream);
/* Field replay, Algorithm 2 (compute_path_fields paths.py:1302-1399 +
 * accumulate_doppler 1410-1426) for records with status OK: complex gain
 * (re, im), delay, doppler, departure / arrival directions. */
int sbr_cir_fields(const SbrScene* scene, const SbrFieldParams* params, const SbrRecordBuf* rec,
                   const double* path_vertices_dev, const int32_t* status_dev, int64_t n,
                   double* gain_dev, double* delay_dev, double* doppler_dev,
                   double* departure_dev, double* arrival_dev, void* stream);
/* Path count per link from which sbr_cfr contracts on the FP64 tensor cores
 * (mma.sync m8n8k4 f64; fused multiply-adds, ~1e-16 of max|H| from the
 * path-order sum) instead of the path-order SIMT kernel; < 0 disables it.
 * Default 16.  No reference counterpart. */
int sbr_set_cfr_dmma_min_paths(int64_t min_paths);
/* Channel frequency response of one link (frequency_response paths.py:1519-1547):
 * H[r, t, f] = sum_p a_p u_rx,r(arrival_p) u_tx,t(departure_p) e^{-j 2 pi f tau_p},
 * accumulated in path order in float64.  synthetic = 0: element-indexed paths
 * (path_rx_el / path_tx_el) add a_p e^{-j 2 pi f tau_p} to H[rx_el, tx_el]. */
int sbr_cfr(const double* gain_dev, const double* delay_dev, const double* departure_dev,
            const double* arrival_dev, const int32_t* path_rx_el_dev,
            const int32_t* path_tx_el_dev, int64_t n_paths, const double* freqs_dev,
            int32_t n_freq, const double* tx_offsets_dev, int32_t n_tx,
            const double* rx_offsets_dev, int32_t n_rx, double wavelength, int32_t synthetic,
            double* h_dev /* (n_rx, n_tx, n_freq) complex128 */, void* stream);

/* ---- misc ----------------------------------------------------------------- */
const char* sbr_last_error(void);
int sbr_version(void);
/* Number of CUDA kernels this library launched since load (evidence counter). */
uint64_t sbr_kernel_launches(void);
/* Per-kernel CUDA-event timing of the library's hot launches (bench.py uses it
 * for the roofline): enable (resets the accumulators) / query the summed
 * milliseconds and launch count of one kernel name (synchronises). */
int sbr_profile_enable(int on);
double sbr_profile_kernel_ms(const char* name, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* SBR_H */
