/*
 * svx.h -- C ABI of the B200-native SLIM-VDB integration engine (libsvx.so).
 *
 * This is the drop-in boundary for the reference's per-frame integration hot
 * path.  The reference (semvox, /root/reference/pkg) exposes that path through
 * a Python backend-module protocol (pkg/src/semvox/backend.py:1-7) whose
 * compiled member is the Cython GridCore + integrate_points
 * (pkg/src/semvox/_core.pyx:79-472, 621-858), driven by
 * semvox_bindings.Mapper (pkg/bindings/src/semvox_bindings/__init__.py:58-201).
 * Each entry point below cites the reference interface it replaces.
 *
 * Conventions
 *   - Plain C types only; no torch/CUDA types in signatures.  Streams are
 *     passed as `void*` (a cudaStream_t; NULL = the legacy default stream).
 *   - Input/output array pointers may be HOST or DEVICE memory: the library
 *     inspects each pointer and stages host buffers through device memory on
 *     the caller's stream.  Device pointers are borrowed for the call only.
 *   - Every call returns an svx_status.  On failure a thread-local message is
 *     available from svx_last_error().  Status codes map 1:1 onto the
 *     reference's exception classes (pkg/src/semvox/errors.py:4-25).
 *   - One host thread per map handle (the reference Mapper is
 *     "single-threaded from the scripting side", bindings/__init__.py:14-16).
 */
#ifndef SVX_H
#define SVX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVX_ABI_VERSION 1

/* Status codes -> semvox.errors classes (errors.py:4-25). */
typedef enum {
    SVX_OK = 0,
    SVX_E_CONFIG = 1,   /* ConfigError          (errors.py:12) */
    SVX_E_PAYLOAD = 2,  /* PayloadMismatchError (errors.py:16) */
    SVX_E_INPUT = 3,    /* UserInputError       (errors.py:8)  */
    SVX_E_RANGE = 4,    /* OutOfRangeError      (errors.py:24) */
    SVX_E_FORMAT = 5,   /* FormatError          (errors.py:20) */
    SVX_E_INTERNAL = 6, /* SemvoxError          (errors.py:4)  */
    SVX_E_CUDA = 7      /* SemvoxError (device failure; message carries the CUDA error) */
} svx_status;

/* Semantic payload kind (grid.py:26-28 KIND_TSDF/KIND_CLOSED/KIND_OPEN). */
enum { SVX_SEM_NONE = 0, SVX_SEM_CLOSED = 1, SVX_SEM_OPEN = 2 };

/* Element type codes for arrays crossing the boundary. */
enum { SVX_F32 = 0, SVX_F64 = 1 };
/* OR-ed into points_dtype / feats_dtype: every input array of the call is a
 * device pointer (skips the per-call pointer-attribute queries).  Without it
 * the library detects host arrays and stages them itself. */
#define SVX_DEVICE_INPUTS 0x100
/* OR-ed into points_dtype of svx_integrate: the library checks the pose
 * itself (finite, bottom row exactly [0 0 0 1], rotation rows orthonormal
 * within 0.5e-4, det > 0 -- the fast acceptance test of fusion.py:31-77) and
 * returns SVX_POSE_NEEDS_HOST, doing nothing, when the pose needs the host's
 * full validation (validate_rotation's polar fix or its error messages). */
#define SVX_POSE_CHECK 0x200
#define SVX_POSE_NEEDS_HOST 8

/*
 * Map construction parameters.  Mirrors the union of FusionConfig,
 * ClosedSetConfig and OpenSetConfig (config.py:36-110) as routed by
 * Mapper.__init__ (bindings/__init__.py:77-116); validation of the values
 * (messages included) happens on the host side before svx_create.
 */
typedef struct {
    double voxel_size;       /* FusionConfig.voxel_size */
    double truncation;       /* FusionConfig.truncation */
    double max_range;        /* FusionConfig.max_range  */
    int32_t weight_fn;       /* 0 constant_one, 1 linear_dropoff (fusion.py:270) */
    int32_t space_carving;   /* FusionConfig.space_carving */
    int32_t sem_kind;        /* SVX_SEM_* */
    int32_t num_classes;     /* ClosedSetConfig.num_classes (closed) */
    int32_t last_wins;       /* ClosedSetConfig.fusion == "last_wins" */
    int32_t count_dtype;     /* SVX_F32 / SVX_F64: ClosedSetConfig.count_dtype */
    int32_t feature_dim;     /* OpenSetConfig.feature_dim (open) */
    int32_t state_dtype;     /* SVX_F32 / SVX_F64: OpenSetConfig.state_dtype */
    double prior_beta;       /* OpenSetConfig.prior_beta (background of beta) */
    double lambda_floor;     /* OpenSetConfig.lambda_floor */
    int32_t tsdf_dtype;      /* SVX_F64: reference layout (grid.py:45-47, bit-exact);
                                SVX_F32: compact fp32 d/w (f64 math, f32 store) */
    int32_t device;          /* CUDA device ordinal */
    int64_t reserve_voxels;  /* initial voxel-pool capacity (0 = default) */
    int64_t reserve_blocks;  /* initial block-pool capacity (0 = default) */
} svx_config;

/*
 * Per-frame report.  Fields points_in..touched_voxels are
 * IntegrationReport (fusion.py:103-117); band_hits/touched_voxels follow the
 * reference's kernel report (_core.pyx:666,747).
 */
typedef struct {
    int64_t points_in;
    int64_t points_used;
    int64_t skipped_nonfinite;
    int64_t skipped_range;
    int64_t skipped_degenerate;
    int64_t skipped_bad_label;
    int64_t band_hits;
    int64_t touched_voxels;
    int64_t new_blocks;      /* leaves allocated by this frame */
    int64_t new_voxels;      /* voxels activated by this frame */
    double kernel_ms;        /* device time of the frame (CUDA events) */
} svx_report;

/* Map occupancy (grid.py:194-202 MemoryStats; evalbench.py:297-327). */
typedef struct {
    int64_t leaf_count;      /* allocated 8^3 blocks */
    int64_t active_voxels;
    int64_t resident_bytes;  /* device bytes held by live blocks + voxel payloads */
    int64_t payload_bytes_per_voxel;
    int64_t frames_integrated;
    int64_t hash_capacity;
    int64_t voxel_capacity;
    int64_t block_capacity;
    int64_t frames_slot_mode;     /* frames finished in slot mode (svx_set_update_mode) */
    int64_t slot_overflow_reruns; /* slot-mode attempts re-run in segment mode */
    int64_t async_reruns;         /* asynchronous frames re-run after an overflow */
    int64_t frames_leaf_mode;     /* frames finished in leaf mode */
    int64_t last_h2d_bytes;       /* host -> device bytes of the last frame's inputs */
    int64_t last_d2h_bytes;       /* device -> host bytes of the last frame's report */
} svx_stats;

typedef struct svx_map svx_map;

/* ---- lifetime ---------------------------------------------------------- */

/* Replaces make_grids (fusion.py:296-314) + GridCore.__init__ (_core.pyx:104-141). */
svx_status svx_create(const svx_config* cfg, svx_map** out);
svx_status svx_destroy(svx_map* map);
/* Pre-size the voxel and leaf pools (and the leaf hash) so later frames do
 * not pay pool growth (the reference grows by doubling, _core.pyx:154-183). */
svx_status svx_reserve(svx_map* map, int64_t voxels, int64_t blocks);

/* ---- integration ---------------------------------------------------------
 * Replaces integrate_frame (fusion.py:200-293) from the world transform on,
 * including backend.integrate_points (_core.pyx:621-858 / _pycore.py:449-539).
 *   points   (n,3) SVX_F32|SVX_F64, sensor frame
 *   pose     4x4 row-major sensor-to-world, already validated/orthonormalised
 *            on the host (fusion.py:31-77)
 *   labels   (n,) int32 class ids 1..k (closed) or NULL
 *   feats    (n,D) SVX_F32|SVX_F64 (open) or NULL
 * The transform is p_w = ((R0*x + R1*y) + R2*z) + t without FMA contraction
 * (identity rotations are exact, matching numpy's BLAS result).
 */
svx_status svx_integrate(svx_map* map, const void* points, int32_t points_dtype, int64_t n,
                         const double pose[16], const int32_t* labels, const void* feats,
                         int32_t feats_dtype, void* stream, svx_report* report);

/* Asynchronous integrate_frame (fusion.py:200-293) for closed-set and
 * geometry maps: enqueues the frame on `stream` and returns at once with a
 * ticket; svx_report_wait(ticket) gives its IntegrationReport.  Same inputs,
 * results and errors as svx_integrate -- a frame goes asynchronous only when
 * none of the reference's frame errors (step budget, 2^21 extent, +/-2^30
 * range, _core.pyx:661-712) can occur for it, which a finite max_range and
 * bounded bands (no space carving) decide from the configuration and the
 * origin; otherwise the frame runs synchronously and its report is held for
 * the ticket the same way.  Host input arrays have been read when the call
 * returns; device inputs are copied on the device by the frame itself (a
 * frame stopped by a pool or slot overflow is re-run from that copy).  Every
 * other entry point first finishes the frames in flight, so it sees the map
 * after all of them.  At most svx_set_async frames (default 2, max 4)
 * are in flight (svx_set_async); the last 64 reports are held. */
svx_status svx_integrate_async(svx_map* map, const void* points, int32_t points_dtype, int64_t n,
                               const double pose[16], const int32_t* labels, void* stream,
                               uint64_t* ticket);
svx_status svx_report_wait(svx_map* map, uint64_t ticket, svx_report* report);
/* depth: frames in flight (0 = every frame synchronous, at most 4).
 * leaf_headroom: leaf-pool room kept per frame in flight (0 = automatic:
 * twice the most leaves a recent frame created, at least 4096); a frame that
 * still runs out is re-run as described above. */
svx_status svx_set_async(svx_map* map, int32_t depth, int64_t leaf_headroom);

/* Same, for points already in the world frame with the sensor origin given:
 * the reference's backend seam (fusion.py:229-263 -> integrate_points), where
 * delta = p - origin, t = sqrt((dx*dx + dy*dy) + dz*dz), u = delta / t. */
svx_status svx_integrate_world(svx_map* map, const void* points_world, int32_t points_dtype,
                               int64_t n, const double origin[3], const int32_t* labels,
                               const void* feats, int32_t feats_dtype, void* stream,
                               svx_report* report);

/* ---- snapshots ------------------------------------------
 * Load a map state into an EMPTY map: leaves in the snapshot's order become
 * leaf ids 0..nl-1 (the reference's allocation order, grid.py:372-426
 * read_grid_block), voxels in (leaf, slot) order become voxel ids 0..nv-1.
 *   leaf_coords (nl, 3) int32 leaf coordinates (voxel >> 3)
 *   voxel_leaf  (nv,) int32 leaf index of each voxel, non-decreasing
 *   voxel_slot  (nv,) int32 slot (x&7)<<6 | (y&7)<<3 | (z&7), ascending within a leaf
 *   d, w        (nv,) f64 TSDF; sem0 / sem1 (nv, C|D) in the map's storage dtype (or NULL)
 * Host or device arrays.  The file format itself is written and parsed on the
 * host (paper_2512_12945_b200/snapshot.py). */
svx_status svx_import(svx_map* map, int64_t nl, const int32_t* leaf_coords, int64_t nv,
                      const int32_t* voxel_leaf, const int32_t* voxel_slot, const double* d,
                      const double* w, const void* sem0, const void* sem1, void* stream);

/* ---- surface extraction ---------------------------------
 * Mapper.extract = extract_mesh (mesh.py:419-545) on the device map.
 * svx_extract_mesh triangulates the D = 0 level set over voxels with weight
 * >= min_weight and keeps the mesh on the device; *n_vertices / *n_triangles
 * get its size.  emb (k, D) f64: open-set vertex labels by classify_means
 * (temperature, confidence_threshold); NULL = the dominant feature axis
 * (voxel_labels, mesh.py:392-416).  Fails with SVX_E_RANGE when the kept
 * voxels span more than 2^20 voxels on an axis (mesh.py:461-466).
 * svx_mesh_read copies the last mesh out (host or device pointers, any may be
 * NULL): vertices (nv,3) f64, triangles (nt,3) int32, labels (nv,) int32,
 * colors (nv,3) u8 = palette row of the label (palette_colors,
 * mesh.py:382-389; palette (npal,3) u8, npal >= 2). */
svx_status svx_extract_mesh(svx_map* map, double min_weight, const double* emb, int32_t k,
                            double temperature, double confidence_threshold, int64_t* n_vertices,
                            int64_t* n_triangles, void* stream);
svx_status svx_mesh_read(svx_map* map, double* vertices, int32_t* triangles, int32_t* labels,
                         uint8_t* colors, const uint8_t* palette, int32_t npal, void* stream);

/* ---- rendering ------------------------------------------
 * render (render.py:214-272) = ray-march of the device map from a pinhole
 * camera (RenderCamera, render.py:33-85: x right, y down, z forward; pose =
 * camera-to-world 4x4 row-major with a validated rotation).  Outputs, row-major
 * pixels, background 0:
 *   SVX_RENDER_DEPTH    (H, W) f64 distance along the ray
 *   SVX_RENDER_SEMANTIC (H, W, 3) u8 palette colour of the nearest voxel's label
 *                       (palette (npal,3) u8, npal >= 2; emb (k, D) f64 labels
 *                       open-set maps by classify_means, NULL = dominant axis)
 *   SVX_RENDER_NORMAL   (H, W, 3) f64 unit outward normal (central differences)
 * `out` may be a host or device pointer. */
#define SVX_RENDER_DEPTH 0
#define SVX_RENDER_SEMANTIC 1
#define SVX_RENDER_NORMAL 2

typedef struct svx_render_camera {
    double pose[16];
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
} svx_render_camera;

svx_status svx_render(svx_map* map, const svx_render_camera* camera, int32_t mode,
                      const double* emb, int32_t k, double temperature,
                      double confidence_threshold, const uint8_t* palette, int32_t npal, void* out,
                      void* stream);

/* sample_distance (render.py:88-113): trilinear D at n world points (n,3) f64;
 * valid[i] = 0 and vals[i] = NaN where a surrounding voxel centre is inactive. */
svx_status svx_sample_distance(svx_map* map, const double* points, int64_t n, double* vals,
                               uint8_t* valid, void* stream);

/* ---- depth frames ---------------------------------------
 * Replaces ingest.project_depth (ingest.py:285-322) followed by integrate on
 * the returned Frame: pixel (u, v) of the raster, sampled every `stride`
 * pixels from (0, 0), with depth d > 0 and finite maps to the sensor-frame
 * point (((u - cx) * d) / fx, ((v - cy) * d) / fy, d) * depth_scale, in f64;
 * the payload raster gives the point's label (int32, (H, W)) or features
 * ((H, W, D), SVX_F32 | SVX_F64).  Invalid pixels are not points (they do not
 * count in points_in or any skip counter), exactly as project_depth drops them.
 * depth_dtype: SVX_F32, SVX_F64 or SVX_U16.  Camera validation follows
 * CameraConfig.validate (config.py:126-134) -> SVX_E_CONFIG. */
enum { SVX_U16 = 2 };
typedef struct {
    double fx, fy, cx, cy;
    double depth_scale;
    int32_t width, height;
    int32_t stride;
    int32_t pad;
} svx_camera;
svx_status svx_integrate_depth(svx_map* map, const void* depth, int32_t depth_dtype,
                               const svx_camera* camera, const double pose[16],
                               const int32_t* labels, const void* feats, int32_t feats_dtype,
                               void* stream, svx_report* report);

/* ---- sharded integration (no reference counterpart) -----------
 * A map sharded over G ranks (one GPU each): rank r holds the leaves with
 * svx_leaf_owner(leaf, G) == r.  Each frame is split into G contiguous point
 * slices; rank r marches slice r and a frame takes four calls per rank with
 * two host collectives in between, done by the caller's transport
 * (torch.distributed over NCCL, or gloo):
 *
 *   svx_shard_march   march this rank's slice (masks, fp64 band walk) and
 *                     fill its local summary
 *   -- all-reduce the summaries: counters summed, bbox_min min, bbox_max and
 *      flags max
 *   svx_shard_plan    apply the reference's frame checks to the global
 *                     summary (every rank fails identically, before any map
 *                     mutation); bucket this rank's rows by owning rank and
 *                     return the send size per destination.  *remarch = 1
 *                     asks for svx_shard_march again with key_base =
 *                     global bbox_min (packed-key window overflow).
 *   svx_shard_pack    write the send buffer: per destination, the points
 *                     that have rows there (ray direction, distance, label or
 *                     feature) and the rows (voxel key, point)
 *   -- all-to-all of the sizes, then of the buffers (rank order)
 *   svx_shard_apply   resolve, group and update the received rows -- this
 *                     rank's leaves only -- exactly as svx_integrate does.
 *
 * Points keep their global order (slices are contiguous and concatenated in
 * rank order), so every voxel's rows are reduced in the reference's
 * (voxel, point) order and the union of the shards equals the single-GPU map
 * bit for bit.  svx_export_leaf_stamps gives the keys that merge the shards'
 * active lists into the reference's global active order. */
#define SVX_MAX_SHARDS 16

typedef struct svx_shard_summary {
    int64_t points_in;     /* slice sizes (summed) */
    int64_t nonfinite, range, degenerate, bad_label, used, band_hits, rows; /* summed */
    int64_t bbox_min[3];   /* min over ranks (INT64_MAX when no rows) */
    int64_t bbox_max[3];   /* max over ranks (INT64_MIN when no rows) */
    int64_t err_budget;    /* max over ranks */
    int64_t err_pack;      /* max over ranks */
} svx_shard_summary;

int32_t svx_leaf_owner(int64_t bx, int64_t by, int64_t bz, int32_t nranks);

/* pose (4x4, sensor-frame points) or, when pose is NULL, origin (world-frame
 * points, svx_integrate_world semantics).  Slice r must hold the frame's
 * points [n*r/G, n*(r+1)/G) (any contiguous split in rank order works).
 * key_base NULL = the default packed-key window.  All four calls of a frame
 * must use the same stream. */
svx_status svx_shard_march(svx_map* map, const void* points, int32_t points_dtype, int64_t n,
                           const double pose[16], const double origin[3],
                           const int32_t* labels, const void* feats, int32_t feats_dtype,
                           const int64_t key_base[3], void* stream, svx_shard_summary* local);
svx_status svx_shard_plan(svx_map* map, const svx_shard_summary* global, int32_t rank,
                          int32_t nranks, int64_t* send_bytes, int32_t* remarch);
/* send: device buffer of at least sum(send_bytes) bytes, 16-byte aligned. */
svx_status svx_shard_pack(svx_map* map, void* send, int64_t capacity, void* stream);
/* recv: device buffer holding recv_bytes[s] bytes from each source s, in
 * rank order, 16-byte aligned. */
svx_status svx_shard_apply(svx_map* map, const void* recv, const int64_t* recv_bytes,
                           int32_t nranks, void* stream, svx_report* report);

/* Device-planned frames: the same four phases with every size and check kept
 * on the device, so a frame takes exactly one host synchronisation (after
 * its last collective) instead of one per phase.  The caller's transport
 * runs, on the same stream and without reading anything back:
 *
 *   svx_shard_march_async   march the slice; write the local summary vector
 *                           (SVX_SHARD_SUMMARY_WORDS int64, device memory)
 *   -- all-reduce: words [0, SVX_SHARD_SUM_WORDS) summed, the rest max
 *   svx_shard_plan_async    the frame checks on the global summary into the
 *                           device abort vector (SVX_SHARD_ABORT_WORDS int64);
 *                           bucket the rows by owner into sections of a fixed
 *                           capacity `cap` bytes per destination
 *   svx_shard_pack_async    write the sections (send: nranks * cap bytes)
 *   -- all-reduce (max) of the abort vector; all-to-all of equal cap-byte
 *      blocks (no size exchange)
 *   svx_shard_apply_async   K2-K5 on the received sections, or nothing when
 *                           the frame is aborted; writes 4 report words
 *                           (touched, new leaves, new voxels, redo flag)
 *   -- optional all-reduce (sum) of the report words
 *   -- the one host synchronisation: read back summary, abort, report
 *   svx_shard_finish        raise the frame's error (same messages as
 *                           svx_shard_plan, on every rank), or *action:
 *                           0 done; 1 redo the frame on every rank (key
 *                           rebase to the summary's bbox minimum, larger
 *                           scratch, or *need bytes of section capacity);
 *                           2 redo this rank's apply (scratch / pools grown;
 *                           nothing was changed); 3 done here, but another
 *                           rank redoes its apply: repeat the report sum.
 * A frame aborted on the device changes no map: the checks run before any
 * rank's K2. */
#define SVX_SHARD_SUM_WORDS 10
#define SVX_SHARD_SUMMARY_WORDS 18
#define SVX_SHARD_ABORT_WORDS 8
svx_status svx_shard_march_async(svx_map* map, const void* points, int32_t points_dtype, int64_t n,
                                 const double pose[16], const double origin[3], const int32_t* labels,
                                 const void* feats, int32_t feats_dtype, const int64_t key_base[3],
                                 void* stream, int64_t* summary);
svx_status svx_shard_plan_async(svx_map* map, const int64_t* global_summary, int32_t rank,
                                int32_t nranks, int64_t cap, void* stream, int64_t* abort_words);
svx_status svx_shard_pack_async(svx_map* map, void* send, int64_t cap, void* stream,
                                const int64_t* abort_words);
/* frame_points: the whole frame's point count (bounds the received points). */
svx_status svx_shard_apply_async(svx_map* map, const void* recv, int64_t cap, int32_t nranks,
                                 const int64_t* abort_words, int64_t frame_points, void* stream,
                                 int64_t* report_words);
/* Host copies of the reduced summary / abort words and (NULL when the caller
 * did not sum them) the summed report words. */
svx_status svx_shard_finish(svx_map* map, const int64_t* summary, const int64_t* abort_words,
                            const int64_t* report_sum, svx_report* report, int32_t* action,
                            int64_t* need);

/* Per leaf, in this map's active (leaf) order: creation frame, the leaf's
 * smallest packed key in that frame, and its active voxel count.  Sorting
 * the concatenated shards' leaves by (frame, key) gives the global order. */
svx_status svx_export_leaf_stamps(svx_map* map, int64_t capacity, int32_t* frame, uint64_t* key,
                                  int32_t* count, int64_t* nleaves, void* stream);

/* ---- queries ---------------------------------------------------------------
 * Active order is leaf-allocation then slot order, identical to
 * GridCore.active_slots (_core.pyx:424-444) + slots_to_coords (:446-463).
 */
svx_status svx_stats_get(svx_map* map, svx_stats* out);
svx_status svx_active_count(svx_map* map, int64_t* count);

/* SparseGrid.active_values (grid.py:163-168).  Outputs (any may be NULL):
 *   coords (count,3) int64; d, w (count,) in tsdf_dtype; sem0 (count,C|D) and
 *   sem1 (count,D) in count_dtype/state_dtype.  `capacity` = rows the buffers
 *   hold; fails with SVX_E_INPUT if smaller than the active count. */
svx_status svx_export_active(svx_map* map, int64_t capacity, int64_t* coords, void* d, void* w,
                             void* sem0, void* sem1, void* stream);

/* SparseGrid.probe_many (grid.py:176-190) via GridCore.probe_coords
 * (_core.pyx:324-375): background values where inactive; never allocates. */
svx_status svx_probe(svx_map* map, const int64_t* coords, int64_t m, void* d, void* w,
                     void* sem0, void* sem1, uint8_t* active, void* stream);

/* Mapper.query (bindings/__init__.py:153-169) = cosine_to_embeddings
 * (gaussian.py:158-170) of every active mean against one query (D,) f64;
 * sims (count,) f64 in active order, NaN where the mean is all zero. */
svx_status svx_query_cosine(svx_map* map, const double* query, int64_t capacity, double* sims,
                            void* stream);

/* classify_means (gaussian.py:132-155) over all active voxels, weights = the
 * TSDF weight (mesh.py:419-445).  emb (k,D) f64.  labels (count,) int32
 * (0 = reject), best (count,) f64; sims (count,k) f64 optional. */
svx_status svx_classify(svx_map* map, const double* emb, int32_t k, double temperature,
                        double confidence_threshold, int64_t capacity, int32_t* labels,
                        double* best, double* sims, void* stream);

/* Score path of svx_classify: 0 = auto (the exact int8 split GEMM on the
 * tcgen05 tensor cores for more than 64 queries with f32 means, the FP64 DMMA
 * kernel otherwise), 1 = DMMA, 2 = tcgen05 (f32 means; else DMMA).  All give
 * labels equal to the reference's and scores within f64 rounding of it. */
svx_status svx_set_score_path(svx_map* map, int32_t path);

/* Closed-set readout over active voxels: mode 0 = dirichlet.label_map
 * (argmax+1, ties to lowest, dirichlet.py:81-88); mode 1 = evalbench.grid_labels
 * (0 when all counts are zero, evalbench.py:30-55). */
svx_status svx_label_map(svx_map* map, int32_t mode, int64_t capacity, int32_t* labels,
                         void* stream);

/* ---- diagnostics --------------------------------------------------------- */
/* Per-kernel device timing of integrate calls.  With profiling on, each kernel
 * of the frame graph records its span [first CTA start, last warp end] with
 * %globaltimer (the graph, caches and programmatic overlap are unchanged).
 * Entries, in order (ms; 0 when the kernel did not run):
 *   0 walk     (K1: masks + fp64 band walk -> row keys; gate)
 *   1 resolve  (K2: rows -> leaf/voxel ids, per-voxel counts)
 *   2 seg      (K3: row segments; segment mode)
 *   3 scatter  (K4: rows into segments; segment mode)
 *   4 update   (K5: slot update, short segments, or open-set voxels)
 *   5 update_b (K5: long and huge segments)
 *   6 frame    (first kernel start to last kernel end)
 * svx_stage_times writes up to n last-frame values and returns SVX_N_STAGES. */
#define SVX_N_STAGES 7
svx_status svx_set_profiling(svx_map* map, int32_t enable);

/* Row-grouping strategy of closed-set / geometry maps with bounded bands.
 *   SVX_UPDATE_AUTO      slot mode while recent frames average <= 3 rows per
 *                        touched voxel (LiDAR), segment mode otherwise
 *   SVX_UPDATE_SEGMENTS  always segments (K3 scan, K4 scatter, K5 sorted update)
 *   SVX_UPDATE_SLOTS     always try slot mode (K2 writes point indices into the
 *                        voxel's 16-entry slot record; K5 per touched voxel)
 *   SVX_UPDATE_LEAVES    always try leaf mode (rows binned by 8^3 leaf; one warp
 *                        or CTA per touched leaf sorts its rows in shared memory
 *                        and updates its voxels)
 * A slot-mode frame with a voxel of more than 16 rows, or a leaf-mode frame
 * with a leaf of more than 8192 rows, stops before any payload changes and is
 * re-run in segment mode, so all four give identical maps.
 * Open-set and space-carving maps always use segments.  The reference has no
 * equivalent knob (its grouping is one sort, _core.pyx:707-753). */
#define SVX_UPDATE_AUTO 0
#define SVX_UPDATE_SEGMENTS 1
#define SVX_UPDATE_SLOTS 2
#define SVX_UPDATE_LEAVES 3
svx_status svx_set_update_mode(svx_map* map, int32_t mode);
int32_t svx_stage_times(svx_map* map, double* ms, int32_t n);
/* Diagnostics: the last finished frame's internal counters, in this order:
 * rows, touched voxels, listed leaves (leaf mode), leaves taken by the CTA
 * path (leaf mode), long voxels, huge voxels.  Writes up to n, returns 6. */
int32_t svx_frame_counters(svx_map* map, int64_t* out, int32_t n);

const char* svx_last_error(void);
int32_t svx_abi_version(void);
/* Number of kernels this library launched since load (evidence counter). */
int64_t svx_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SVX_H */
