/*
 * nif_b200.h -- C-ABI of the B200 Neural Intersection Function engine.
 *
 * Plain pointers and sizes only: no torch, no C++ types. Every function
 * returns an int status (NIF_OK == 0); on failure nif_last_error() holds a
 * one-line message whose wording follows the reference's exception text so
 * the Python shim can re-raise the same exception type.
 *
 * Device-pointer entry points ("_dev") are stream-ordered and asynchronous:
 * all array arguments are device pointers and the work is enqueued on
 * `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 * Host-pointer entry points ("_host") copy in, compute and copy out
 * synchronously.
 *
 * Each entry point names the reference function it replaces
 * (paths relative to the reference package root pkg/src/niftrace/).
 */
#ifndef NIF_B200_H
#define NIF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ----------------------------------------------------------- */
#define NIF_OK 0
#define NIF_ERR_VALUE 1       /* reference raises ValueError            */
#define NIF_ERR_TYPE 2        /* reference raises TypeError             */
#define NIF_ERR_CUDA 3        /* device / driver failure (RuntimeError) */
#define NIF_ERR_UNSUPPORTED 4 /* configuration this build cannot run    */

const char* nif_last_error(void);
int nif_abi_version(void);
/* 1 when the library was built for and runs on an sm_100a device. */
int nif_device_check(int device);

/* ---- scene ------------------------------------------------------------
 * Flat two-level BVH, packed once per scene (bvh.py:958-1045 ScenePack).
 * nif_node is 64 bytes: the slab box followed by the child/leaf words.
 *   leaf == 1: a = first triangle slot, b = triangle count
 *   leaf == 0: a = left child, b = right child (global node indices)     */
typedef struct nif_node {
  double lo[3];
  double hi[3];
  int32_t a;
  int32_t b;
  int32_t leaf;
  int32_t pad;
} nif_node;

typedef struct nif_scene_view {
  int32_t n_obj;
  int32_t pad0;
  int64_t n_nodes;
  int64_t n_tris;
  double eps;               /* epsilon_t = 1e-4 * diagonal (renderer.py:424) */
  double tol;               /* containment tolerance 1e-6 (renderer.py:631)  */
  const double* obox;       /* [n_obj][6] = lo.xyz, hi.xyz (pack.obox_lo/hi)   */
  const int32_t* t_order;   /* [n_obj] top-level leaf order (DFS order)        */
  const int32_t* roots;     /* [n_obj] root node of each object                */
  const nif_node* nodes;    /* [n_nodes]                                       */
  const double* tris;       /* [n_tris][9] v0.xyz v1.xyz v2.xyz (leaf order)   */
  const double* normals;    /* [n_tris][9] n0 n1 n2 (closest-hit shading)      */
  const double* obj_albedo; /* [n_obj][3] (optional, shading)                  */
  const nif_node* top_nodes; /* [n_top] top-level tree, leaf a/b index top_order */
  const int32_t* top_order;  /* [n_obj] top-level leaf slots -> object id        */
  int64_t n_top;
} nif_scene_view;

/* Binned SAH build, node-for-node identical to bvh.py:34-303 (_build_sah).
 * lo/hi/ce: [n][3]; outputs sized for 2n nodes; order: [n]. Host memory. */
int nif_build_sah(const double* lo, const double* hi, const double* ce, int64_t n,
                  int64_t max_leaf, int64_t n_bins, double c_trav, double c_isect,
                  double* node_lo, double* node_hi, int64_t* node_a, int64_t* node_b,
                  uint8_t* node_leaf, int64_t* order, int64_t* n_nodes_out);

/* The same build on the GPU (level-synchronous; a warp, a CTA or a chunked
 * multi-CTA pass per node by segment size), node-for-node identical to
 * nif_build_sah / bvh.py:34-303: lo/hi/ce and every output are DEVICE
 * arrays (outputs sized for 2n nodes), n_nodes_out is host memory.
 * workspace: nif_build_sah_workspace_bytes(n) bytes of device memory, or
 * NULL to allocate per call. Synchronises `stream` (one host round trip per
 * tree level). Serves build_bottom / build_top (bvh.py:400-437) when the
 * primitive bounds are already resident. */
size_t nif_build_sah_workspace_bytes(int64_t n);
int nif_build_sah_dev(const double* lo, const double* hi, const double* ce, int64_t n,
                      int64_t max_leaf, int64_t n_bins, double c_trav, double c_isect,
                      double* node_lo, double* node_hi, int64_t* node_a, int64_t* node_b,
                      uint8_t* node_leaf, int64_t* order, int64_t* n_nodes_out,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- phase 1: gather (bvh.py:772-901 _k_gather_queries,
 *                       renderer.py:613-644 gather_queries) --------------
 * Rays use the reference layout: origins/dirs [n][3] f64, tmaxs [n] f64.
 * route: [n_obj] u8 (1 = answered by the network, 0 = own tree).
 *
 * Pass A counts records per ray and resolves routed-away objects into
 * bvh_occ; pass B writes the records in the reference order (ray-major,
 * top-level DFS order within a ray). Offsets come from an exclusive scan
 * run between the passes inside nif_gather_dev.
 *
 * Records are written twice-shaped:
 *  - family queues (hot path): outer {obj, ray, coord4 f32[4]} and inner
 *    {obj, ray, coord4 f32[4], r f32}; totals in counts_dev[0..1].
 *  - optionally the reference's interleaved QueryRecords arrays
 *    (kind u8, obj i32, ray i32, coord f64[5]) when rec_kind != NULL.
 * Capacity arguments bound the writes; counts_dev always holds the true
 * totals so the caller can detect overflow.                              */
typedef struct nif_gather_out {
  int32_t* outer_obj;
  int32_t* outer_ray;
  float* outer_coord;   /* [cap_outer][4]: p_u p_v d_u d_v              */
  int32_t* inner_obj;
  int32_t* inner_ray;
  float* inner_coord;   /* [cap_inner][4]                               */
  float* inner_r;       /* [cap_inner]                                  */
  int64_t cap_outer;
  int64_t cap_inner;
  uint8_t* rec_kind;    /* optional interleaved view, [cap_total]       */
  int32_t* rec_obj;
  int32_t* rec_ray;
  double* rec_coord;    /* [cap_total][5]                               */
  int64_t cap_total;
  uint8_t* bvh_occ;     /* [n] hybrid (route == 0) any-hit result       */
  int64_t* counts;      /* [4]: n_outer, n_inner, n_total, n_degenerate */
} nif_gather_out;

/* The workspace (nif_gather_workspace_bytes) must be zero-filled before its
 * first use and not shared by concurrent gathers: the hot-path kernel keeps
 * its counters in it and re-arms them itself (no memset per call).     */
size_t nif_gather_workspace_bytes(int64_t n_rays);
int nif_gather_dev(const nif_scene_view* scene, const uint8_t* route_dev,
                   const double* origins, const double* dirs, const double* tmaxs,
                   int64_t n, const nif_gather_out* out, void* workspace,
                   size_t workspace_bytes, void* stream);

/* ---- labels and the BVH comparator ------------------------------------
 * nif_label_visible_dev: bvh.py:904-916 _k_label_visible -- per record,
 * any-hit in that record's object only, t in (eps, tmax); 1 = visible.
 * fp64, no FMA contraction, reference operation order: bit-exact.
 * nif_bvh_occluded_dev: bvh.py:744-756 _k_occluded (BvhBackend.occluded,
 * renderer.py:598-610), the two-level any-hit comparator.               */
int nif_label_visible_dev(const nif_scene_view* scene, const int32_t* rec_obj,
                          const int32_t* rec_ray, int64_t m, const double* origins,
                          const double* dirs, const double* tmaxs, uint8_t* out_vis,
                          void* stream);
int nif_bvh_occluded_dev(const nif_scene_view* scene, const double* origins,
                         const double* dirs, const double* tmaxs, int64_t n,
                         uint8_t* out_occ, void* stream);

/* ---- model ------------------------------------------------------------
 * One network family (outer or inner) of a NifModel (nif.py:173-255).
 * Latent tables are fp32 masters laid out like the reference arrays
 * latents[u_idx][v_idx][n] per object; MLP weights are the _flat_mlp
 * concatenation (nif.py:362-367) per head (1 head when sharing=shared). */
#define NIF_FAMILY_OUTER 0
#define NIF_FAMILY_INNER 1
#define NIF_MAX_LAYERS 8

typedef struct nif_family_view {
  int32_t family;
  int32_t n_obj;
  int32_t R, N;          /* 2D grid resolution / latents (pos and dir)   */
  int32_t Rd, Nd;        /* 1D distance grid (inner); 0 for outer        */
  int32_t n_layers;      /* dense layers = hidden_layers + 1             */
  int32_t dims[NIF_MAX_LAYERS + 1];
  int32_t n_heads;       /* 1 (shared) or n_obj (per_object)             */
  int32_t sigmoid_head;  /* 1 occlusion, 0 geometry (identity)           */
  int32_t w_stride;      /* floats of weights per head                   */
  int32_t b_stride;      /* floats of biases per head                    */
  const float* pos;      /* [n_obj][R][R][N]                             */
  const float* dir;      /* [n_obj][R][R][N]                             */
  const float* dist;     /* [n_obj][Rd][Nd] or NULL                      */
  const float* w;        /* [n_heads][w_stride]                          */
  const float* b;        /* [n_heads][b_stride]                          */
  const void* fast;      /* device blob from nif_fast_pack_dev or NULL   */
} nif_family_view;

/* Feature encoding (nif.py:286-311 encode_*_arrays; grids.py:125-206).
 * coord: [m][4] (outer) or [m][5] (inner) f64; out: [m][in_dim] f64 holding
 * fp32-rounded values, weights in fp64 exactly as the reference.        */
int nif_encode_dev(const nif_family_view* f, const int64_t* obj, const double* coord,
                   int64_t m, double* out, void* stream);

/* Row-sequential dense forward, fp32 weights / fp64 accumulation
 * (nif.py:321-359 _k_dense_forward). x: [m][in_dim] f64, out: [m][out] f64.
 * sigmoid_head overrides the family's head (0 -> logits).              */
int nif_forward_dev(const nif_family_view* f, const int64_t* obj, const double* x,
                    int64_t m, int32_t sigmoid_head, double* out, void* stream);

/* ---- fast fused query path (tcgen05 / TMEM) ---------------------------
 * nif_fast_pack_dev builds the fp16 tables and the UMMA-canonical fp16
 * weight tiles from the fp32 masters (re-run after every optimizer step
 * the renderer wants to see). nif_query_dev runs encode + MLP + threshold
 * for one family queue and ORs occlusion into occ_ray[ray] (NULL: skip);
 * logits (NULL: skip) receives the fp32 head output per record. The
 * record count is read on the device from count_dev (no host sync).    */
size_t nif_fast_pack_bytes(const nif_family_view* f);
int nif_fast_pack_dev(const nif_family_view* f, void* blob, void* stream);
int nif_query_dev(const nif_family_view* f, const int32_t* obj, const int32_t* ray,
                  const float* coord4, const float* r, const int64_t* count_dev,
                  int64_t capacity, uint8_t* occ_ray, float* logits, int32_t impl,
                  void* stream);
/* Split variant: a standalone grid-encoding kernel writes 16 fp16 features
 * per record (32 B, row-major) into feat (nif_feat_scratch_bytes of
 * capacity), then the tcgen05 MLP kernel (A operand in TMEM) reads them
 * row by row. flags: bit 1 runs only the encoding kernel, bit 2 only the
 * MLP kernel (over features already in feat) -- for per-stage timing.  */
size_t nif_feat_scratch_bytes(int64_t capacity);
int nif_query_split_dev(const nif_family_view* f, const int32_t* obj, const int32_t* ray,
                        const float* coord4, const float* r, const int64_t* count_dev,
                        int64_t capacity, uint8_t* occ_ray, float* logits, void* feat,
                        int32_t flags, void* stream);
/* per_object sharing (one MLP per object, nif.py:91-92, 380-397) on the
 * tensor cores: the queue is counting-sorted by object into 128-row tiles
 * (padding rows inert) inside scratch (nif_bucket_scratch_bytes), then the
 * TMEM-operand kernel runs each tile with its object's weights. Same
 * outputs as nif_query_dev; without bucketing per-object MLPs run on the
 * SIMT kernel. The scratch must be zero-filled before its first use and
 * not shared by concurrent calls (the histogram is re-zeroed in place). */
size_t nif_bucket_scratch_bytes(int64_t capacity, int32_t n_obj);
int nif_query_bucketed_dev(const nif_family_view* f, const int32_t* obj, const int32_t* ray,
                           const float* coord4, const float* r, const int64_t* count_dev,
                           int64_t capacity, uint8_t* occ_ray, float* logits, void* scratch,
                           void* stream);
#define NIF_IMPL_AUTO 0
#define NIF_IMPL_SIMT 1    /* fp32 CUDA-core reference kernel */
#define NIF_IMPL_TCGEN05 2 /* fused tcgen05/TMEM fp16 kernel (shape-specialised
                              when instantiated, else generic) */
#define NIF_IMPL_TCGEN05_GENERIC 3 /* force the runtime-shape tcgen05 kernel */

/* occ_ray |= bvh_occ (renderer.py:680-683 seeds the OR with bvh_occ).  */
int nif_occ_init_dev(const uint8_t* bvh_occ, int64_t n, uint8_t* occ_ray, void* stream);

/* ---- training (nif.py:682-749 _train_batch, mlp.py:82-167,
 *      grids.py:31-56 / 171-202) ------------------------------------------
 * One family's optimiser state. params/grad/m/v are flat fp32 buffers of
 * identical layout; the family view's pos/dir/dist/w/b point into params
 * at the given element offsets. Step counters are per object grid set and
 * per MLP head (every tensor of a set steps together in the reference). */
typedef struct nif_train_view {
  float* params;
  float* grad;
  float* m;
  float* v;
  int64_t numel;
  int64_t off_pos, off_dir, off_dist, off_w, off_b;
  int64_t* grid_steps;  /* [n_obj]   */
  int64_t* mlp_steps;   /* [n_heads] */
  int32_t* counts;      /* [n_obj] rows per object in the current batch */
} nif_train_view;

/* Per-object row counts of one (global) batch: counts[o] = #{r: obj[idx[r]] == o}
 * (idx NULL: identity). The reference normalises each object group's
 * loss by its own size (nif.py:686-692, mlp.py:166).                    */
int nif_batch_counts_dev(const int64_t* obj, const int64_t* idx, int64_t n_rows, int32_t n_obj,
                         int32_t* counts, void* stream);

/* Fused forward + L2 loss + backward for rows idx[row0 + k*row_step]
 * (data-parallel ranks take interleaved rows of the global batch).
 * Accumulates MLP and grid gradients into t->grad and the sum of squared
 * errors into *sq_err (device fp64). coord: [n][4|5] f64, label: [n] f32. */
int nif_train_fwdbwd_dev(const nif_family_view* f, const nif_train_view* t, const int64_t* obj,
                         const double* coord, const float* label, const int64_t* idx,
                         int64_t n_rows, int64_t row0, int64_t row_step, double* sq_err,
                         void* stream);

/* Graph-replayable variants: the batch's rows start at idx + *cursor
 * (cursor: device int64), advanced on the device by nif_cursor_advance_dev,
 * so one captured optimiser step is replayed for every full batch.      */
int nif_batch_counts_cur_dev(const int64_t* obj, const int64_t* idx, const int64_t* cursor,
                             int64_t n_rows, int32_t n_obj, int32_t* counts, void* stream);
int nif_train_fwdbwd_cur_dev(const nif_family_view* f, const nif_train_view* t,
                             const int64_t* obj, const double* coord, const float* label,
                             const int64_t* idx, const int64_t* cursor, int64_t n_rows,
                             int64_t row0, int64_t row_step, double* sq_err, void* stream);
int nif_cursor_advance_dev(int64_t* cursor, int64_t delta, void* stream);
/* The three-launch step of a captured graph: prologue (one CTA: this
 * batch's per-object counts, overwritten, plus the Adam step counters of
 * the touched objects / heads), nif_train_fwdbwd_cur_dev, then the dense
 * update alone (nif_adam_dev minus its step-counter and count-clearing
 * kernels), which also advances the cursor by delta (cursor may be NULL).
 * Counts are left holding the last batch's: clear them before using the
 * accumulate-style nif_batch_counts_dev again.                             */
int nif_train_prologue_cur_dev(const nif_family_view* f, const nif_train_view* t,
                               const int64_t* obj, const int64_t* idx, const int64_t* cursor,
                               int64_t n_rows, void* stream);
int nif_adam_units_dev(const nif_family_view* f, const nif_train_view* t, double lr,
                       double beta1, double beta2, double eps, int64_t* cursor, int64_t delta,
                       void* stream);

/* Data-parallel / deterministic form of the fused step (nif.py:682-749):
 * the same forward / loss / backward over rows idx[(cursor ? *cursor : 0) +
 * row0 + k*row_step], with the gradients routed to caller buffers:
 *   mlp_grad  (NULL: t->grad + t->off_w) receives the MLP gradients in the
 *             family layout [w | pad | b] (off_b - off_w + n_heads*b_stride
 *             floats), accumulated by fp32 atomics, or
 *   mlp_part  (non-NULL: deterministic) per-CTA partial sums, reduced in CTA
 *             order into mlp_grad after the kernel (part_floats >=
 *             nif_train_part_floats(n_rows));
 *   dx_out    (non-NULL) the fp32 input gradient of batch row g at
 *             dx_out[g*IN + k] (IN = dims[0]) instead of the grid scatter,
 *             which nif_grid_scatter_dev then applies for the whole batch.
 * A data-parallel rank writes only its own rows of dx_out: zero the buffer,
 * all-reduce [dx_out | mlp_grad] (one collective), scatter every row.     */
int nif_train_fwdbwd_ex_dev(const nif_family_view* f, const nif_train_view* t,
                            const int64_t* obj, const double* coord, const float* label,
                            const int64_t* idx, const int64_t* cursor, int64_t n_rows,
                            int64_t row0, int64_t row_step, double* sq_err, float* dx_out,
                            float* mlp_grad, float* mlp_part, int64_t part_floats, void* stream);
int64_t nif_train_part_floats(const nif_family_view* f, const nif_train_view* t, int64_t n_rows);

/* Grid-gradient scatter of a whole batch from its input gradients dx
 * [n_rows][IN] (grids.py:171-202 accumulate_grad_{2d,1d}_batch: corner
 * contribution (float)(w_fp64 * dx), added into t->grad).
 *   deterministic=0: fp32 atomics, warp-aggregated (lanes hitting one cell
 *     are summed in lane order, one atomic per group and latent);
 *   deterministic=1: contributions stably sorted by (cell, corner) in batch
 *     row order -- the reference's np.add.at order -- and summed
 *     sequentially per cell: bit-identical to the reference's scatter;
 *   deterministic=2: order-independent fixed point (int64 atomics at a
 *     per-batch power-of-two scale, one fp32 rounding per cell):
 *     bit-reproducible on every run and every data-parallel rank at the
 *     cost of the atomic scatter.
 * Modes 1 and 2 need ws_bytes >= nif_grid_scatter_ws_bytes(...,
 * deterministic) of device workspace (mode 2: zeroed once before its first
 * use; the scatter leaves it ready for the next call).                     */
size_t nif_grid_scatter_ws_bytes(const nif_family_view* f, const nif_train_view* t,
                                 int64_t n_rows, int deterministic);
int nif_grid_scatter_dev(const nif_family_view* f, const nif_train_view* t, const int64_t* obj,
                         const double* coord, const int64_t* idx, const int64_t* cursor,
                         int64_t n_rows, const float* dx, int deterministic, void* ws,
                         size_t ws_bytes, void* stream);

/* Adam (grids.py:31-45) on every touched object's grids (dense, all
 * cells) and on each touched MLP head; fp64 moments over fp32 storage,
 * numba's integer power for the bias correction; clears the gradients of
 * the stepped tensors and the batch counts.                              */
int nif_adam_dev(const nif_family_view* f, const nif_train_view* t, double lr, double beta1,
                 double beta2, double eps, void* stream);

/* ---- shadow-ray generation (renderer.py:743-805 sample_pass) ---------- */
typedef struct nif_camera {
  double pos[3];
  double fwd[3];
  double right[3];
  double up[3];
  double tan_half;
  double aspect;
  int32_t width;
  int32_t height;
} nif_camera;

typedef struct nif_lights_view {
  int32_t n_lights;        /* entries of the flux CDF                     */
  int32_t pad0;
  const uint8_t* kind;     /* [n] 0 point, 1 area (env unsupported here)  */
  const double* data;      /* [n][16] renderer.py:223-259 _pack_lights    */
  const double* cum;       /* [n] flux CDF                                */
} nif_lights_view;

typedef struct nif_pass_out {
  uint8_t* hit;       /* [n_pix] */
  double* t;          /* [n_pix] */
  int32_t* obj;       /* [n_pix] */
  double* point;      /* [n_pix][3] */
  double* normal;     /* [n_pix][3] */
  double* pdir;       /* [n_pix][3] */
  double* ldir;       /* [n_pix][3] */
  double* tmax;       /* [n_pix] */
  double* pdf;        /* [n_pix] */
  double* emit;       /* [n_pix][3] */
} nif_pass_out;

/* sampler: 0 importance (light CDF), 1 uniform sphere. pix0/n_pix select a
 * contiguous pixel range (image-tile sharding across GPUs).            */
int nif_sample_pass_dev(const nif_scene_view* scene, const nif_camera* cam,
                        const nif_lights_view* lights, int64_t seed, int64_t sample,
                        int32_t sampler, int64_t pix0, int64_t n_pix,
                        const nif_pass_out* out, void* stream);

/* Geometry-head labels (bvh.py:920-950 _k_label_geometry): per record,
 * closest hit in the record's own object; labels[m][4] = (unit normal,
 * t / diagonal) as f32, hit[m] = 1 when something was hit (keep).      */
int nif_label_geometry_dev(const nif_scene_view* s, const int32_t* rec_obj,
                           const int32_t* rec_ray, int64_t m, const double* origins,
                           const double* dirs, double diagonal, float* labels, uint8_t* hit,
                           void* stream);

/* ---- native engine: the whole pass behind one handle ------------------
 * (SURVEY.md §8b "nif_occluded"; replaces PredictorBackend.occluded,
 * renderer.py:675-683, of a NifBackend, nif.py:486-499, for FFI callers
 * with rays in host memory). The engine owns the device ray buffers
 * (`capacity` rays), the record queues (a few slots per ray, grown when a
 * chunk overflows), the gather workspace, the per_object bucketing scratch
 * and a ring of pinned host staging slots; scene / route / families are
 * views of caller-owned device memory.
 * producer_stream: the stream the caller enqueued the model's
 * nif_fast_pack_dev on (NULL = legacy stream); the engine's streams wait
 * for it before the next query, so a repack can never be read half-written.
 * After optimiser steps: repack, then nif_engine_update_model.
 * nif_engine_occluded_host: pageable host rays in, one byte per ray out
 * (1 = shadowed), synchronous. Rays stream through the pinned ring in
 * chunks (chunks = 0: 256K-ray chunks; > 0: at least that many chunks):
 * the staging memcpy of chunk k+1 (host thread pool), its upload and the
 * device pass of chunk k overlap.
 * nif_engine_info: out4 = {chunk rays, record slots per ray, staging
 * threads, overflow re-runs so far}.                                     */
typedef struct nif_engine nif_engine;
int nif_engine_create(const nif_scene_view* scene, const uint8_t* route_dev, int32_t n_net_obj,
                      const nif_family_view* outer, const nif_family_view* inner,
                      int64_t capacity, void* producer_stream, nif_engine** out_engine);
int nif_engine_update_model(nif_engine* e, const nif_family_view* outer,
                            const nif_family_view* inner, void* producer_stream);
int nif_engine_occluded_host(nif_engine* e, const double* origins, const double* dirs,
                             const double* tmaxs, int64_t n, uint8_t* occ_out, int32_t chunks);
int nif_engine_info(const nif_engine* e, int64_t* out4);
int nif_engine_destroy(nif_engine* e);

/* One progressive sample's shading (renderer.py:826-849): for the n_cast
 * shadow-cast pixels idx[k] with visibility occ[k] (1 = shadowed), adds
 * albedo[obj] / pi * emit * (vis * cos / pdf) to the fp64 HDR buffer
 * buf[n_pix][3], in the reference's evaluation order.                  */
int nif_shade_accumulate_dev(const nif_pass_out* pass, const double* albedo, const int64_t* idx,
                             const uint8_t* occ, int64_t n_cast, double* buf, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NIF_B200_H */
