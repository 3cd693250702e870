/*
 * rfb.h -- C ABI of the B200 Radiant Foam hot path (librfb.so, sm_100a).
 *
 * Plain pointers and sizes only.  Every pointer is a DEVICE pointer unless
 * marked (host); `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Calls enqueue work on `stream` and return without
 * synchronising.  Return value: 0 (RFB_OK) on success, RFB_EINVAL (-1) for an
 * argument error, or a positive cudaError_t from the launch.
 *
 * Each entry point replaces one reference operator (paths are relative to
 * the reference tree pkg/src/rfoam/):
 *
 *   rfb_pack_scene      diffrender/render.py:49-54  scene_arrays()  (+ the
 *                        int64 -> int32 CSR narrowing and the per-site
 *                        {x,y,z,sigma} record the kernels gather)
 *   rfb_softplus        foam.py:22-25               softplus()  (device-side
 *                        activation for device-resident training; the parity
 *                        shim uploads the host numpy value instead)
 *   rfb_camera_rays     tracer/camera.py:66-92      CameraModel.ray_directions()
 *                        (pinhole and fisheye)
 *   rfb_effect_rays     tracer/rays.py:123-176      EffectPlane/reflect/refract/
 *                        apply_effect, batched
 *   rfb_build_adjacency geometry/delaunay.py:445-520 build() +
 *                        adjacency.py:46-64 from_triangulation() (Voronoi
 *                        cell clipping on the GPU; rfb_adjacency.cu)
 *   rfb_sh_basis, rfb_cell_colors, rfb_composite_segments,
 *   rfb_backward_segments, rfb_quantile_segments
 *                        tracer/kernels.py:38-73, 165-196, 250-369, 456-567
 *                        over given segments (rfb_segments.cu)
 *   rfb_locate, rfb_locate_seeded, rfb_build_locate_grid
 *                       geometry/adjacency.py:85-100 nearest_site()
 *                        (greedy walk on the CSR; same distance expression
 *                        and lowest-id tie rule as _grid_nearest 140-203)
 *   rfb_render_rays     tracer/kernels.py:199-247   render_rays()
 *                        (walk_ray 76-162 + sh_basis_into 38-58 +
 *                        cell_color 61-73 + composite_segments 165-196)
 *   rfb_render_image    diffrender/render.py:128-149 render_image() (fused
 *                        ray generation + shared-origin start cell + render,
 *                        over a list of image tiles for multi-GPU sharding)
 *   rfb_cull_scene, rfb_cull_view  (no reference counterpart: an exact pre-pass for
 *                        render_image() / a view's train_batch) drops from a
 *                        copy of the packed rows every neighbour that
 *                        kernels.py:118-119 skips as back-facing for EVERY ray
 *                        of a frame (pinhole: the 4 corner-pixel directions
 *                        generate the frame's direction cone)
 *   rfb_host_device_pointer  render_image() returns a host image: the mapped
 *                        address of a pinned host frame, so rfb_render_image
 *                        stores the image to host memory during the walk
 *   rfb_backward_rays   diffrender/render.py:152-221 render_rays_with_gradients()
 *                        (backward_ray 250-337 + face_t_gradient 340-369)
 *   rfb_train_batch     tracer/kernels.py:372-453   train_batch()
 *                        (+ quantile_backward_ray 456-567)
 *   rfb_post_grad_adam  optim/train.py:195-209 + optim/adam.py:15-31
 *   rfb_refresh_scene   diffrender/render.py:49-54 after a device-side update
 *                        (moved sites: re-derives the packed copies and bounds)
 *
 * Per-ray status semantics are the reference's (tracer/kernels.py:11-21):
 * 0 ok, 2 step limit, 3 cycle; failed rays render the background with
 * residual 1, wsum 0 and contribute no gradient.
 */
#ifndef RFB_H
#define RFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RFB_OK 0
#define RFB_EINVAL (-1)
#define RFB_ECAPACITY (-2)   /* a caller-sized buffer / row capacity is too small */
#define RFB_EDEGENERATE (-3) /* non-finite, duplicate or degenerate input points */

#define RFB_STATUS_OK 0
#define RFB_STATUS_STEP_LIMIT 2
#define RFB_STATUS_CYCLE 3

#define RFB_ABI_VERSION 15

/* Capacity (records) of the packed edge arrays rfb_pack_scene fills: rows are
 * padded to an even length, so E + n_sites slots suffice (+2 spare). */
#define RFB_PACKED_EDGE_SLOTS(n_sites, n_edges) ((n_edges) + (n_sites) + 2)

/* Device-resident scene, produced by rfb_pack_scene.  Two layouts:
 *  generic: site4 + offsets + neighbors (+ sh), any fp64 positions;
 *  packed (packed != 0): per-site 32-byte cell headers {float x,y,z; int k0;
 *   double sigma; int k1; float n1max} and per-edge 16-byte records
 *   {float xj,yj,zj; int j} (the neighbour's fp32 site copy and id) in CSR
 *   order, each row starting at an even slot k0 and padded to an even length
 *   with an all-NaN record (k1 = k0 + degree), so rows are read as whole
 *   32-byte pairs; edge_nbr holds every slot's neighbour id (-1 for a pad);
 *   plus fp32 SH (sh32) with the fp64 table kept for the exact clamp
 *   fallback.  With positions_f64 == 0 the fp32 coordinates are the sites
 *   themselves; with positions_f64 != 0 they are rounded copies, n1max
 *   carries the widened pre-filter bound and the exact phase reads site4
 *   (rfb_pack_scene and rfb_refresh_scene derive both).  The generic arrays
 *   are always present (backward, locate). */
typedef struct rfb_scene {
    int64_t n_sites;
    int64_t n_edges;
    const double *site4;      /* [n_sites][4]: x, y, z, sigma (activated density) */
    const int32_t *offsets;   /* [n_sites + 1] CSR row starts */
    const int32_t *neighbors; /* [n_edges] ascending per site */
    const double *sh;         /* [n_sites][48], index k*3 + ch (render.py:53) */
    const void *cells;        /* packed: [n_sites] 32-byte headers (nullable) */
    const void *edges;        /* packed: [RFB_PACKED_EDGE_SLOTS] 16-byte records (nullable) */
    const int32_t *edge_nbr;  /* packed: [RFB_PACKED_EDGE_SLOTS] neighbour id per slot */
    const float *sh32;        /* packed: [n_sites][3][16] fp32 channel-major copy of sh (nullable)
                                 cells, edges and sh32 must be 32-byte aligned (EINVAL) */
    int32_t packed;           /* 1: use cells/edges/edge_nbr/sh32 for the walk */
    float sh_absmax;          /* packed: >= max |sh| over the scene (fp32 colour bound) */
    int32_t sh_degree;        /* 0: read the DC band only (exact when bands 1..15 are
                                 all zero), 3: all 16 bands */
    int32_t positions_f64;    /* packed: 0 = every coordinate is fp32-exact; 1 = not: the
                                 fp32 copies are rounded, the pre-filter bound is widened
                                 (n1max) and the exact phase reads site4 */
    double background[3];     /* (host value) */
    const float *sh_absmax_dev; /* nullable device scalar; when set the kernels read the colour
                                 bound from it instead of sh_absmax (rfb_post_grad_adam raises it
                                 after every update, so a training scene needs no host refresh) */
    const int32_t *pk_of;     /* packed, nullable: [n_sites] packed index of each site (the
                                 packed arrays cells/edges/edge_nbr/sh32 are in the internal
                                 Morton order rfb_pack_scene chose; NULL = site order) */
    const int32_t *pk_id;     /* packed, nullable: [n_sites] site id of each packed index */
    int32_t view_rx, view_ry; /* view-culled scenes (rfb_cull_view): cells / edges hold
                                 view_rx * view_ry region copies -- region r's headers at
                                 cells[r * n_sites ...], its rows at edge slot
                                 r * RFB_VIEW_STRIDE(n_sites, n_edges) + k (the headers' k0/k1
                                 are absolute).  A camera pixel (px, py) walks region
                                 (py * view_ry / height) * view_rx + px * view_rx / width;
                                 ray batches take rfb_rays.region.  0, 0: one region */
} rfb_scene;

/* Edge-slot stride between the region copies of a view-culled scene (even, so
 * every row stays 32-byte aligned). */
#define RFB_VIEW_STRIDE(n_sites, n_edges) (((n_edges) + (n_sites) + 3) & ~(int64_t)1)

/* Walk parameters (tracer/rays.py:12-14). */
typedef struct rfb_params {
    double epsilon;       /* early-termination transmittance, 0 disables */
    double width_floor;   /* WIDTH_FLOOR_SCALE * diagonal */
    int32_t step_limit;   /* hard per-ray cell cap */
    int32_t lanes_per_ray;/* forward: 1, 2, 4, 8, 16 or 32 lanes cooperate on one ray;
                             0 = auto: the largest power of two <= 8 whose lanes x rays fit
                             the resident threads (small batches use more lanes).
                             backward / training: 1 or 2; 0 = auto (2 when the batch fills
                             at most half the resident threads) */
} rfb_params;

/* A batch of rays (render.py:57-125 arguments). */
typedef struct rfb_rays {
    int64_t m;
    const double *origins;     /* [m][3] */
    const double *directions;  /* [m][3], unit length */
    const double *t_min;       /* [m] */
    const double *t_max;       /* [m] */
    const int32_t *start_sites;/* [m] */
    const int32_t *order;      /* [m] nullable: processing order, a permutation of 0..m-1
                                  (coherence only; outputs stay indexed by ray id) */
    const uint8_t *region;     /* [m] nullable: region of a view-culled scene each ray walks
                                  (its direction must lie in that region's cone); NULL = 0 */
} rfb_rays;

/* Forward outputs.  rgb/residual/wsum are float32 unless f64_outputs != 0,
 * in which case they are float64.  Nullable fields are skipped. */
typedef struct rfb_fwd_out {
    void *rgb;                 /* [m][3] (required) */
    void *residual;            /* [m] nullable */
    void *wsum;                /* [m] nullable */
    int8_t *status;            /* [m] nullable */
    int32_t *nseg;             /* [m] nullable: recorded segments per ray */
    int32_t *ray_counters;     /* [m][2] nullable: cells stepped, neighbour visits */
    unsigned long long *counters; /* [2] nullable: totals, ACCUMULATED (kernels.py:8-9) */
    int32_t f64_outputs;
    int32_t seg_capacity;      /* > 0 enables the segment dump below */
    int32_t *seg_cells;        /* [seg rows][seg_capacity] */
    double *seg_t0;            /* [seg rows][seg_capacity] */
    double *seg_t1;            /* [seg rows][seg_capacity] */
    int64_t seg_first;         /* the dump holds rays seg_first .. seg_first + seg_count - 1 */
    int64_t seg_count;         /* (row r of the dump = ray seg_first + r); 0 = every ray */
} rfb_fwd_out;

/* Gradient accumulators (ACCUMULATED, like the reference's += buffers).
 * One flat float32 allocation of n_sites * 52 floats is the intended layout:
 * site4g = [n][4] (dpos x, y, z, dsigma) followed by sh = [n][48]. */
typedef struct rfb_grads {
    float *site4g;  /* [n][4]: dL/dposition (3) and dL/dsigma (activated) */
    float *sh;      /* [n][48] */
} rfb_grads;

/* Camera (camera.py:20-92). pose is row-major world-from-camera. */
typedef struct rfb_camera {
    double pose[16]; /* (host value) */
    int32_t width;
    int32_t height;
    double focal;
    double cx;
    double cy;
    int32_t kind;    /* 0 pinhole, 1 fisheye (equidistant, theta = r) */
    int32_t pad_;
} rfb_camera;

int rfb_abi_version(void);
const char *rfb_error_string(int code); /* (host) static string */
int rfb_device_ok(void);                /* 1 when an sm_100 device is current */

/* Device address of page-locked host memory (cudaHostGetDevicePointer), so a
 * kernel can store its per-ray outputs straight into the caller's host frame
 * (the D2H then overlaps the walk; render.py:128-149 returns a host image).
 * Returns 0, RFB_EINVAL, or the cudaError_t when the memory is not mapped. */
int rfb_host_device_pointer(void *host, void **device_ptr);

/* Build the device layout from fp64/int64 device arrays:
 * positions [n][3], sigma [n], sh [n][48], offsets [n+1], neighbors [E]
 * -> site4 [n][4] f64, offsets32 [n+1], neighbors32 [E] and, when
 * cells/edges/edge_nbr/sh32 are non-NULL, the packed layout (edges and
 * edge_nbr hold RFB_PACKED_EDGE_SLOTS(n, E) slots).  positions_f64 must be
 * nonzero unless every coordinate is exactly representable in fp32 (and
 * stays so: set it for scenes whose sites will move); the same value goes
 * into rfb_scene.positions_f64.  pk_of / pk_id (nullable, both or neither,
 * [n] each): when given, the packed arrays are laid out in a Morton order of
 * the sites (cells a ray visits in turn sit near each other) and the two
 * permutations are written there; every row keeps its site's CSR order, and
 * all inputs and outputs of the other calls stay in site ids.  Uses
 * stream-ordered scratch (cudaMallocAsync): not a hot-path call. */
int rfb_pack_scene(const double *positions, const double *sigma, const double *sh,
                   const int64_t *offsets, const int64_t *neighbors, int64_t n_sites,
                   int64_t n_edges, double *site4, int32_t *offsets32, int32_t *neighbors32,
                   void *cells, void *edges, int32_t *edge_nbr, float *sh32, int32_t *pk_of,
                   int32_t *pk_id, int32_t positions_f64, void *stream);

/* sigma = softplus_10(raw) for device-resident training, written to out
 * (nullable), site4[:,3] (nullable) and the packed headers (nullable; rows
 * permuted by pk_of when given). */
int rfb_softplus(const double *raw, int64_t n, double *out, double *site4, void *cells,
                 const int32_t *pk_of, void *stream);

/* Fused gradient post-processing + Adam after the gradient all-reduce
 * (optim/train.py:195-209 + optim/adam.py:15-31).  grads_flat is the [n*52]
 * fp32 buffer of rfb_grads; positions [n][3], raw_density [n], sh [n][48] are
 * the fp64 parameters updated in place; adam_state holds m_pos, v_pos (3n
 * each), m_raw, v_raw (n each), m_sh, v_sh (48n each).  hyper (host) is
 * 3 x {lr, beta1, beta2, eps, 1-beta1^step, 1-beta2^step} for positions,
 * densities and SH.  sh_warmup zeroes the SH bands 1..15 gradient;
 * update_positions = 0 skips positions (lr_pos == 0 tail).  sh32 (nullable):
 * the packed scene's fp32 channel-major SH copy (rfb_scene.sh32), rewritten
 * from the updated coefficients in the same pass.  sh_absmax_dev (nullable):
 * the scene's device colour bound (rfb_scene.sh_absmax_dev), raised to at
 * least max |sh| of the updated coefficients (a running maximum: never
 * lowered, so it stays an upper bound of every coefficient).  pk_of: the
 * scene's packed order (rfb_scene.pk_of) for the sh32 rows, nullable. */
int rfb_post_grad_adam(int64_t n_sites, const float *grads_flat, double *positions,
                       double *raw_density, double *sh, double *adam_state, double clip,
                       int32_t sh_warmup, int32_t update_positions, const double *hyper,
                       float *sh32, float *sh_absmax_dev, const int32_t *pk_of, void *stream);

/* After a parameter update: site4 = {positions, softplus(raw)}, packed
 * headers' sigma and, when refresh_sh32 is nonzero, the fp32 SH copy are
 * refreshed from scene->sh (pass 0 when rfb_post_grad_adam already wrote
 * scene->sh32).  A packed scene with positions_f64 != 0 also gets its fp32
 * copies, face records and widened bounds re-derived from the moved sites;
 * one with positions_f64 == 0 cannot take moved sites (re-pack it). */
int rfb_refresh_scene(const rfb_scene *scene, const double *positions, const double *raw_density,
                      int32_t refresh_sh32, void *stream);

/* dirs [pix_count][3] f64 for row-major pixels pix_begin .. pix_begin+count-1. */
int rfb_camera_rays(const rfb_camera *camera, int64_t pix_begin, int64_t pix_count,
                    double *dirs, void *stream);

/* Effect rays (tracer/rays.py:123-176 EffectPlane / reflect / refract /
 * apply_effect): ray q continues from origins[q] + t_at[q] * directions[q]
 * with the mirrored (kind RFB_EFFECT_MIRROR) or refracted (RFB_EFFECT_REFRACT,
 * relative index eta, total internal reflection -> mirror, back side -> flipped
 * normal and 1/eta) unit direction.  normal (host, 3 doubles) need not be
 * unit length.  New rays start at t_min = 0 with the old t_max. */
#define RFB_EFFECT_MIRROR 0
#define RFB_EFFECT_REFRACT 1
int rfb_effect_rays(const double *origins, const double *directions, const double *t_at,
                    int64_t m, const double *normal, int32_t kind, double eta,
                    double *out_origins, double *out_directions, void *stream);

/* Delaunay adjacency on the device (geometry/delaunay.py:445-520 build +
 * geometry/adjacency.py:46-64 from_triangulation): per-site Voronoi cell
 * clipping, one warp per site.  positions [n][3] f64 (device).  Writes
 * offsets [n+1] (int64, device) and, when neighbors is non-NULL and
 * neighbor_capacity >= the edge count, the ascending symmetric neighbour
 * lists (int64) and hull flags (uint8, nullable).  stats (host, 8 int64):
 * [0] directed edge count E, [1] reverse edges added by the symmetrisation,
 * [2] sites that needed the ring scan, [3] max cell vertices, [4] max
 * planes.  With neighbors == NULL the call is a size query: allocate E and
 * finish with rfb_adjacency_emit on the same workspace.  max_degree <= 128
 * is the per-site row capacity (RFB_ECAPACITY beyond).  Synchronises the
 * stream.  RFB_EDEGENERATE: non-finite input or two sites within
 * 1e-7 x the bounding-box diagonal (delaunay.py:436-467). */
size_t rfb_adjacency_workspace_bytes(int64_t n_sites, int32_t max_degree);
int rfb_build_adjacency(const double *positions, int64_t n_sites, int32_t max_degree,
                        int64_t *offsets, int64_t *neighbors, int64_t neighbor_capacity,
                        uint8_t *hull, int64_t *stats, void *workspace, size_t workspace_bytes,
                        void *stream);
int rfb_adjacency_emit(int64_t n_sites, int32_t max_degree, const int64_t *offsets,
                       int64_t *neighbors, uint8_t *hull, const void *workspace,
                       size_t workspace_bytes, void *stream);

/* The reference's per-ray building blocks over caller-held segment lists
 * (rfb_segments.cu; the hot path fuses them into rfb_render_rays, rfb_render_image
 * and rfb_train_batch).
 * Segments are CSR per ray: ray r owns seg_offsets[r] .. seg_offsets[r+1]-1
 * (int64 offsets, int32 cells, f64 t0/t1).  All device pointers, fp64, the
 * reference's operation order; background is host (3 doubles); gradient
 * outputs accumulate (fp64 atomics).  Workspace: rfb_segments_workspace_bytes
 * (rays, total segments). */
int rfb_sh_basis(const double *dirs, int64_t m, double *out /* [m][16] */, void *stream);
int rfb_cell_colors(const double *sh, const int32_t *cells, const double *basis, int64_t m,
                    double *out /* [m][3] */, int32_t *masks /* nullable */, void *stream);
int rfb_composite_segments(const double *sigma, const double *sh, const double *bases /* [m][16] */,
                           int64_t m, const int64_t *seg_offsets, const int32_t *seg_cells,
                           const double *seg_t0, const double *seg_t1, const double *background,
                           double *out_rgb, double *out_T /* nullable */,
                           double *out_wsum /* nullable */, void *stream);
/* face_t_gradient (kernels.py:340-369) for m boundaries: ij [m][2] sites
 * (i, j), ray q's origin/direction, crossing depth t[q] and dt[q]. */
int rfb_face_t_gradients(const double *positions, const int32_t *ij, const double *origins,
                         const double *directions, const double *t, const double *dt, int64_t m,
                         double *d_pos, void *stream);
size_t rfb_segments_workspace_bytes(int64_t m, int64_t n_segments);
int rfb_backward_segments(const double *positions, const double *sigma, const double *sh,
                          const double *background, const double *origins,
                          const double *directions, const double *bases /* [m][16] */,
                          const double *adjoints, int64_t m, const int64_t *seg_offsets,
                          const int32_t *seg_cells, const double *seg_t0, const double *seg_t1,
                          double *d_sigma, double *d_sh, double *d_pos, void *workspace,
                          size_t workspace_bytes, void *stream);
int rfb_quantile_segments(const double *positions, const double *sigma, const double *origins,
                          const double *directions, int64_t m, const int64_t *seg_offsets,
                          const int32_t *seg_cells, const double *seg_t0, const double *seg_t1,
                          const double *u_pairs /* [m][P][2] */, int32_t n_pairs,
                          double weight_floor, double scale, double *d_sigma, double *d_pos,
                          double *loss_out /* [m], nullable */, void *workspace,
                          size_t workspace_bytes, void *stream);

/* Seed grid for point location (the reference's bucket grid role,
 * adjacency.py:140-203): hint [dims] int32 device array, cell size `cell`,
 * origin lo.  rfb_build_locate_grid fills every cell with the largest site id
 * inside it (-1 if empty); rfb_locate_seeded starts each query's greedy walk
 * from the nearest non-empty cell within two rings (else seed_site).  The walk
 * is exact from any seed; the grid only shortens it. */
typedef struct rfb_locate_grid {
    double lo[3];
    double cell;
    int32_t dims[3];
    int32_t pad_;
    int32_t *hint;
} rfb_locate_grid;
int rfb_build_locate_grid(const rfb_scene *scene, rfb_locate_grid *grid, void *stream);
int rfb_locate_seeded(const rfb_scene *scene, const double *queries, int64_t m,
                    const rfb_locate_grid *grid, int32_t seed_site, int32_t *out, void *stream);

/* out[q] = nearest site to queries[q] (greedy CSR walk from seed_site). */
int rfb_locate(const rfb_scene *scene, const double *queries, int64_t m, int32_t seed_site,
               int32_t *out, void *stream);

int rfb_render_rays(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                    const rfb_fwd_out *out, void *workspace, size_t workspace_bytes, void *stream);

/* Renders the listed tile_w x tile_h pixel tiles (multiples of 32) (tile id = ty * tiles_x + tx,
 * tiles_x = ceil(W / tile_w)) of the frame; outputs are full-frame [H*W]
 * arrays indexed by pixel (row-major), untouched outside the listed tiles.
 * start_site < 0: locate the camera position's nearest site on device from
 * seed site 0.  t_max <= 0: render.py:72-76 fallback computed by the caller. */
int rfb_render_image(const rfb_scene *scene, const rfb_camera *camera, const rfb_params *params,
                     double t_min, double t_max, int32_t start_site, const int32_t *tile_ids,
                     int64_t n_tiles, int32_t tile_w, int32_t tile_h, const rfb_fwd_out *out,
                     void *workspace, size_t workspace_bytes, void *stream);

/* Workspace bytes needed by the calls above for m rays (kind: 0 forward,
 * 1 backward/train with any loss, 2 backward / train without the quantile
 * term).  Forward calls accept >= 256 bytes; from 256 + 8 (SMs + 1) on they
 * keep one work queue per SM (an SM's warps walk neighbouring pixel patches
 * together and share the cells' data in L1; same results).  Backward / train:
 * a 4 KB header of work counters, then the segment records of the resident
 * rays. */
size_t rfb_workspace_bytes(int64_t m, int32_t step_limit, int32_t kind);

/* Forward + reverse pass for arbitrary colour adjoints [m][3] f64.  out.rgb
 * receives the forward colour; gradients accumulate into grads. */
/* View culling: `dirs` (host, [n_dirs][3], 1 <= n_dirs <= 8) generate a cone
 * (positive combinations) that must contain the direction of every ray the
 * culled scene will walk -- for a pinhole camera the directions of its four
 * corner pixels.  Writes a copy of the packed rows into cells_out
 * ([n_sites] 32-byte headers) and edges_out ([RFB_PACKED_EDGE_SLOTS] 16-byte
 * records), both 32-byte aligned, leaving out every neighbour whose face is
 * back-facing (d . n < -1e-9 |n|_1) for every direction of the cone, and fills
 * *view_out (host) with the scene using them.  The walk over the view is
 * bit-identical to the walk over the full rows for every ray in the cone
 * (the dropped faces fail `denom <= 0` there), counters included.  Packed
 * scenes only; any later rfb_refresh_scene / re-pack invalidates the view. */
int rfb_cull_scene(const rfb_scene *scene, const double *dirs, int32_t n_dirs, void *cells_out,
                   void *edges_out, rfb_scene *view_out, void *stream);

/* The same per region of a pinhole camera's image: an rx x ry grid of pixel
 * rectangles (pixel (px, py) belongs to region (py * ry / height) * rx +
 * px * rx / width, integer division), each culled against the cone of its own
 * four corner pixels into its own copy: cells_out [rx*ry][n_sites] headers,
 * edges_out [rx*ry][RFB_VIEW_STRIDE] records (32-byte aligned).  Smaller
 * cones drop more faces (1080p, 0.9 rad: 25% of the neighbour records for the
 * whole frame, ~44% per region of a 4 x 4 grid).  rfb_render_image on the view
 * picks each pixel's region itself; ray batches pass rfb_rays.region.
 * rx * ry <= 32, width >= rx, height >= ry, pinhole only. */
int rfb_cull_view(const rfb_scene *scene, const rfb_camera *camera, int32_t rx, int32_t ry,
                  void *cells_out, void *edges_out, rfb_scene *view_out, void *stream);

int rfb_backward_rays(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                      const double *adjoints, const rfb_fwd_out *out, const rfb_grads *grads,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Fused training pass: L2 adjoint 2*rgb_scale*(rgb - target) plus, when
 * quantile_scale > 0, n_pairs Monte-Carlo quantile pairs per ray
 * (u_pairs [m][n_pairs][2] f64).  loss [2] f64 ACCUMULATES (sum sq err,
 * sum quantile terms) like loss_w in kernels.py:433,445. */
int rfb_train_batch(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                    const double *targets, double rgb_scale, double quantile_scale,
                    const double *u_pairs, int32_t n_pairs, double weight_floor,
                    const rfb_fwd_out *out, const rfb_grads *grads, double *loss,
                    void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RFB_H */
