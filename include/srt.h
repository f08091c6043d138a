/*
 * srt.h -- C ABI of libsrt, the sm_100a stochastic Gaussian ray tracer.
 *
 * Plain pointers and sizes only; every entry point returns an srt_status and
 * never throws.  Host-pointer entry points are synchronous and mirror the
 * reference operator boundary (/root/reference/pkg/src/splatray/kernels.py);
 * *_device entry points take device pointers plus a cudaStream_t (passed as
 * void*) and are asynchronous on that stream.
 *
 * Interface map (reference file:line -> entry point):
 *   SplatAsset.packed          assets.py:145-171   -> srt_scene_create
 *   scene_bvh / bvh.build      render.py:97-100,
 *                              bvh.py:87-193       -> srt_bvh_build (GPU LBVH)
 *   bvh= argument of render()  render.py:129,164   -> srt_bvh_upload
 *   kernels.trace_batch        kernels.py:527-540  -> srt_trace_rays
 *   kernels.render_stochastic  kernels.py:622-673  -> srt_render
 *                                                     (= srt_trace_pass_device
 *                                                      + srt_shade_pass_device
 *                                                      per pass)
 *   kernels.transmittance_batch kernels.py:544-557 -> srt_transmittance_rays
 *   kernels.exact_batch        kernels.py:584-604  -> srt_exact_rays
 *   kernels.render_exact       kernels.py:677-723  -> srt_render_exact
 *   kernels.biased_batch       kernels.py:561-580  -> srt_biased_rays
 *   cli._biased_frame          cli.py:164-203      -> srt_render_biased
 *   kernels.hash_position_batch kernels.py:119-122 -> srt_hash_positions
 *   kernels.pixel_jitter_batch kernels.py:125-135  -> srt_pixel_jitter
 *   (new) multi-GPU tile gather                    -> srt_unpack_tiles_device
 */
#ifndef SRT_H
#define SRT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t srt_status;
#define SRT_OK 0
#define SRT_ERR_INVALID_ARG 1
#define SRT_ERR_CUDA 2
#define SRT_ERR_OOM 3
#define SRT_ERR_NO_BVH 4
#define SRT_ERR_STACK_OVERFLOW 5
#define SRT_ERR_UNSUPPORTED 6

/* acceptance-draw generators (kernels.py:354 is the reference's trig hash) */
#define SRT_RNG_COUNTER 1 /* u = U24(mix(seed, ray_id, sample, prim)) */
#define SRT_RNG_TABLE 2   /* u = table[prim * table_slots + slot] (scripted tests) */
#define SRT_RNG_TRIG64 3  /* the reference's own draw: trig hash of the fp64 hit position,
                             fp64 candidate in the reference's expression order
                             (kernels.py:47-60,139-189); parity mode, one ray per thread */

typedef struct SrtScene SrtScene;

/* Inputs of SplatAsset.packed (assets.py:188-195): C-contiguous float64. */
typedef struct {
    int64_t n;               /* primitives (>= 0) */
    const double *means;     /* (n, 3) */
    const double *cov_inv6;  /* (n, 6): a00 a01 a02 a11 a12 a22 (assets.py:156-162) */
    const double *opacities; /* (n,) */
    const double *sh;        /* (n, 3, K), K = (sh_degree + 1)^2, channel major; may be NULL */
    int32_t sh_degree;       /* 0..3 */
} SrtSceneDesc;

/* The 14 camera scalars of render.py:144-150, in that order. */
typedef struct {
    double position[3];
    double right[3];
    double up[3];
    double forward[3];
    double half_w, half_h;
} SrtCamera;

typedef struct {
    int32_t width, height;
    int32_t passes;     /* ceil(spp / multisample)  (config.py:87-89) */
    int32_t nslots;     /* multisample N, 1..256    (config.py:79-80) */
    int32_t mode;       /* 0 = mean depth, 1 = center depth (render.py:153) */
    int32_t clip;       /* far-bound clipping (render() always passes 1) */
    double s2;          /* cutoff_s^2 (render.py:154) */
    uint32_t seed;      /* jitter + counter RNG seed */
    int32_t pass0;      /* global index of the first pass (sample sharding) */
    double background[3];
    int32_t shard_index; /* image-tile sharding: this rank renders 16x16 tiles */
    int32_t shard_count; /* t with t % shard_count == shard_index (1 = all)   */
    int32_t rng;         /* 0 or SRT_RNG_COUNTER (default), SRT_RNG_TRIG64 */
} SrtRenderParams;

typedef struct {
    double t_min, t_max;
    int32_t mode;
    int32_t clip;
    double s2;
    int32_t rng;             /* SRT_RNG_COUNTER, SRT_RNG_TABLE or SRT_RNG_TRIG64 */
    uint32_t seed;
    uint32_t ray_id0;        /* ray i uses ray_id = ray_id0 + i */
    uint32_t sample0;        /* slot k uses sample = sample0 + k */
    const double *table;     /* SRT_RNG_TABLE: host (n, table_slots) uniforms */
    int64_t table_slots;
} SrtTraceParams;

/* Raw splats (SplatAsset fields, assets.py:60-102) for on-device packing. */
typedef struct {
    int64_t n;
    const double *means;     /* (n, 3) */
    const double *rotations; /* (n, 4) unit quaternions (w, x, y, z) */
    const double *scales;    /* (n, 3) > 0 */
    const double *opacities; /* (n,) */
    const double *sh;        /* (n, 3, K); may be NULL */
    int32_t sh_degree;
} SrtSplatDesc;

/* ---- library ----------------------------------------------------------- */
const char *srt_last_error(void);      /* thread-local message of the last failure */
const char *srt_version(void);
const char *srt_build_id(void);        /* content hash of the sources this library was built from */
/* Measured L2 read bandwidth (GB/s, best of `reps`) of `device`: a `bytes`
 * buffer resident in L2 read with L1-bypassing 16-byte loads.  The
 * denominator of the benchmark's physical L2 fraction. */
srt_status srt_probe_l2_bandwidth(int32_t device, int64_t bytes, int32_t reps, double *gbs);
int32_t srt_device_count(void);

/* Page-locked host memory (cudaHostAlloc) for host outputs: device->host
 * copies into it run at full link speed.  srt_host_free releases it. */
srt_status srt_host_alloc(int64_t bytes, void **out);
srt_status srt_host_free(void *ptr);
/* Page-lock and map existing host memory (e.g. a shared-memory frame every
 * rank of a multi-GPU render writes its tiles into); undo with unregister. */
srt_status srt_host_register(void *ptr, int64_t bytes);
srt_status srt_host_unregister(void *ptr);

/* ---- scene ------------------------------------------------------------- */
/* Upload a packed scene to `device` (fp32 SoA records in HBM). */
srt_status srt_scene_create(const SrtSceneDesc *desc, int32_t device, SrtScene **out);
srt_status srt_scene_destroy(SrtScene *scene);
/* Upload raw splats and pack them on the device: A = R diag(1/s^2) R^T in
 * fp64 per primitive (replaces SplatAsset.packed, assets.py:145-171). */
srt_status srt_scene_create_from_splats(const SrtSplatDesc *desc, int32_t device, SrtScene **out);
/* Build the GPU BVH over each primitive's cutoff-ellipsoid AABB
 * (Mahalanobis radius cutoff_s), collapsed to 4-wide nodes.  Replaces
 * bvh.build (bvh.py:87-193).  srt_bvh_build uses SRT_BVH_PLOC. */
#define SRT_BVH_LBVH 0 /* Morton codes, radix sort, Karras radix tree, atomic refit */
#define SRT_BVH_PLOC 1 /* Morton order + PLOC agglomerative clustering (better trees) */
srt_status srt_bvh_build(SrtScene *scene, double cutoff_s);
srt_status srt_bvh_build_ex(SrtScene *scene, double cutoff_s, int32_t method);
/* Upload a reference-layout BVH (bvh.py:29-47): node_lo/node_hi (M,3) f64,
 * node_left/node_right/node_count (M,) i64, prim_order (n,) i64,
 * prim_lo/prim_hi (n,3) f64. */
srt_status srt_bvh_upload(SrtScene *scene, int64_t num_nodes, const double *node_lo,
                          const double *node_hi, const int64_t *node_left,
                          const int64_t *node_right, const int64_t *node_count,
                          const int64_t *prim_order, const double *prim_lo,
                          const double *prim_hi);
/* Introspection: node count, tree depth, primitive count, device bytes. */
srt_status srt_bvh_info(const SrtScene *scene, int64_t *num_nodes, int32_t *depth,
                        int64_t *num_prims, int64_t *device_bytes);
/* The packet walk's spatially split tree (PLOC builds of >= 16,384
 * primitives): leaf references (>= num_prims when built, 0 when the packet
 * walk uses the unsplit tree), its 4-wide node count and grid cells per axis. */
srt_status srt_bvh_split_info(const SrtScene *scene, int64_t *num_refs, int32_t *num_nodes4,
                              int32_t *cells);
/* Copy the built BVH back in the reference layout (for invariant tests).
 * Arrays sized by srt_bvh_info: nodes M = 2n-1 (or 0), prims n. */
srt_status srt_bvh_download(const SrtScene *scene, float *node_lo, float *node_hi,
                            int64_t *node_left, int64_t *node_right, int64_t *node_count,
                            int64_t *prim_order, float *prim_lo, float *prim_hi);

/* ---- explicit rays (kernels.trace_batch) --------------------------------- */
/* origins/dirs: host (R,3) f64.  out_t (R,nslots) f64 (+inf on miss),
 * out_id (R,nslots) i64 (-1 on miss).  Counter-RNG batches of >= 4096 rays
 * whose directions share a hemisphere (camera batches, parallel jittered
 * rays) are walked as warp packets; others per lane (sorted when large).
 * The route never changes a result; env SRT_PACKET_RAYS=0/1 pins it.
 * nslots <= 256 (walked as slot groups of <= 8). */
srt_status srt_trace_rays(const SrtScene *scene, const SrtTraceParams *params,
                          const double *origins, const double *dirs, int64_t num_rays,
                          int32_t nslots, double *out_t, int64_t *out_id);
/* Device variant: d_rays is (R, 6) f64 [ox oy oz dx dy dz]; out_t f32, out_id i32.
 * Batches of >= 4096 rays synchronise `stream` once to read a 64-ray probe
 * (the packet / sort decision); the walk itself stays asynchronous. */
srt_status srt_trace_rays_device(const SrtScene *scene, const SrtTraceParams *params,
                                 const double *d_rays, int64_t num_rays, int32_t nslots,
                                 float *d_out_t, int32_t *d_out_id, void *stream);
/* kernels.transmittance_batch: prod(1 - alpha) over every valid candidate. */
srt_status srt_transmittance_rays(const SrtScene *scene, const double *origins,
                                  const double *dirs, int64_t num_rays, double t_min,
                                  double t_max, int32_t mode, double s2, double *out);

/* ---- exact compositing (kernels.exact_batch / render_exact) -------------- */
/* Every valid candidate along the ray, sorted by (t, prim id), composited
 * front to back over `background` (kernels.py:441-475, 584-604).  out_rgb
 * (R,3) f64, out_op (R,) f64.  Any number of candidates per ray (packets keep
 * up to 1,024 per ray in a list; longer ones, and incoherent batches, peel
 * them 256 at a time).  Host arrays may be pageable (staged through the
 * scene's page-locked ring) or page-locked. */
srt_status srt_exact_rays(const SrtScene *scene, const double *origins, const double *dirs,
                          int64_t num_rays, double t_min, double t_max, int32_t mode, double s2,
                          const double *background, double *out_rgb, double *out_op);
/* render_exact (kernels.py:677-723): per-pixel mean of the exact composite over
 * params->passes jittered rays (passes pass0..pass0+passes-1).  Host outputs
 * (H,W,3) and (H,W) f64. */
srt_status srt_render_exact(const SrtScene *scene, const SrtCamera *camera,
                            const SrtRenderParams *params, double *out_rgb, double *out_op);

/* ---- biased k-nearest composite (kernels.biased_batch) ------------------- */
/* One acceptance draw per candidate (slot 0 of the ray's stream: counter key
 * (seed, ray_id0+i, sample0), table column 0, or the reference trig hash with
 * SRT_RNG_TRIG64); the kk nearest accepted candidates, sorted by (t, prim id),
 * are composited front to back with their own alphas over `background`
 * (kernels.py:479-518, 561-580).  kk >= 1; params->nslots/clip are ignored.
 * out_rgb (R,3) f64.  Any kk and any number of accepted candidates
 * (one-hemisphere batches of >= 4096 rays with counter / table draws walk as
 * packets keeping the kk nearest per ray; the rest, and rays with more than
 * 1,024 accepted, peel them 128 at a time). */
srt_status srt_biased_rays(const SrtScene *scene, const SrtTraceParams *params, const double *origins,
                           const double *dirs, int64_t num_rays, int32_t kk, const double *background,
                           double *out_rgb);
/* The cli's --compare-biased frame (cli.py:164-203): per-pixel mean over
 * params->passes jittered camera rays of the biased composite.  Counter draw
 * of pixel (px,py), pass f: (seed, py*W+px, f); params->rng SRT_RNG_TRIG64
 * uses the reference hash.  Host output (H,W,3) f64. */
srt_status srt_render_biased(const SrtScene *scene, const SrtCamera *camera, const SrtRenderParams *params,
                             int32_t kk, double *out_rgb);

/* ---- sampling utilities (the rest of kernels.py's public surface) -------- */
/* kernels.hash_position_batch (kernels.py:119-122): out[i] = the trig hash of
 * points[i] (host (n,3) f64) for `slot`, in fp64 on `device` (device sin: equal
 * to the CPU value up to ~1e-5 after the hash's scaling). */
srt_status srt_hash_positions(const double *points, int64_t n, int64_t slot, double *out, int32_t device);
/* kernels.pixel_jitter_batch (kernels.py:125-135): out (n,2) f64 = the scrambled
 * Sobol jitter of pixel (px, py) for frames[i] (host (n,) i64), integer exact. */
srt_status srt_pixel_jitter(int64_t px, int64_t py, const int64_t *frames, int64_t n, uint32_t seed, double *out,
                            int32_t device);

/* ---- full frames (kernels.render_stochastic) ----------------------------- */
/* Host outputs out_rgb (H,W,3) f64 and out_op (H,W) f64 = per-pixel means.
 * out_ids (optional, may be NULL): (H,W,nslots) i64 slot ids of pass pass0.
 * With shard_count > 1 only the shard's 16x16 tiles are rendered and written,
 * which needs mapped host outputs (srt_host_alloc / srt_host_register). */
srt_status srt_render(const SrtScene *scene, const SrtCamera *camera,
                      const SrtRenderParams *params, double *out_rgb, double *out_op,
                      int64_t *out_ids);
/* One pass, device buffers.  d_hits: (H*W*nslots) i32 scratch written by the
 * trace stage and read by the shade stage.  d_accum: (H*W) float4 running
 * sums (rgb, hits); pass `pass` (absolute) is traced, and the shade stage
 * adds it, zeroing the accumulator first when `first` is set.  When `last`
 * is set the shade stage also resolves accum / (passes * nslots) into d_out
 * ((H*W) float4 rgba, rgba = (r, g, b, opacity)).  With shard_count > 1 the
 * buffers are tile-compact: local tile j occupies pixels [256 j, 256 j + 256). */
srt_status srt_trace_pass_device(const SrtScene *scene, const SrtCamera *camera,
                                 const SrtRenderParams *params, int32_t pass, int32_t *d_hits,
                                 void *stream);
srt_status srt_shade_pass_device(const SrtScene *scene, const SrtCamera *camera,
                                 const SrtRenderParams *params, int32_t pass,
                                 const int32_t *d_hits, float *d_accum, int32_t first,
                                 int32_t last, float *d_out, void *stream);
/* One pass traced AND shaded by a single kernel (the walk's hits are
 * SH-shaded and accumulated in place; no hit buffer).  Same d_accum/first/
 * last/d_out contract as srt_shade_pass_device. */
srt_status srt_render_pass_device(const SrtScene *scene, const SrtCamera *camera,
                                  const SrtRenderParams *params, int32_t pass, float *d_accum,
                                  int32_t first, int32_t last, float *d_out, void *stream);
/* srt_render_pass_device writing the ROW-MAJOR full (H*W) float4 frame even
 * for a shard: each shard stores only its own pixels, so several GPUs can
 * assemble one frame in place.  d_frame may be a peer GPU's buffer (CUDA IPC,
 * srt_ipc_open): with peer != 0 the kernel ends with a system-scope fence, so
 * its stores are visible to the peer before any later signal from this GPU
 * (e.g. a collective on the same stream). */
srt_status srt_render_pass_frame_device(const SrtScene *scene, const SrtCamera *camera,
                                        const SrtRenderParams *params, int32_t pass, float *d_accum,
                                        int32_t first, int32_t last, float *d_frame, int32_t peer,
                                        void *stream);
/* Device buffers shared between processes (one rank per GPU): srt_ipc_alloc
 * allocates on `device` and returns a 64-byte handle, srt_ipc_open maps a
 * handle from another process on `device` (peer access over NVLink). */
srt_status srt_ipc_alloc(int32_t device, int64_t bytes, void **d_ptr, uint8_t *handle);
srt_status srt_ipc_open(int32_t device, const uint8_t *handle, void **d_ptr);
srt_status srt_ipc_close(int32_t device, void *d_ptr);
srt_status srt_ipc_free(int32_t device, void *d_ptr);
/* Whole frame on device: all passes, d_out (H*W) float4 rgba means. */
/* All params->passes passes of a frame in ONE launch over every (packet,
 * pass): samples are summed in 2^-32 fixed point with integer atomics (order
 * independent, bitwise deterministic) into d_acc ((local tiles*256) * 4
 * uint64, zeroed by the call), then resolved to float4 means in d_out
 * (row-major H*W, or tile-compact when sharded).  Counter stream only.
 * Balances small frames and many-pass convergence runs far better than one
 * launch per pass.  d_out may be NULL: only the sums are produced (see
 * srt_resolve_frame_device). */
srt_status srt_render_frame_device(const SrtScene *scene, const SrtCamera *camera,
                                   const SrtRenderParams *params, uint64_t *d_acc, float *d_out,
                                   void *stream);
/* Fixed-point sums of the shard params->shard_index / shard_count (as left by
 * srt_render_frame_device) -> f64 means written row-major into the full-frame
 * device (or mapped host) buffers d_rgb (H,W,3) and d_op (H,W); each shard
 * writes only its own pixels.  Runs on the current device. */
srt_status srt_resolve_frame_device(const SrtRenderParams *params, const uint64_t *d_acc, double *d_rgb,
                                    double *d_op, void *stream);
srt_status srt_render_device(const SrtScene *scene, const SrtCamera *camera,
                             const SrtRenderParams *params, int32_t *d_hits, float *d_accum,
                             float *d_out, void *stream);
/* Device error flag of the scene (traversal stack overflow), raised by any
 * launch since the last reset.  Host-pointer entry points clear it when they
 * start and report it when they finish; the *_device entry points never read
 * it, so asynchronous callers check here after synchronising.  Synchronises
 * the scene's device; returns SRT_ERR_STACK_OVERFLOW when set (clearing it if
 * reset != 0), else SRT_OK. */
srt_status srt_scene_check(const SrtScene *scene, int32_t reset);
/* Traversal work counters accumulated while the environment variable
 * SRT_TRACE_STATS=1 is set: out[8] = node visits, leaf visits, screen
 * passes, exact evaluations, accepted slot updates, stack pops, culled
 * pops, walks.  reset != 0 zeroes them. */
srt_status srt_trace_stats(const SrtScene *scene, uint64_t *out, int32_t reset);
/* The first n (<= 16) counters; 8.. are packet-walk diagnostics: visits with a
 * leaf child hit, leaf / inner children hit by any lane, lanes with a hit per
 * visit, lanes without an accepted hit per visit, job rounds, empty visits. */
srt_status srt_trace_counters(const SrtScene *scene, uint64_t *out, int32_t n, int32_t reset);
/* Number of 16x16 tiles a shard owns (buffer sizing for tile-compact layout). */
int64_t srt_shard_tiles(int32_t width, int32_t height, int32_t shard_index,
                        int32_t shard_count);
/* Scatter gathered tile-compact shards [shard_count][max_tiles*256] float4
 * into a full (H*W) float4 frame. */
srt_status srt_unpack_tiles_device(const float *d_gathered, int32_t width, int32_t height,
                                   int32_t shard_count, int64_t max_tiles, float *d_frame,
                                   void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SRT_H */
