// srt_internal.h -- host-side scene object and helpers shared by the .cu files.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/srt.h"
#include "srt_device.cuh"

struct SrtScene {
    int device = 0;
    int64_t n = 0;
    int32_t sh_deg = 0;
    int32_t sh_k = 1;
    // device records
    double *d_means = nullptr;  // (n,3) f64 (LBVH box computation)
    double *d_cov6 = nullptr;   // (n,6) f64
    double *d_opac = nullptr;   // (n,)  f64
    float *d_sh = nullptr;      // (n,3,K) f32, original order
    srt::Geom *d_geom = nullptr;   // (n,) slot order (valid once a BVH exists)
    srt::Node2 *d_nodes = nullptr; // (num_nodes,) binary tree (build / upload output)
    int32_t num_nodes = 0;
    srt::Node4 *d_nodes4 = nullptr; // (num_nodes4,) 4-wide tree traced by the kernels
    srt::Node4 *d_nodes8 = nullptr; // (8, num_nodes4) the same tree per direction octant (packet kernel)
    int32_t num_nodes4 = 0;
    // Spatially split copy of the tree for the closest-hit walks (split.cu):
    // leaf references to primitives clipped at the planes of a uniform cell
    // grid, so the top of the tree has no overlap.  Only the 4-wide tree, its
    // octant copies and the reference-ordered records are kept.  Null: the
    // walks use the tree above (small scenes, uploaded reference BVHs).
    srt::Geom *d_geom_split = nullptr;    // (n_refs,) reference (slot) order
    srt::Node4 *d_nodes4_split = nullptr; // (num_nodes4_split,)
    srt::Node4 *d_nodes8_split = nullptr; // (8, num_nodes4_split)
    int32_t num_nodes4_split = 0;
    int64_t n_refs = 0;
    int32_t split_cells = 0;  // cells per axis of the split grid (0: no split tree)
    unsigned long long *d_stats = nullptr;  // traversal counters (srt_trace_stats)
    int32_t depth = 0;
    bool has_bvh = false;
    int32_t *h_flag = nullptr;  // error flag (stack overflow) in mapped page-locked host memory
    int32_t *d_flag = nullptr;  // its device alias
    // work counter pair (work, done) of launches on the scene's own stream:
    // stream-ordered, reset by the last block of each launch (release_counter)
    uint32_t *d_counter = nullptr;
    // cached scratch for the host-pointer entry points
    void *d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // page-locked staging ring for pageable caller arrays (hostcopy.cu)
    void *h_stage[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    cudaStream_t stream = nullptr;
    // Host entry points that use the scene's stream and scratch serialise on
    // `mu` (calls on one handle serialise).  Every persistent
    // launch takes its own work counter from stream-ordered scratch
    // (LaunchCounter), so launches on concurrent caller streams never share one.
    mutable std::mutex mu;
    srt::SceneView view() const {
        srt::SceneView v;
        v.means64 = d_means;
        v.cov64 = d_cov6;
        v.opac64 = d_opac;
        v.nodes = d_nodes;
        v.nodes4 = d_nodes4;
        v.nodes8 = d_nodes8;
        v.num_nodes4 = num_nodes4;
        v.geom = d_geom;
        v.sh = d_sh;
        v.num_nodes = num_nodes;
        v.root = 0;
        v.sh_k = sh_k;
        v.sh_deg = sh_deg;
        v.n = n;
        return v;
    }
    // The view the closest-hit walks (k_trace_packet, k_trace, k_trace_coop,
    // the trig64 bridge walks)
    // traverse: the split tree when one exists.  Leaf codes index
    // d_geom_split; duplicate references of a primitive give the same (t, id)
    // key and draw, so the order-free closest-accepted slots are unchanged
    // (split.cu).  Compositing walks keep view().
    srt::SceneView walk_view() const {
        srt::SceneView v = view();
        if (d_nodes8_split) {
            v.nodes = nullptr;
            v.nodes4 = d_nodes4_split;
            v.nodes8 = d_nodes8_split;
            v.num_nodes4 = num_nodes4_split;
            v.geom = d_geom_split;
            v.n = n_refs;
        }
        return v;
    }
};

namespace srt {

void set_error(const std::string &msg);
srt_status cuda_status(cudaError_t e, const char *what);

// RAII device guard: switch to the scene's device for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// fp64 box -> fp32, rounded outward and inflated (conservative slab tests).
float box_lo_f32(double x);
float box_hi_f32(double x);

// build / launch helpers (lbvh.cu, trace.cu, shade.cu)
srt_status lbvh_build(SrtScene *s, double cutoff_s, int method);
srt_status ploc_build(SrtScene *s, int64_t n, const uint32_t *slot_prim, const float *plo, const float *phi,
                      int *parent_int, int *parent_leaf, cudaStream_t st, Node2 *nodes,
                      const int *cell = nullptr);
srt_status collapse4(SrtScene *s);
// binary tree (m2 Node2, root 0) -> greedy 4-wide tree and its octant copies
srt_status collapse_tree(const Node2 *n2, int32_t m2, Node4 **out4, int32_t *m4, cudaStream_t st);
srt_status octant_copies(const Node4 *n4, int32_t m, Node4 **out8, cudaStream_t st);
srt_status launch_geom(int64_t n, const uint32_t *slot_prim, const SrtScene *s, Geom *out, cudaStream_t st);
// the packet walk's split tree (split.cu); free_split drops it
srt_status split_build(SrtScene *s, const float *plo, const float *phi, const int *cbounds, cudaStream_t st);
void free_split(SrtScene *s);
srt_status scratch_reserve(SrtScene *s, size_t bytes);
srt_status launch_pack_splats(int64_t n, const double *d_q, const double *d_scales, double *d_cov6, cudaStream_t st);

struct RenderArgs {
    int width, height, passes, nslots, mode, clip;
    float s2;
    double s2d;
    uint32_t seed;
    int pass0;
    float bg[3];
    int shard_index, shard_count;
    int tiles_x;
    int64_t local_tiles;
    int rng;
};
RenderArgs make_render_args(const SrtRenderParams *p);
CamD make_cam(const SrtCamera *c);

srt_status launch_trace_pass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, int32_t *d_hits,
                             cudaStream_t st);
srt_status launch_render_pass_fused(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass,
                                   float4 *d_accum, bool first, bool last, float4 *d_out, cudaStream_t st,
                                   int32_t *d_hits = nullptr, double *d_rgb64 = nullptr, double *d_op64 = nullptr,
                                   bool out_rowmajor = false, bool sys_fence = false);
srt_status launch_render_frame_multipass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass0,
                                         int npass, unsigned long long *d_acc64, cudaStream_t st);
srt_status launch_resolve_fixed(const RenderArgs &a, const unsigned long long *d_acc, int npass, float4 *d_out,
                                double *d_rgb, double *d_op, cudaStream_t st);
srt_status launch_shade_pass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass,
                             const int32_t *d_hits, float4 *d_accum, bool first, bool last, float4 *d_out,
                             cudaStream_t st);
srt_status launch_trace_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R,
                             int nslots, const double *d_table, float *d_t, int32_t *d_id, cudaStream_t st);
srt_status launch_trace_rays_trig64(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R,
                                    int nslots, double *d_t, int32_t *d_id, cudaStream_t st);
srt_status launch_trace_pass_trig64(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, double s2,
                                    int32_t *d_hits, cudaStream_t st);
srt_status launch_biased_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R, int kk,
                              const double *bg, const double *d_table, double *d_rgb, cudaStream_t st);
srt_status launch_biased_frame(const SrtScene *s, const CamD &cam, const SrtRenderParams *p, int kk,
                               double *d_rgb, cudaStream_t st);
srt_status launch_exact_rays(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max, int mode,
                             double s2, const double *bg, double *d_rgb, double *d_op, cudaStream_t st);
srt_status launch_exact_frame(const SrtScene *s, const CamD &cam, const RenderArgs &a, double *d_rgb, double *d_op,
                              cudaStream_t st);
srt_status launch_transmittance(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max,
                                int mode, double s2, double *d_out, cudaStream_t st);
srt_status launch_resolve_f64(const RenderArgs &a, const float4 *d_out, double *d_rgb, double *d_op,
                              cudaStream_t st);
srt_status launch_unpack(const float4 *d_gathered, int width, int height, int shard_count, int64_t max_tiles,
                         float4 *d_frame, cudaStream_t st);
// explicit-ray batches (trace.cu): a 64-ray probe for one origin / one
// hemisphere, the smallest batch walked as packets, and a coherence sort
// (Morton code of the origin + direction signs) returning a permutation
srt_status probe_rays(const double *d_rays, uint32_t R, bool &one_origin, bool &one_hemisphere, cudaStream_t st);
int64_t packet_min(bool one_origin);
srt_status sort_rays(const double *d_rays, uint32_t R, uint32_t **d_perm_out, void **d_mem_out, cudaStream_t st);
srt_status check_flag(const SrtScene *s, cudaStream_t st);
srt_status clear_flag(const SrtScene *s, cudaStream_t st);

// Work counter of ONE persistent-kernel launch on a caller's stream: 128 B of
// stream-ordered scratch (cudaMallocAsync from the device pool), zeroed on
// `st` and released on `st` after the launch.  Launches on different streams
// therefore never share a counter, whatever their number.
// Launches on the scene's own stream (the serialised host entry points) reuse
// the scene's counter pair, which every persistent kernel leaves zeroed
// (release_counter), so they add no allocation and no memset to the stream.
struct LaunchCounter {
    uint32_t *p = nullptr;
    cudaStream_t st = nullptr;
    bool owned = false;
    srt_status init(const SrtScene *s, cudaStream_t stream) {
        st = stream;
        if (stream == s->stream && s->d_counter) {
            p = s->d_counter;
            return SRT_OK;
        }
        owned = true;
        srt_status rc = cuda_status(cudaMallocAsync((void **)&p, 128, st), "work counter alloc");
        if (!rc) rc = cuda_status(cudaMemsetAsync(p, 0, 128, st), "work counter reset");
        return rc;
    }
    ~LaunchCounter() {
        if (owned && p) cudaFreeAsync(p, st);
    }
};

int64_t shard_tiles(int width, int height, int shard_index, int shard_count);

// Caller-array transfers (hostcopy.cu): pageable memory through the scene's
// page-locked ring with parallel host copies, pinned memory directly.  Both
// return with the host side complete (d2h: the data is in dst).
srt_status copy_h2d(SrtScene *s, void *dst, const void *src, size_t bytes, cudaStream_t st);
srt_status copy_d2h(SrtScene *s, void *dst, const void *src, size_t bytes, cudaStream_t st);
void stage_release(SrtScene *s);

}  // namespace srt
