// capi.cu -- extern "C" entry points of libsrt (include/srt.h).  No
// exception or CUDA error crosses the ABI: every failure becomes an
// srt_status plus a thread-local message (srt_last_error).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "srt_internal.h"

namespace srt {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

srt_status cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return SRT_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? SRT_ERR_OOM : SRT_ERR_CUDA;
}

float box_lo_f32(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -INFINITY);
    return f - (std::fabs(f) * 9.5367431640625e-07f + 1e-30f);
}
float box_hi_f32(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, INFINITY);
    return f + (std::fabs(f) * 9.5367431640625e-07f + 1e-30f);
}

srt_status scratch_reserve(SrtScene *s, size_t bytes) {
    if (bytes <= s->scratch_bytes) return SRT_OK;
    if (s->d_scratch) cudaFree(s->d_scratch);
    s->d_scratch = nullptr;
    s->scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&s->d_scratch, bytes);
    if (e != cudaSuccess) return cuda_status(e, "scratch allocation");
    s->scratch_bytes = bytes;
    return SRT_OK;
}

__global__ void k_pack_rays(const double *__restrict__ o, const double *__restrict__ d, int64_t R, double *rays) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    double *q = rays + i * 6;
    q[0] = o[i * 3], q[1] = o[i * 3 + 1], q[2] = o[i * 3 + 2];
    q[3] = d[i * 3], q[4] = d[i * 3 + 1], q[5] = d[i * 3 + 2];
}

static srt_status launch_pack_rays(const double *d_o, const double *d_d, int64_t R, double *d_rays, cudaStream_t st) {
    k_pack_rays<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(d_o, d_d, R, d_rays);
    return cuda_status(cudaGetLastError(), "k_pack_rays");
}

// The caller's (R,3) origin and direction arrays -> (R,6) ray records on the
// device: two contiguous uploads into `stage` (48 R bytes), interleaved there
// (no host packing pass).
static srt_status upload_rays(SrtScene *s, const double *o, const double *d, int64_t R, double *stage,
                              double *d_rays, cudaStream_t st) {
    srt_status rc = copy_h2d(s, stage, o, sizeof(double) * 3 * R, st);
    if (!rc) rc = copy_h2d(s, stage + 3 * R, d, sizeof(double) * 3 * R, st);
    if (!rc) rc = launch_pack_rays(stage, stage + 3 * R, R, d_rays, st);
    return rc;
}

// t32 (f32 walk depths) or t64 (trig64 depths); misses (id < 0) -> +inf
__global__ void k_widen_hits(const float *__restrict__ t32, const double *__restrict__ t64,
                             const int32_t *__restrict__ id, int64_t m, double *t, int64_t *id64) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int32_t h = id[i];
    double v = t32 ? (double)t32[i] : t64[i];
    t[i] = t32 && h < 0 ? INFINITY : v;
    id64[i] = h;
}

static srt_status launch_widen_hits(const float *t32, const double *t64, const int32_t *id, int64_t m, double *t,
                             int64_t *id64, cudaStream_t st) {
    k_widen_hits<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(t32, t64, id, m, t, id64);
    return cuda_status(cudaGetLastError(), "k_widen_hits");
}

int64_t shard_tiles(int width, int height, int shard_index, int shard_count) {
    int64_t total = (int64_t)((width + 15) / 16) * ((height + 15) / 16);
    if (shard_count <= 1) return total;
    if (shard_index >= total) return 0;
    return (total - shard_index + shard_count - 1) / shard_count;
}

RenderArgs make_render_args(const SrtRenderParams *p) {
    RenderArgs a;
    a.width = p->width;
    a.height = p->height;
    a.passes = p->passes;
    a.nslots = p->nslots;
    a.mode = p->mode;
    a.clip = p->clip;
    a.s2 = (float)p->s2;
    a.s2d = p->s2;
    a.seed = p->seed;
    a.pass0 = p->pass0;
    for (int k = 0; k < 3; ++k) a.bg[k] = (float)p->background[k];
    a.shard_count = p->shard_count < 1 ? 1 : p->shard_count;
    a.shard_index = p->shard_count < 1 ? 0 : p->shard_index;
    a.tiles_x = (p->width + 15) / 16;
    a.local_tiles = shard_tiles(p->width, p->height, a.shard_index, a.shard_count);
    a.rng = p->rng;
    return a;
}

CamD make_cam(const SrtCamera *c) {
    CamD d;
    for (int k = 0; k < 3; ++k) {
        d.e[k] = c->position[k];
        d.r[k] = c->right[k];
        d.u[k] = c->up[k];
        d.f[k] = c->forward[k];
    }
    d.half_w = c->half_w;
    d.half_h = c->half_h;
    return d;
}

// The flag lives in mapped host memory: synchronise, then read it directly.
srt_status check_flag(const SrtScene *s, cudaStream_t st) {
    srt_status rc = cuda_status(cudaStreamSynchronize(st), "stream sync");
    if (rc) return rc;
    if (*(volatile int32_t *)s->h_flag) {
        *(volatile int32_t *)s->h_flag = 0;
        set_error("traversal stack overflow (BVH deeper than the 128-entry stack)");
        return SRT_ERR_STACK_OVERFLOW;
    }
    return SRT_OK;
}

srt_status clear_flag(const SrtScene *s, cudaStream_t) {
    *(volatile int32_t *)s->h_flag = 0;  // host memory: no stream operation
    return SRT_OK;
}

static srt_status validate_render(const SrtScene *s, const SrtRenderParams *p) {
    if (!s) {
        set_error("null scene");
        return SRT_ERR_INVALID_ARG;
    }
    if (!s->has_bvh) {
        set_error("scene has no BVH (call srt_bvh_build or srt_bvh_upload)");
        return SRT_ERR_NO_BVH;
    }
    if (!p || p->width < 1 || p->height < 1 || p->passes < 1 || p->nslots < 1 || p->nslots > 256 ||
        (p->mode != 0 && p->mode != 1) || !(p->s2 > 0.0) || p->pass0 < 0 ||
        (p->rng != 0 && p->rng != SRT_RNG_COUNTER && p->rng != SRT_RNG_TRIG64)) {
        set_error("invalid render parameters");
        return SRT_ERR_INVALID_ARG;
    }
    if (p->shard_count > 1 && (p->shard_index < 0 || p->shard_index >= p->shard_count)) {
        set_error("invalid shard index");
        return SRT_ERR_INVALID_ARG;
    }
    return SRT_OK;
}

}  // namespace srt

using namespace srt;

// serialise host entry points on one scene handle (null-safe)
#define SRT_LOCK(sc)                              \
    std::unique_lock<std::mutex> srt_lock_;       \
    if (sc) srt_lock_ = std::unique_lock<std::mutex>((sc)->mu)

extern "C" {

const char *srt_last_error(void) { return g_last_error.c_str(); }
const char *srt_version(void) { return "libsrt 0.2 (sm_100a)"; }
#ifndef SRT_BUILD_ID
#define SRT_BUILD_ID "unknown"
#endif
const char *srt_build_id(void) { return SRT_BUILD_ID; }

int32_t srt_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Device address of a mapped page-locked host buffer, or nullptr for
// pageable / device memory.
static double *mapped_host(double *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return (double *)at.devicePointer;
}

srt_status srt_host_alloc(int64_t bytes, void **out) {
    if (!out || bytes < 0) {
        set_error("invalid host allocation");
        return SRT_ERR_INVALID_ARG;
    }
    *out = nullptr;
    return cuda_status(cudaHostAlloc(out, (size_t)(bytes ? bytes : 1), cudaHostAllocPortable | cudaHostAllocMapped),
                       "cudaHostAlloc");
}

srt_status srt_host_register(void *ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) {
        set_error("invalid host registration");
        return SRT_ERR_INVALID_ARG;
    }
    return cuda_status(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterPortable | cudaHostRegisterMapped),
                       "cudaHostRegister");
}

srt_status srt_host_unregister(void *ptr) {
    if (!ptr) return SRT_OK;
    return cuda_status(cudaHostUnregister(ptr), "cudaHostUnregister");
}

srt_status srt_host_free(void *ptr) {
    if (!ptr) return SRT_OK;
    return cuda_status(cudaFreeHost(ptr), "cudaFreeHost");
}

srt_status srt_scene_create(const SrtSceneDesc *desc, int32_t device, SrtScene **out) {
    if (!desc || !out || desc->n < 0 || desc->sh_degree < 0 || desc->sh_degree > 3 ||
        (desc->n > 0 && (!desc->means || !desc->cov_inv6 || !desc->opacities))) {
        set_error("invalid scene description");
        return SRT_ERR_INVALID_ARG;
    }
    *out = nullptr;
    int ndev = srt_device_count();
    if (device < 0 || device >= ndev) {
        set_error("CUDA device " + std::to_string(device) + " not available (" + std::to_string(ndev) + " devices)");
        return SRT_ERR_CUDA;
    }
    DeviceGuard g(device);
    {
        // stream-ordered scratch (ray sorting) stays pooled between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    SrtScene *s = new SrtScene();
    s->device = device;
    s->n = desc->n;
    s->sh_deg = desc->sh_degree;
    s->sh_k = (desc->sh_degree + 1) * (desc->sh_degree + 1);
    const int64_t n = desc->n;
    srt_status rc = SRT_OK;
    std::vector<float> shf;
    rc = cuda_status(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "stream create");
    if (!rc) rc = cuda_status(cudaHostAlloc(&s->h_flag, sizeof(int32_t), cudaHostAllocMapped), "flag alloc");
    if (!rc) {
        *s->h_flag = 0;
        rc = cuda_status(cudaHostGetDevicePointer(&s->d_flag, s->h_flag, 0), "flag map");
    }
    if (!rc) rc = cuda_status(cudaMalloc(&s->d_counter, 128), "work counter alloc");
    if (!rc) rc = cuda_status(cudaMemset(s->d_counter, 0, 128), "work counter init");
    if (!rc) rc = cuda_status(cudaMalloc(&s->d_stats, sizeof(unsigned long long) * 16), "stats alloc");
    if (!rc) rc = cuda_status(cudaMemset(s->d_stats, 0, sizeof(unsigned long long) * 16), "stats init");
    if (!rc && n > 0) {
        // uploads are ordered on the scene's stream: cudaMemcpy from pageable
        // memory may return before the DMA lands, and the scene's stream does
        // not synchronise with the legacy default stream
        cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
        rc = cuda_status(cudaMalloc(&s->d_means, sizeof(double) * n * 3), "means alloc");
        if (!rc) rc = cuda_status(cudaMalloc(&s->d_cov6, sizeof(double) * n * 6), "cov alloc");
        if (!rc) rc = cuda_status(cudaMalloc(&s->d_opac, sizeof(double) * n), "opacity alloc");
        if (!rc) rc = cuda_status(cudaMalloc(&s->d_sh, sizeof(float) * n * 3 * s->sh_k), "sh alloc");
        if (!rc) rc = copy_h2d(s, s->d_means, desc->means, sizeof(double) * n * 3, st);
        if (!rc) rc = copy_h2d(s, s->d_cov6, desc->cov_inv6, sizeof(double) * n * 6, st);
        if (!rc) rc = copy_h2d(s, s->d_opac, desc->opacities, sizeof(double) * n, st);
        if (!rc) {
            shf.assign((size_t)n * 3 * s->sh_k, 0.0f);
            if (desc->sh)
                for (size_t i = 0; i < shf.size(); ++i) shf[i] = (float)desc->sh[i];
            rc = cuda_status(cudaMemcpyAsync(s->d_sh, shf.data(), sizeof(float) * shf.size(), cudaMemcpyHostToDevice, st), "sh upload");
        }
        if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "scene upload");
    }
    if (rc) {
        srt_scene_destroy(s);
        return rc;
    }
    *out = s;
    return SRT_OK;
}

srt_status srt_scene_create_from_splats(const SrtSplatDesc *desc, int32_t device, SrtScene **out) {
    if (!desc || !out || desc->n < 0 || (desc->n > 0 && (!desc->means || !desc->rotations || !desc->scales ||
                                                         !desc->opacities))) {
        set_error("invalid splat description");
        return SRT_ERR_INVALID_ARG;
    }
    const int64_t n = desc->n;
    // create with a placeholder covariance, then pack on the device
    std::vector<double> zero6((size_t)(n > 0 ? n : 1) * 6, 0.0);
    SrtSceneDesc d{n, desc->means, zero6.data(), desc->opacities, desc->sh, desc->sh_degree};
    srt_status rc = srt_scene_create(&d, device, out);
    if (rc || n == 0) return rc;
    SrtScene *s = *out;
    DeviceGuard g(s->device);
    double *d_q = nullptr, *d_s = nullptr;
    rc = cuda_status(cudaMalloc(&d_q, sizeof(double) * n * 4), "quaternion alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&d_s, sizeof(double) * n * 3), "scale alloc");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(d_q, desc->rotations, sizeof(double) * n * 4, cudaMemcpyHostToDevice, s->stream), "q upload");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(d_s, desc->scales, sizeof(double) * n * 3, cudaMemcpyHostToDevice, s->stream), "s upload");
    if (!rc) rc = launch_pack_splats(n, d_q, d_s, s->d_cov6, s->stream);
    if (!rc) rc = cuda_status(cudaStreamSynchronize(s->stream), "pack");
    cudaFree(d_q);
    cudaFree(d_s);
    if (rc) {
        srt_scene_destroy(s);
        *out = nullptr;
    }
    return rc;
}

srt_status srt_scene_destroy(SrtScene *s) {
    if (!s) return SRT_OK;
    DeviceGuard g(s->device);
    cudaFree(s->d_means);
    cudaFree(s->d_cov6);
    cudaFree(s->d_opac);
    cudaFree(s->d_sh);
    cudaFree(s->d_geom);
    cudaFree(s->d_nodes);
    cudaFree(s->d_nodes4);
    cudaFree(s->d_nodes8);
    free_split(s);
    cudaFree(s->d_stats);
    if (s->h_flag) cudaFreeHost(s->h_flag);
    cudaFree(s->d_counter);
    cudaFree(s->d_scratch);
    stage_release(s);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return SRT_OK;
}

srt_status srt_bvh_build_ex(SrtScene *s, double cutoff_s, int32_t method) {
    SRT_LOCK(s);
    if (!s || !(cutoff_s > 0.0) || !std::isfinite(cutoff_s) || (method != SRT_BVH_LBVH && method != SRT_BVH_PLOC)) {
        set_error("invalid scene, cutoff or build method");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return lbvh_build(s, cutoff_s, method);
}

srt_status srt_bvh_build(SrtScene *s, double cutoff_s) { return srt_bvh_build_ex(s, cutoff_s, SRT_BVH_PLOC); }

// Reference layout (bvh.py:29-47) -> Node2 tree.  A reference leaf with k
// primitives becomes a balanced subtree over the k primitive boxes, so the
// per-primitive box test of kernels.py:344 is kept exactly (boxes widened
// to fp32 outward).
srt_status srt_bvh_upload(SrtScene *s, int64_t M, const double *node_lo, const double *node_hi, const int64_t *node_left,
                          const int64_t *node_right, const int64_t *node_count, const int64_t *prim_order,
                          const double *prim_lo, const double *prim_hi) {
    SRT_LOCK(s);
    if (!s || M < 0 || (M > 0 && (!node_lo || !node_hi || !node_left || !node_right || !node_count || !prim_order ||
                                  !prim_lo || !prim_hi))) {
        set_error("invalid BVH arrays");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    const int64_t n = s->n;
    std::vector<Node2> nodes;
    struct Box {
        float lo[3], hi[3];
    };
    auto prim_box = [&](int64_t slot) {
        Box b;
        int64_t p = prim_order[slot];
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = box_lo_f32(prim_lo[p * 3 + k]);
            b.hi[k] = box_hi_f32(prim_hi[p * 3 + k]);
        }
        return b;
    };
    auto node_box = [&](int64_t id) {
        Box b;
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = box_lo_f32(node_lo[id * 3 + k]);
            b.hi[k] = box_hi_f32(node_hi[id * 3 + k]);
        }
        return b;
    };
    auto set_node = [&](int32_t idx, int c0, const Box &b0, int c1, const Box &b1) {
        Node2 &nd = nodes[idx];
        nd.xy0 = make_float4(b0.lo[0], b0.hi[0], b0.lo[1], b0.hi[1]);
        nd.xy1 = make_float4(b1.lo[0], b1.hi[0], b1.lo[1], b1.hi[1]);
        nd.z01 = make_float4(b0.lo[2], b0.hi[2], b1.lo[2], b1.hi[2]);
        nd.kids = make_int4(c0, c1, 0, 0);
    };
    Box empty;
    for (int k = 0; k < 3; ++k) {
        empty.lo[k] = 3.0e38f;
        empty.hi[k] = -3.0e38f;
    }
    bool bad = false;
    int32_t max_depth = 0;
    // subtree over leaf slots [start, start+k): returns child code; box out
    std::function<int(int64_t, int64_t, Box &, int)> leaf_tree = [&](int64_t start, int64_t k, Box &box, int depth) -> int {
        max_depth = std::max(max_depth, depth);
        if (k == 1) {
            box = prim_box(start);
            return ~(int)start;
        }
        int32_t idx = (int32_t)nodes.size();
        nodes.emplace_back();
        Box b0, b1;
        int64_t half = k / 2;
        int c0 = leaf_tree(start, half, b0, depth + 1);
        int c1 = leaf_tree(start + half, k - half, b1, depth + 1);
        set_node(idx, c0, b0, c1, b1);
        for (int a = 0; a < 3; ++a) {
            box.lo[a] = std::min(b0.lo[a], b1.lo[a]);
            box.hi[a] = std::max(b0.hi[a], b1.hi[a]);
        }
        return idx;
    };
    std::function<int(int64_t, Box &, int)> emit = [&](int64_t id, Box &box, int depth) -> int {
        if (id < 0 || id >= M || depth > 256) {
            bad = true;
            return kLeafEmpty;
        }
        max_depth = std::max(max_depth, depth);
        int64_t cnt = node_count[id];
        if (cnt > 0) {
            int64_t start = node_left[id];
            if (start < 0 || start + cnt > n) {
                bad = true;
                return kLeafEmpty;
            }
            Box inner;
            int code = leaf_tree(start, cnt, inner, depth);
            box = cnt == 1 ? inner : node_box(id);
            return code;
        }
        int32_t idx = (int32_t)nodes.size();
        nodes.emplace_back();
        Box b0, b1;
        int c0 = emit(node_left[id], b0, depth + 1);
        int c1 = emit(node_right[id], b1, depth + 1);
        set_node(idx, c0, b0, c1, b1);
        box = node_box(id);
        return idx;
    };
    if (M > 0) {
        Box rb;
        nodes.reserve((size_t)(2 * n + 1));
        int root = emit(0, rb, 1);
        if (root < 0 && root != kLeafEmpty) {  // single-primitive root leaf: wrap it
            nodes.emplace_back();
            set_node(0, root, rb, kLeafEmpty, empty);
        }
    }
    if (bad) {
        set_error("malformed reference BVH arrays");
        return SRT_ERR_INVALID_ARG;
    }
    // slot-ordered geometry from prim_order
    free_split(s);
    if (s->d_nodes) cudaFree(s->d_nodes);
    if (s->d_geom) cudaFree(s->d_geom);
    s->d_nodes = nullptr;
    s->d_geom = nullptr;
    s->has_bvh = false;
    srt_status rc = SRT_OK;
    if (!nodes.empty()) {
        rc = cuda_status(cudaMalloc(&s->d_nodes, sizeof(Node2) * nodes.size()), "node alloc");
        if (!rc)
            rc = cuda_status(cudaMemcpyAsync(s->d_nodes, nodes.data(), sizeof(Node2) * nodes.size(),
                                             cudaMemcpyHostToDevice, s->stream),
                             "node upload");
        if (!rc) rc = cuda_status(cudaStreamSynchronize(s->stream), "node upload");
    }
    if (!rc && n > 0) {
        // gather the fp64 records on the host in slot order, convert on device
        std::vector<double> pm(n * 3), pc(n * 6), po(n);
        std::vector<Geom> geom(n);
        std::vector<double> hm(n * 3), hc(n * 6), ho(n);
        rc = cuda_status(cudaMemcpy(hm.data(), s->d_means, sizeof(double) * n * 3, cudaMemcpyDeviceToHost), "means");
        if (!rc) rc = cuda_status(cudaMemcpy(hc.data(), s->d_cov6, sizeof(double) * n * 6, cudaMemcpyDeviceToHost), "cov");
        if (!rc) rc = cuda_status(cudaMemcpy(ho.data(), s->d_opac, sizeof(double) * n, cudaMemcpyDeviceToHost), "opac");
        if (!rc) {
            for (int64_t j = 0; j < n; ++j) {
                int64_t p = prim_order[j];
                if (p < 0 || p >= n) {
                    set_error("prim_order out of range");
                    return SRT_ERR_INVALID_ARG;
                }
                Geom &gg = geom[j];
                gg.m = make_float4((float)hm[p * 3], (float)hm[p * 3 + 1], (float)hm[p * 3 + 2], (float)ho[p]);
                gg.a = make_float4((float)hc[p * 6], (float)hc[p * 6 + 1], (float)hc[p * 6 + 2], (float)hc[p * 6 + 3]);
                int pi = (int)p;
                float pf;
                std::memcpy(&pf, &pi, sizeof(pf));
                const double *cc = &hc[p * 6];
                double tr = std::fabs(cc[0]) + std::fabs(cc[3]) + std::fabs(cc[5]) +
                            2.0 * (std::fabs(cc[1]) + std::fabs(cc[2]) + std::fabs(cc[4]));
                gg.b = make_float4((float)cc[4], (float)cc[5], pf, (float)(std::sqrt(tr) * 1.0000002));
            }
            rc = cuda_status(cudaMalloc(&s->d_geom, sizeof(Geom) * n), "geom alloc");
            if (!rc)
                rc = cuda_status(cudaMemcpyAsync(s->d_geom, geom.data(), sizeof(Geom) * n, cudaMemcpyHostToDevice,
                                                 s->stream),
                                 "geom upload");
            if (!rc) rc = cuda_status(cudaStreamSynchronize(s->stream), "geom upload");
        }
    }
    if (rc) return rc;
    s->num_nodes = (int32_t)nodes.size();
    s->depth = max_depth + 1;
    rc = collapse4(s);
    if (rc) return rc;
    s->has_bvh = true;
    return SRT_OK;
}

srt_status srt_bvh_info(const SrtScene *s, int64_t *num_nodes, int32_t *depth, int64_t *num_prims,
                        int64_t *device_bytes) {
    if (!s) {
        set_error("null scene");
        return SRT_ERR_INVALID_ARG;
    }
    if (num_nodes) *num_nodes = s->num_nodes;
    if (depth) *depth = s->depth;
    if (num_prims) *num_prims = s->n;
    if (device_bytes)
        *device_bytes = (int64_t)sizeof(Node2) * s->num_nodes + (int64_t)sizeof(Node4) * 9 * s->num_nodes4 +
                        (int64_t)sizeof(Geom) * s->n + (int64_t)sizeof(float) * s->n * 3 * s->sh_k +
                        (int64_t)sizeof(Node4) * 9 * s->num_nodes4_split + (int64_t)sizeof(Geom) * s->n_refs;
    return SRT_OK;
}

srt_status srt_bvh_split_info(const SrtScene *s, int64_t *num_refs, int32_t *num_nodes4, int32_t *cells) {
    if (!s) {
        set_error("null scene");
        return SRT_ERR_INVALID_ARG;
    }
    if (num_refs) *num_refs = s->n_refs;
    if (num_nodes4) *num_nodes4 = s->num_nodes4_split;
    if (cells) *cells = s->split_cells;
    return SRT_OK;
}

// Download in the reference layout: internal nodes of the device tree become
// reference inner nodes; each leaf child becomes a one-primitive leaf node.
srt_status srt_bvh_download(const SrtScene *s, float *node_lo, float *node_hi, int64_t *node_left,
                            int64_t *node_right, int64_t *node_count, int64_t *prim_order, float *prim_lo,
                            float *prim_hi) {
    SRT_LOCK(s);
    if (!s || !s->has_bvh) {
        set_error("scene has no BVH");
        return SRT_ERR_NO_BVH;
    }
    DeviceGuard g(s->device);
    const int64_t n = s->n;
    std::vector<Node2> nodes(s->num_nodes);
    std::vector<Geom> geom(n);
    srt_status rc = SRT_OK;
    if (s->num_nodes)
        rc = cuda_status(cudaMemcpy(nodes.data(), s->d_nodes, sizeof(Node2) * nodes.size(), cudaMemcpyDeviceToHost), "nodes");
    if (!rc && n)
        rc = cuda_status(cudaMemcpy(geom.data(), s->d_geom, sizeof(Geom) * n, cudaMemcpyDeviceToHost), "geom");
    if (rc) return rc;
    for (int64_t j = 0; j < n; ++j) {
        int p;
        std::memcpy(&p, &geom[j].b.z, sizeof(int));
        prim_order[j] = p;
    }
    // reference node ids: device inner node i -> i; leaf slot j -> num_nodes + j
    const int64_t Mi = s->num_nodes;
    auto put = [&](int64_t id, const float lo[3], const float hi[3]) {
        for (int k = 0; k < 3; ++k) {
            node_lo[id * 3 + k] = lo[k];
            node_hi[id * 3 + k] = hi[k];
        }
    };
    std::vector<char> seen(n, 0);
    for (int64_t i = 0; i < Mi; ++i) {
        const Node2 &nd = nodes[i];
        float lo0[3] = {nd.xy0.x, nd.xy0.z, nd.z01.x}, hi0[3] = {nd.xy0.y, nd.xy0.w, nd.z01.y};
        float lo1[3] = {nd.xy1.x, nd.xy1.z, nd.z01.z}, hi1[3] = {nd.xy1.y, nd.xy1.w, nd.z01.w};
        int kids[2] = {nd.kids.x, nd.kids.y};
        const float *los[2] = {lo0, lo1}, *his[2] = {hi0, hi1};
        int64_t ref[2];
        for (int c = 0; c < 2; ++c) {
            if (kids[c] == kLeafEmpty) {
                ref[c] = -1;
            } else if (kids[c] < 0) {
                int64_t slot = ~kids[c];
                int64_t id = Mi + slot;
                ref[c] = id;
                put(id, los[c], his[c]);
                node_left[id] = slot;
                node_right[id] = -1;
                node_count[id] = 1;
                seen[slot] = 1;
                int p = (int)prim_order[slot];
                for (int k = 0; k < 3; ++k) {
                    prim_lo[(int64_t)p * 3 + k] = los[c][k];
                    prim_hi[(int64_t)p * 3 + k] = his[c][k];
                }
            } else {
                ref[c] = kids[c];
                put(kids[c], los[c], his[c]);
            }
        }
        node_left[i] = ref[0];
        node_right[i] = ref[1];
        node_count[i] = 0;
    }
    if (Mi > 0) {
        // root box = union of its children
        const Node2 &r = nodes[0];
        float lo[3] = {std::min(r.xy0.x, r.xy1.x), std::min(r.xy0.z, r.xy1.z), std::min(r.z01.x, r.z01.z)};
        float hi[3] = {std::max(r.xy0.y, r.xy1.y), std::max(r.xy0.w, r.xy1.w), std::max(r.z01.y, r.z01.w)};
        if (r.kids.y == kLeafEmpty) {
            float lo0[3] = {r.xy0.x, r.xy0.z, r.z01.x}, hi0[3] = {r.xy0.y, r.xy0.w, r.z01.y};
            put(0, lo0, hi0);
        } else {
            put(0, lo, hi);
        }
    }
    for (int64_t j = 0; j < n; ++j)
        if (!seen[j]) {
            set_error("device BVH does not reference every primitive");
            return SRT_ERR_CUDA;
        }
    return SRT_OK;
}

// ---- explicit rays --------------------------------------------------------

static srt_status validate_trace(const SrtScene *s, const SrtTraceParams *p, int64_t R, int32_t nslots) {
    if (!s || !p || R < 0 || nslots < 1 || nslots > 256 || (p->mode != 0 && p->mode != 1) || !(p->s2 > 0.0) ||
        (p->rng != SRT_RNG_COUNTER && p->rng != SRT_RNG_TABLE && p->rng != SRT_RNG_TRIG64) ||
        (p->rng == SRT_RNG_TABLE && (!p->table || p->table_slots < nslots))) {
        set_error("invalid trace parameters");
        return SRT_ERR_INVALID_ARG;
    }
    if (!s->has_bvh) {
        set_error("scene has no BVH (call srt_bvh_build or srt_bvh_upload)");
        return SRT_ERR_NO_BVH;
    }
    return SRT_OK;
}

srt_status srt_trace_rays_device(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R,
                                 int32_t nslots, float *d_t, int32_t *d_id, void *stream) {
    srt_status rc = validate_trace(s, p, R, nslots);
    if (rc) return rc;
    if (p->rng == SRT_RNG_TABLE || p->rng == SRT_RNG_TRIG64) {
        set_error("table / trig64 RNG need the host entry point (srt_trace_rays)");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return launch_trace_rays(s, p, d_rays, R, nslots, nullptr, d_t, d_id, (cudaStream_t)stream);
}

srt_status srt_trace_rays(const SrtScene *sc, const SrtTraceParams *p, const double *origins, const double *dirs,
                          int64_t R, int32_t nslots, double *out_t, int64_t *out_id) {
    SRT_LOCK(sc);
    srt_status rc = validate_trace(sc, p, R, nslots);
    if (rc) return rc;
    if (R == 0) return SRT_OK;
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    size_t ray_bytes = sizeof(double) * R * 6;
    size_t out_bytes = (sizeof(double) + sizeof(int32_t)) * R * nslots;
    size_t table_bytes = p->rng == SRT_RNG_TABLE ? sizeof(double) * s->n * p->table_slots : 0;
    // staging: the caller's (R,3) origin and direction arrays on the way in,
    // the widened (f64 t, i64 id) outputs on the way out
    size_t stage_bytes = std::max(ray_bytes, sizeof(double) * 2 * R * nslots);
    size_t stage_off = (ray_bytes + out_bytes + table_bytes + 255) & ~(size_t)255;
    rc = scratch_reserve(s, stage_off + stage_bytes);
    if (rc) return rc;
    char *base = (char *)s->d_scratch;
    double *d_rays = (double *)base;
    float *d_t = (float *)(base + ray_bytes);
    int32_t *d_id = (int32_t *)(base + ray_bytes + sizeof(float) * R * nslots);
    double *d_table = table_bytes ? (double *)(base + ((ray_bytes + out_bytes + 15) & ~(size_t)15)) : nullptr;
    double *d_stage = (double *)(base + stage_off);
    // contiguous uploads straight from the caller's arrays, interleaved into
    // the (R,6) ray records on the device (no host packing pass)
    rc = upload_rays(s, origins, dirs, R, d_stage, d_rays, st);
    if (!rc && d_table)
        rc = copy_h2d(s, d_table, p->table, table_bytes, st);
    double *d_t64 = (double *)(base + ray_bytes);
    if (p->rng == SRT_RNG_TRIG64) d_id = (int32_t *)(base + ray_bytes + sizeof(double) * R * nslots);
    if (!rc) {
        if (p->rng == SRT_RNG_TRIG64)
            rc = launch_trace_rays_trig64(s, p, d_rays, R, nslots, d_t64, d_id, st);
        else
            rc = launch_trace_rays(s, p, d_rays, R, nslots, d_table, d_t, d_id, st);
    }
    // widen on the device (f32 t -> f64, +inf on miss; i32 id -> i64) and
    // download straight into the caller's arrays
    const int64_t m = R * (int64_t)nslots;
    double *w_t = d_stage;
    int64_t *w_id = (int64_t *)(d_stage + m);
    if (!rc) rc = launch_widen_hits(p->rng == SRT_RNG_TRIG64 ? nullptr : d_t, p->rng == SRT_RNG_TRIG64 ? d_t64 : nullptr,
                                    d_id, m, w_t, w_id, st);
    if (!rc) rc = copy_d2h(s, out_t, w_t, sizeof(double) * m, st);
    if (!rc) rc = copy_d2h(s, out_id, w_id, sizeof(int64_t) * m, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_transmittance_rays(const SrtScene *sc, const double *origins, const double *dirs, int64_t R,
                                  double t_min, double t_max, int32_t mode, double s2, double *out) {
    SRT_LOCK(sc);
    if (!sc || R < 0 || (mode != 0 && mode != 1) || !(s2 > 0.0)) {
        set_error("invalid transmittance parameters");
        return SRT_ERR_INVALID_ARG;
    }
    if (!sc->has_bvh) {
        set_error("scene has no BVH");
        return SRT_ERR_NO_BVH;
    }
    if (R == 0) return SRT_OK;
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    size_t ray_bytes = sizeof(double) * R * 6;
    srt_status rc = scratch_reserve(s, 2 * ray_bytes + sizeof(double) * R);
    if (rc) return rc;
    double *d_rays = (double *)s->d_scratch;
    double *d_out = d_rays + R * 6;
    rc = upload_rays(s, origins, dirs, R, d_out + R, d_rays, st);
    if (!rc) rc = launch_transmittance(s, d_rays, R, t_min, t_max, mode, s2, d_out, st);
    if (!rc) rc = copy_d2h(s, out, d_out, sizeof(double) * R, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_exact_rays(const SrtScene *sc, const double *origins, const double *dirs, int64_t R, double t_min,
                          double t_max, int32_t mode, double s2, const double *background, double *out_rgb,
                          double *out_op) {
    SRT_LOCK(sc);
    if (!sc || R < 0 || (mode != 0 && mode != 1) || !(s2 > 0.0) || !background || (R > 0 && (!out_rgb || !out_op))) {
        set_error("invalid exact-compositing parameters");
        return SRT_ERR_INVALID_ARG;
    }
    if (!sc->has_bvh) {
        set_error("scene has no BVH");
        return SRT_ERR_NO_BVH;
    }
    if (R == 0) return SRT_OK;
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    size_t ray_bytes = sizeof(double) * R * 6;
    srt_status rc = scratch_reserve(s, 2 * ray_bytes + sizeof(double) * R * 4);
    if (rc) return rc;
    double *d_rays = (double *)s->d_scratch;
    double *d_rgb = d_rays + R * 6;
    double *d_op = d_rgb + R * 3;
    rc = upload_rays(s, origins, dirs, R, d_op + R, d_rays, st);
    if (!rc) rc = launch_exact_rays(s, d_rays, R, t_min, t_max, mode, s2, background, d_rgb, d_op, st);
    if (!rc) rc = copy_d2h(s, out_rgb, d_rgb, sizeof(double) * R * 3, st);
    if (!rc) rc = copy_d2h(s, out_op, d_op, sizeof(double) * R, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_biased_rays(const SrtScene *sc, const SrtTraceParams *p, const double *origins, const double *dirs,
                           int64_t R, int32_t kk, const double *background, double *out_rgb) {
    SRT_LOCK(sc);
    srt_status rc = validate_trace(sc, p, R, 1);
    if (rc) return rc;
    if (kk < 1 || !background || (R > 0 && (!origins || !dirs || !out_rgb))) {
        set_error("invalid biased-composite parameters (k must be >= 1)");
        return SRT_ERR_INVALID_ARG;
    }
    if (R == 0) return SRT_OK;
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    size_t ray_bytes = sizeof(double) * R * 6;
    size_t rgb_bytes = sizeof(double) * R * 3;
    size_t table_bytes = p->rng == SRT_RNG_TABLE ? sizeof(double) * s->n * p->table_slots : 0;
    rc = scratch_reserve(s, 2 * ray_bytes + rgb_bytes + table_bytes);
    if (rc) return rc;
    double *d_rays = (double *)s->d_scratch;
    double *d_rgb = d_rays + R * 6;
    double *d_table = table_bytes ? d_rgb + R * 3 : nullptr;
    rc = upload_rays(s, origins, dirs, R, (double *)((char *)(d_rgb + R * 3) + table_bytes), d_rays, st);
    if (!rc && d_table)
        rc = copy_h2d(s, d_table, p->table, table_bytes, st);
    if (!rc) rc = launch_biased_rays(s, p, d_rays, R, kk, background, d_table, d_rgb, st);
    if (!rc) rc = copy_d2h(s, out_rgb, d_rgb, rgb_bytes, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_render_biased(const SrtScene *sc, const SrtCamera *camera, const SrtRenderParams *p, int32_t kk,
                             double *out_rgb) {
    SRT_LOCK(sc);
    srt_status rc = validate_render(sc, p);
    if (rc) return rc;
    if (!camera || !out_rgb || kk < 1 || p->rng == SRT_RNG_TABLE) {
        set_error("invalid biased-frame parameters (k >= 1; counter or trig64 draws)");
        return SRT_ERR_INVALID_ARG;
    }
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    const int64_t npix = (int64_t)p->width * p->height;
    rc = scratch_reserve(s, sizeof(double) * npix * 3);
    if (rc) return rc;
    double *d_rgb = (double *)s->d_scratch;
    rc = launch_biased_frame(s, make_cam(camera), p, kk, d_rgb, st);
    if (!rc) rc = copy_d2h(s, out_rgb, d_rgb, sizeof(double) * npix * 3, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_render_exact(const SrtScene *sc, const SrtCamera *camera, const SrtRenderParams *p, double *out_rgb,
                            double *out_op) {
    SRT_LOCK(sc);
    srt_status rc = validate_render(sc, p);
    if (rc) return rc;
    if (!camera || !out_rgb || !out_op) {
        set_error("null camera or output");
        return SRT_ERR_INVALID_ARG;
    }
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    const int64_t npix = (int64_t)p->width * p->height;
    rc = scratch_reserve(s, sizeof(double) * npix * 4);
    if (rc) return rc;
    double *d_rgb = (double *)s->d_scratch;
    double *d_op = d_rgb + npix * 3;
    rc = launch_exact_frame(s, make_cam(camera), make_render_args(p), d_rgb, d_op, st);
    if (!rc) rc = copy_d2h(s, out_rgb, d_rgb, sizeof(double) * npix * 3, st);
    if (!rc) rc = copy_d2h(s, out_op, d_op, sizeof(double) * npix, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

// ---- frames ----------------------------------------------------------------

int64_t srt_shard_tiles(int32_t width, int32_t height, int32_t shard_index, int32_t shard_count) {
    return shard_tiles(width, height, shard_index, shard_count);
}

srt_status srt_trace_pass_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p, int32_t pass,
                                 int32_t *d_hits, void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_hits) {
        set_error("null camera or hit buffer");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return launch_trace_pass(s, make_cam(camera), make_render_args(p), pass, d_hits, (cudaStream_t)stream);
}

srt_status srt_shade_pass_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p, int32_t pass,
                                 const int32_t *d_hits, float *d_accum, int32_t first, int32_t last, float *d_out,
                                 void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_hits || !d_accum || (last && !d_out)) {
        set_error("null camera or buffer");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return launch_shade_pass(s, make_cam(camera), make_render_args(p), pass, d_hits, (float4 *)d_accum, first != 0,
                             last != 0, (float4 *)d_out, (cudaStream_t)stream);
}

srt_status srt_render_pass_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p, int32_t pass,
                                  float *d_accum, int32_t first, int32_t last, float *d_out, void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_accum || (last && !d_out)) {
        set_error("null camera or buffer");
        return SRT_ERR_INVALID_ARG;
    }
    if (p->rng == SRT_RNG_TRIG64) {
        set_error("the fused pass draws the counter stream; use the trace/shade entry points for trig64");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return launch_render_pass_fused(s, make_cam(camera), make_render_args(p), pass, (float4 *)d_accum, first != 0,
                                    last != 0, (float4 *)d_out, (cudaStream_t)stream);
}

srt_status srt_render_pass_frame_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p,
                                        int32_t pass, float *d_accum, int32_t first, int32_t last, float *d_frame,
                                        int32_t peer, void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_accum || (last && !d_frame)) {
        set_error("null camera or buffer");
        return SRT_ERR_INVALID_ARG;
    }
    if (p->rng == SRT_RNG_TRIG64) {
        set_error("the fused pass draws the counter stream");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    return launch_render_pass_fused(s, make_cam(camera), make_render_args(p), pass, (float4 *)d_accum, first != 0,
                                    last != 0, (float4 *)d_frame, (cudaStream_t)stream, nullptr, nullptr, nullptr,
                                    true, peer != 0);
}

srt_status srt_ipc_alloc(int32_t device, int64_t bytes, void **d_ptr, uint8_t *handle) {
    if (!d_ptr || !handle || bytes <= 0) {
        set_error("invalid IPC allocation");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(device);
    *d_ptr = nullptr;
    srt_status rc = cuda_status(cudaMalloc(d_ptr, (size_t)bytes), "IPC buffer");
    cudaIpcMemHandle_t h;
    if (!rc) rc = cuda_status(cudaIpcGetMemHandle(&h, *d_ptr), "cudaIpcGetMemHandle");
    if (rc) {
        if (*d_ptr) cudaFree(*d_ptr);
        *d_ptr = nullptr;
        return rc;
    }
    std::memcpy(handle, &h, sizeof(h));
    return SRT_OK;
}

srt_status srt_ipc_open(int32_t device, const uint8_t *handle, void **d_ptr) {
    if (!d_ptr || !handle) {
        set_error("invalid IPC handle");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    *d_ptr = nullptr;
    return cuda_status(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

srt_status srt_ipc_close(int32_t device, void *d_ptr) {
    if (!d_ptr) return SRT_OK;
    DeviceGuard g(device);
    return cuda_status(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
}

srt_status srt_ipc_free(int32_t device, void *d_ptr) {
    if (!d_ptr) return SRT_OK;
    DeviceGuard g(device);
    return cuda_status(cudaFree(d_ptr), "cudaFree");
}

srt_status srt_render_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p, int32_t *d_hits,
                             float *d_accum, float *d_out, void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_hits || !d_accum || !d_out) {
        set_error("null camera or buffer");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    CamD cam = make_cam(camera);
    RenderArgs a = make_render_args(p);
    cudaStream_t st = (cudaStream_t)stream;
    for (int f = 0; f < p->passes && !rc; ++f) {
        int pass = p->pass0 + f;
        if (a.rng == SRT_RNG_TRIG64) {
            rc = launch_trace_pass(s, cam, a, pass, d_hits, st);
            if (!rc)
                rc = launch_shade_pass(s, cam, a, pass, d_hits, (float4 *)d_accum, f == 0, f == p->passes - 1,
                                       (float4 *)d_out, st);
        } else {
            rc = launch_render_pass_fused(s, cam, a, pass, (float4 *)d_accum, f == 0, f == p->passes - 1,
                                          (float4 *)d_out, st);
        }
    }
    return rc;
}

srt_status srt_render_frame_device(const SrtScene *s, const SrtCamera *camera, const SrtRenderParams *p,
                                   uint64_t *d_acc, float *d_out, void *stream) {
    srt_status rc = validate_render(s, p);
    if (rc) return rc;
    if (!camera || !d_acc) {
        set_error("null camera or buffer");
        return SRT_ERR_INVALID_ARG;
    }
    if (p->rng == SRT_RNG_TRIG64) {
        set_error("the one-launch frame draws the counter stream; use srt_render_device for trig64");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    RenderArgs a = make_render_args(p);
    cudaStream_t st = (cudaStream_t)stream;
    rc = cuda_status(cudaMemsetAsync(d_acc, 0, sizeof(uint64_t) * 4 * a.local_tiles * 256, st), "accumulator reset");
    if (!rc)
        rc = launch_render_frame_multipass(s, make_cam(camera), a, p->pass0, p->passes,
                                           (unsigned long long *)d_acc, st);
    if (!rc && d_out)
        rc = launch_resolve_fixed(a, (unsigned long long *)d_acc, p->passes, (float4 *)d_out, nullptr, nullptr, st);
    return rc;
}

srt_status srt_resolve_frame_device(const SrtRenderParams *p, const uint64_t *d_acc, double *d_rgb, double *d_op,
                                    void *stream) {
    if (!p || !d_acc || !d_rgb || !d_op || p->width < 1 || p->height < 1 || p->passes < 1 || p->nslots < 1 ||
        p->shard_count < 0 || (p->shard_count > 0 && (p->shard_index < 0 || p->shard_index >= p->shard_count))) {
        set_error("invalid resolve parameters");
        return SRT_ERR_INVALID_ARG;
    }
    RenderArgs a = make_render_args(p);
    return launch_resolve_fixed(a, (const unsigned long long *)d_acc, p->passes, nullptr, d_rgb, d_op,
                                (cudaStream_t)stream);
}

srt_status srt_render(const SrtScene *sc, const SrtCamera *camera, const SrtRenderParams *p, double *out_rgb,
                      double *out_op, int64_t *out_ids) {
    SRT_LOCK(sc);
    srt_status rc = validate_render(sc, p);
    if (rc) return rc;
    if (!camera || !out_rgb || !out_op) {
        set_error("null camera or output");
        return SRT_ERR_INVALID_ARG;
    }
    // A tile shard (shard_count > 1) writes only its own pixels, straight into
    // mapped host outputs shared by every shard (multi-GPU frames assembled in
    // one host buffer, each GPU over its own PCIe link).
    if (p->shard_count > 1 && (!mapped_host(out_rgb) || !mapped_host(out_op) || out_ids || p->rng == SRT_RNG_TRIG64)) {
        set_error("a shard of srt_render needs mapped host outputs (srt_host_alloc / srt_host_register), "
                  "the counter stream and no ids");
        return SRT_ERR_INVALID_ARG;
    }
    SrtScene *s = const_cast<SrtScene *>(sc);
    DeviceGuard g(s->device);
    cudaStream_t st = s->stream;
    if (srt_status frc = clear_flag(s, st)) return frc;  // errors belong to this call
    RenderArgs a = make_render_args(p);
    CamD cam = make_cam(camera);
    const int64_t npix = (int64_t)p->width * p->height;
    const int64_t cpix = a.local_tiles * 256;  // tile-compact pixel count
    size_t hits_bytes = sizeof(int32_t) * cpix * p->nslots;
    size_t acc_bytes = sizeof(float4) * cpix;
    size_t out_bytes = sizeof(float4) * npix;
    size_t f64_bytes = sizeof(double) * npix * 4;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    rc = scratch_reserve(s, al(hits_bytes) + al(acc_bytes) + al(out_bytes) + al(f64_bytes));
    if (rc) return rc;
    char *base = (char *)s->d_scratch;
    int32_t *d_hits = (int32_t *)base;
    float4 *d_acc = (float4 *)(base + al(hits_bytes));
    float4 *d_out = (float4 *)(base + al(hits_bytes) + al(acc_bytes));
    double *d_rgb = (double *)(base + al(hits_bytes) + al(acc_bytes) + al(out_bytes));
    double *d_op = d_rgb + npix * 3;
    // Several counter-stream passes: one balanced launch over every (packet,
    // pass), fixed-point sums, one resolve straight into the f64 outputs.
    if (p->passes > 1 && a.rng != SRT_RNG_TRIG64 && !out_ids) {
        size_t acc_bytes64 = sizeof(unsigned long long) * 4 * cpix;
        rc = scratch_reserve(s, al(acc_bytes64) + al(f64_bytes));
        if (rc) return rc;
        unsigned long long *d_acc64 = (unsigned long long *)s->d_scratch;
        double *f_rgb = (double *)((char *)s->d_scratch + al(acc_bytes64));
        double *f_op = f_rgb + npix * 3;
        double *m_rgb = mapped_host(out_rgb), *m_op = mapped_host(out_op);
        bool direct = m_rgb && m_op;
        rc = cuda_status(cudaMemsetAsync(d_acc64, 0, acc_bytes64, st), "accumulator reset");
        if (!rc) rc = launch_render_frame_multipass(s, cam, a, p->pass0, p->passes, d_acc64, st);
        if (!rc)
            rc = launch_resolve_fixed(a, d_acc64, p->passes, nullptr, direct ? m_rgb : f_rgb, direct ? m_op : f_op,
                                      st);
        if (!rc && !direct) {
            rc = copy_d2h(s, out_rgb, f_rgb, sizeof(double) * npix * 3, st);
            if (!rc)
                rc = copy_d2h(s, out_op, f_op, sizeof(double) * npix, st);
        }
        if (!rc) rc = check_flag(s, st);
        return rc;
    }
    // Outputs in mapped page-locked memory (srt_host_alloc): the last fused
    // pass stores the f64 frame straight into them, so the device->host
    // transfer overlaps the walk and no resolve kernel or copy follows.
    double *m_rgb = mapped_host(out_rgb), *m_op = mapped_host(out_op);
    const bool direct = m_rgb && m_op && a.rng != SRT_RNG_TRIG64 && !(out_ids && p->passes == 1);
    for (int f = 0; f < p->passes && !rc; ++f) {
        int pass = p->pass0 + f;
        if (a.rng != SRT_RNG_TRIG64 && !(out_ids && f == 0)) {
            const bool last = f == p->passes - 1;
            rc = launch_render_pass_fused(s, cam, a, pass, d_acc, f == 0, last, d_out, st, nullptr,
                                          last && direct ? m_rgb : nullptr, last && direct ? m_op : nullptr);
            continue;
        }
        rc = launch_trace_pass(s, cam, a, pass, d_hits, st);
        if (!rc && out_ids && f == 0) {
            // slot ids of the first pass, un-tiled on the host
            std::vector<int32_t> hh((size_t)cpix * p->nslots);
            rc = cuda_status(cudaMemcpyAsync(hh.data(), d_hits, hits_bytes, cudaMemcpyDeviceToHost, st), "ids");
            if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "ids");
            if (!rc) {
                int tiles_x = a.tiles_x;
                for (int64_t lt = 0; lt < a.local_tiles; ++lt)
                    for (int tid = 0; tid < 256; ++tid) {
                        int tx = (int)(lt % tiles_x), ty = (int)(lt / tiles_x);
                        int w = tid >> 5, lane = tid & 31;
                        int px = tx * 16 + (w & 1) * 8 + (lane & 7);
                        int py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
                        if (px >= p->width || py >= p->height) continue;
                        for (int k = 0; k < p->nslots; ++k)
                            out_ids[((int64_t)py * p->width + px) * p->nslots + k] = hh[(lt * 256 + tid) * p->nslots + k];
                    }
            }
        }
        if (!rc) rc = launch_shade_pass(s, cam, a, pass, d_hits, d_acc, f == 0, f == p->passes - 1, d_out, st);
    }
    if (direct) {
        if (!rc) rc = check_flag(s, st);
        return rc;
    }
    if (!rc) rc = launch_resolve_f64(a, d_out, d_rgb, d_op, st);
    if (!rc) rc = copy_d2h(s, out_rgb, d_rgb, sizeof(double) * npix * 3, st);
    if (!rc) rc = copy_d2h(s, out_op, d_op, sizeof(double) * npix, st);
    if (!rc) rc = check_flag(s, st);
    return rc;
}

srt_status srt_scene_check(const SrtScene *s, int32_t reset) {
    if (!s) {
        set_error("null scene");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    srt_status rc = cuda_status(cudaDeviceSynchronize(), "sync");
    if (rc) return rc;
    if (!*(volatile int32_t *)s->h_flag) return SRT_OK;
    if (reset) *(volatile int32_t *)s->h_flag = 0;
    set_error("traversal stack overflow (BVH deeper than the 128-entry stack)");
    return SRT_ERR_STACK_OVERFLOW;
}

srt_status srt_trace_counters(const SrtScene *s, uint64_t *out, int32_t n, int32_t reset) {
    if (!s || !out || n < 1 || n > 16) {
        set_error("null scene or output, or n outside 1..16");
        return SRT_ERR_INVALID_ARG;
    }
    DeviceGuard g(s->device);
    srt_status rc = cuda_status(cudaDeviceSynchronize(), "sync");
    if (!rc) rc = cuda_status(cudaMemcpy(out, s->d_stats, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost), "stats");
    if (!rc && reset) rc = cuda_status(cudaMemset(s->d_stats, 0, sizeof(uint64_t) * 16), "stats reset");
    return rc;
}

srt_status srt_trace_stats(const SrtScene *s, uint64_t *out, int32_t reset) {
    return srt_trace_counters(s, out, 8, reset);
}

srt_status srt_unpack_tiles_device(const float *d_gathered, int32_t width, int32_t height, int32_t shard_count,
                                   int64_t max_tiles, float *d_frame, void *stream) {
    if (!d_gathered || !d_frame || width < 1 || height < 1 || shard_count < 1 || max_tiles < 0) {
        set_error("invalid unpack arguments");
        return SRT_ERR_INVALID_ARG;
    }
    return launch_unpack((const float4 *)d_gathered, width, height, shard_count, max_tiles, (float4 *)d_frame,
                         (cudaStream_t)stream);
}

}  // extern "C"
