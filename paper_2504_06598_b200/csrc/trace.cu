// trace.cu -- stochastic BVH walk (kernels.py:312-388) for camera rays and
// explicit rays, plus the unclipped transmittance walk (kernels.py:392-432).
//
// One thread per ray.  Camera rays are mapped 8x4 pixels per warp inside
// 16x16 tiles so a warp's rays are coherent and share node fetches.  Each
// visit reads one 64-B Node2 (both children's boxes), tests both boxes,
// resolves leaf children (single primitives) on the spot and descends into
// the nearer inner child, pushing the farther one with its entry distance.
#include <cfloat>

#include "srt_internal.h"

namespace srt {

template <int NS>
struct Slots {
    float t[NS];
    int id[NS];
    uint32_t key[NS];
};

// Acceptance draw of slot k for primitive `pid` (kernels.py:354 with the
// counter generator; RNG==SRT_RNG_TABLE reads an explicit uniform).
template <int RNG>
__device__ __forceinline__ bool accepts(uint32_t key, const double *table, int64_t tstride, int pid, int k,
                                        float alpha) {
    if (RNG == SRT_RNG_TABLE) return __ldg(table + (int64_t)pid * tstride + k) < (double)alpha;
    return counter_u(key, (uint32_t)pid) < alpha;
}

template <int NS, int MODE, int RNG>
__device__ __forceinline__ void visit_leaf(const SceneView &s, const RayState &r, float s2, int clip, int slot,
                                           Slots<NS> &sl, float &far, const double *table, int64_t tstride) {
    const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
    float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
    Cand c = candidate<MODE>(r, m, a, b, s2);
    if (!c.valid) return;
    int pid = __float_as_int(b.z);
    bool improved = false;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        // strict t < slot_t (kernels.py:354); an exact tie goes to the
        // smaller primitive id so the result is visit-order independent
        bool nearer = c.t < sl.t[k] || (c.t == sl.t[k] && pid < sl.id[k]);
        if (nearer && accepts<RNG>(sl.key[k], table, tstride, pid, k, c.alpha)) {
            sl.t[k] = c.t;
            sl.id[k] = pid;
            improved = true;
        }
    }
    if (improved && clip) {
        // clip to the farthest slot once every slot holds a hit (kernels.py:358-364);
        // inactive slots hold -inf and never bind
        float worst = sl.t[0];
#pragma unroll
        for (int k = 1; k < NS; ++k) worst = fmaxf(worst, sl.t[k]);
        far = fminf(far, worst);
    }
}

template <int NS, int MODE, int RNG>
__device__ __forceinline__ void walk(const SceneView &s, const RayState &r, float s2, int clip, Slots<NS> &sl,
                                     const double *table, int64_t tstride, int *overflow) {
    if (s.num_nodes == 0) return;
    float far = r.t_max0;
    int stk_node[kStackSize];
    float stk_t[kStackSize];
    int sp = 0;
    int cur = 0;
    while (true) {
        const float4 *np = reinterpret_cast<const float4 *>(s.nodes + cur);
        float4 xy0 = __ldg(np), xy1 = __ldg(np + 1), z01 = __ldg(np + 2);
        int4 kids = __ldg(reinterpret_cast<const int4 *>(np + 3));
        float e0, e1;
        bool h0, h1;
        slab2(r, xy0, xy1, z01, far, e0, e1, h0, h1);
        int c0 = kids.x, c1 = kids.y;
        if (e1 < e0) {  // near child first
            int ti = c0; c0 = c1; c1 = ti;
            float tf = e0; e0 = e1; e1 = tf;
            bool tb = h0; h0 = h1; h1 = tb;
        }
        if (h0 && c0 < 0) {
            if (c0 != kLeafEmpty) visit_leaf<NS, MODE, RNG>(s, r, s2, clip, ~c0, sl, far, table, tstride);
            h0 = false;
        }
        if (h1 && c1 < 0) {
            if (c1 != kLeafEmpty && e1 <= far) visit_leaf<NS, MODE, RNG>(s, r, s2, clip, ~c1, sl, far, table, tstride);
            h1 = false;
        }
        h0 = h0 && e0 <= far;
        h1 = h1 && e1 <= far;
        if (h0) {
            if (h1) {
                if (sp >= kStackSize) {
                    atomicExch(overflow, 1);
                    return;
                }
                stk_node[sp] = c1;
                stk_t[sp] = e1;
                ++sp;
            }
            cur = c0;
            continue;
        }
        if (h1) {
            cur = c1;
            continue;
        }
        // pop, culling entries beyond the (possibly clipped) far bound
        bool found = false;
        while (sp > 0) {
            --sp;
            if (stk_t[sp] <= far) {
                cur = stk_node[sp];
                found = true;
                break;
            }
        }
        if (!found) return;
    }
}

template <int NS>
__device__ __forceinline__ void init_slots(Slots<NS> &sl, int nslots) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        sl.t[k] = k < nslots ? INFINITY : -INFINITY;  // inactive slots never accept, never bind the clip
        sl.id[k] = -1;
        sl.key[k] = 0;
    }
}

// ---------------------------------------------------------------------------
// camera rays: one pass of render_stochastic (kernels.py:644-656)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_pixel(const RenderArgs &a, int64_t lt, int tid, int &px, int &py) {
    int64_t gt = lt * a.shard_count + a.shard_index;
    int tx = (int)(gt % a.tiles_x), ty = (int)(gt / a.tiles_x);
    int w = tid >> 5, lane = tid & 31;
    px = tx * 16 + (w & 1) * 8 + (lane & 7);
    py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
}

template <int NS, int MODE>
__global__ void __launch_bounds__(256) k_trace_pass(SceneView s, CamD cam, RenderArgs a, int pass, int32_t *hits,
                                                    int *overflow) {
    int64_t lt = blockIdx.x;
    int px, py;
    tile_pixel(a, lt, threadIdx.x, px, py);
    int64_t slot_base = (lt * 256 + threadIdx.x) * a.nslots;
    if (px >= a.width || py >= a.height) return;
    double dx, dy, dz;
    camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)pass, a.seed, a.width, a.height, dx, dy, dz);
    RayState r;
    init_ray(r, cam.e[0], cam.e[1], cam.e[2], dx, dy, dz, 0.0, DBL_MAX);
    Slots<NS> sl;
    init_slots<NS>(sl, a.nslots);
    uint32_t fk = frame_key(a.seed);
    uint32_t ray_id = (uint32_t)py * (uint32_t)a.width + (uint32_t)px;
#pragma unroll
    for (int k = 0; k < NS; ++k) sl.key[k] = walk_key(fk, ray_id, (uint32_t)pass * (uint32_t)a.nslots + k);
    walk<NS, MODE, SRT_RNG_COUNTER>(s, r, a.s2, a.clip, sl, nullptr, 0, overflow);
#pragma unroll
    for (int k = 0; k < NS; ++k)
        if (k < a.nslots) hits[slot_base + k] = sl.id[k];
}

template <int NS, int MODE>
static void launch_trace_pass_t(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, int32_t *d_hits,
                                cudaStream_t st) {
    if (a.local_tiles <= 0) return;
    k_trace_pass<NS, MODE><<<(unsigned)a.local_tiles, 256, 0, st>>>(s->view(), cam, a, pass, d_hits, s->d_flag);
}

srt_status launch_trace_pass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, int32_t *d_hits,
                             cudaStream_t st) {
#define SRT_DISPATCH_MODE(NS)                                               \
    if (a.mode == 0)                                                        \
        launch_trace_pass_t<NS, 0>(s, cam, a, pass, d_hits, st);            \
    else                                                                    \
        launch_trace_pass_t<NS, 1>(s, cam, a, pass, d_hits, st);
    if (a.nslots <= 1) {
        SRT_DISPATCH_MODE(1)
    } else if (a.nslots <= 2) {
        SRT_DISPATCH_MODE(2)
    } else if (a.nslots <= 4) {
        SRT_DISPATCH_MODE(4)
    } else if (a.nslots <= 8) {
        SRT_DISPATCH_MODE(8)
    } else if (a.nslots <= 16) {
        SRT_DISPATCH_MODE(16)
    } else {
        set_error("nslots > 16 is not supported by the GPU tracer yet");
        return SRT_ERR_UNSUPPORTED;
    }
#undef SRT_DISPATCH_MODE
    return cuda_status(cudaGetLastError(), "k_trace_pass launch");
}

// ---------------------------------------------------------------------------
// explicit rays (kernels.trace_batch, kernels.py:527-540)
// ---------------------------------------------------------------------------
struct TraceArgs {
    double t_min, t_max;
    float s2;
    int clip, nslots;
    uint32_t seed, ray_id0, sample0;
    int64_t tstride;
};

template <int NS, int MODE, int RNG>
__global__ void __launch_bounds__(128) k_trace_rays(SceneView s, TraceArgs a, const double *__restrict__ rays,
                                                    int64_t R, const double *table, float *out_t, int32_t *out_id,
                                                    int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double *q = rays + i * 6;
    RayState r;
    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], a.t_min, a.t_max);
    Slots<NS> sl;
    init_slots<NS>(sl, a.nslots);
    uint32_t fk = frame_key(a.seed);
#pragma unroll
    for (int k = 0; k < NS; ++k) sl.key[k] = walk_key(fk, a.ray_id0 + (uint32_t)i, a.sample0 + (uint32_t)k);
    walk<NS, MODE, RNG>(s, r, a.s2, a.clip, sl, table, a.tstride, overflow);
#pragma unroll
    for (int k = 0; k < NS; ++k)
        if (k < a.nslots) {
            out_t[i * a.nslots + k] = sl.id[k] >= 0 ? sl.t[k] : INFINITY;
            out_id[i * a.nslots + k] = sl.id[k];
        }
}

template <int NS>
static void launch_rays_t(const SrtScene *s, const TraceArgs &ta, int mode, int rng, const double *d_rays, int64_t R,
                          const double *d_table, float *d_t, int32_t *d_id, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return;
    SceneView v = s->view();
    if (rng == SRT_RNG_TABLE) {
        if (mode == 0)
            k_trace_rays<NS, 0, SRT_RNG_TABLE><<<blocks, 128, 0, st>>>(v, ta, d_rays, R, d_table, d_t, d_id, s->d_flag);
        else
            k_trace_rays<NS, 1, SRT_RNG_TABLE><<<blocks, 128, 0, st>>>(v, ta, d_rays, R, d_table, d_t, d_id, s->d_flag);
    } else {
        if (mode == 0)
            k_trace_rays<NS, 0, SRT_RNG_COUNTER><<<blocks, 128, 0, st>>>(v, ta, d_rays, R, d_table, d_t, d_id, s->d_flag);
        else
            k_trace_rays<NS, 1, SRT_RNG_COUNTER><<<blocks, 128, 0, st>>>(v, ta, d_rays, R, d_table, d_t, d_id, s->d_flag);
    }
}

srt_status launch_trace_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R, int nslots,
                             const double *d_table, float *d_t, int32_t *d_id, cudaStream_t st) {
    TraceArgs ta;
    ta.t_min = p->t_min;
    ta.t_max = p->t_max;
    ta.s2 = (float)p->s2;
    ta.clip = p->clip;
    ta.nslots = nslots;
    ta.seed = p->seed;
    ta.ray_id0 = p->ray_id0;
    ta.sample0 = p->sample0;
    ta.tstride = p->table_slots;
    if (nslots <= 1)
        launch_rays_t<1>(s, ta, p->mode, p->rng, d_rays, R, d_table, d_t, d_id, st);
    else if (nslots <= 2)
        launch_rays_t<2>(s, ta, p->mode, p->rng, d_rays, R, d_table, d_t, d_id, st);
    else if (nslots <= 4)
        launch_rays_t<4>(s, ta, p->mode, p->rng, d_rays, R, d_table, d_t, d_id, st);
    else if (nslots <= 8)
        launch_rays_t<8>(s, ta, p->mode, p->rng, d_rays, R, d_table, d_t, d_id, st);
    else if (nslots <= 16)
        launch_rays_t<16>(s, ta, p->mode, p->rng, d_rays, R, d_table, d_t, d_id, st);
    else {
        set_error("nslots > 16 is not supported by the GPU tracer yet");
        return SRT_ERR_UNSUPPORTED;
    }
    return cuda_status(cudaGetLastError(), "k_trace_rays launch");
}

// ---------------------------------------------------------------------------
// transmittance: prod(1 - alpha) over every valid candidate, no clipping
// (kernels.py:392-432).  Order of the product differs from the reference's
// walk; the value agrees to product-reordering roundoff.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(128) k_transmittance(SceneView s, const double *__restrict__ rays, int64_t R,
                                                       double t_min, double t_max, float s2, double *out,
                                                       int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double *q = rays + i * 6;
    RayState r;
    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
    double result = 1.0;
    if (s.num_nodes > 0) {
        int stk[kStackSize];
        int sp = 0, cur = 0;
        while (true) {
            const float4 *np = reinterpret_cast<const float4 *>(s.nodes + cur);
            float4 xy0 = __ldg(np), xy1 = __ldg(np + 1), z01 = __ldg(np + 2);
            int4 kids = __ldg(reinterpret_cast<const int4 *>(np + 3));
            float e0, e1;
            bool h0, h1;
            slab2(r, xy0, xy1, z01, r.t_max0, e0, e1, h0, h1);
            int cs[2] = {kids.x, kids.y};
            bool hs[2] = {h0, h1};
            int next = -1;
            for (int c = 0; c < 2; ++c) {
                if (!hs[c]) continue;
                if (cs[c] < 0) {
                    if (cs[c] == kLeafEmpty) continue;
                    const float4 *g = reinterpret_cast<const float4 *>(s.geom + ~cs[c]);
                    float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
                    Cand cd = candidate<MODE>(r, m, a, b, s2);
                    if (cd.valid) result *= 1.0 - (double)cd.alpha;
                } else if (next < 0) {
                    next = cs[c];
                } else {
                    if (sp >= kStackSize) {
                        atomicExch(overflow, 1);
                        out[i] = result;
                        return;
                    }
                    stk[sp++] = cs[c];
                }
            }
            if (next >= 0) {
                cur = next;
                continue;
            }
            if (sp == 0) break;
            cur = stk[--sp];
        }
    }
    out[i] = result;
}

srt_status launch_transmittance(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max,
                                int mode, double s2, double *d_out, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    if (mode == 0)
        k_transmittance<0><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, d_out, s->d_flag);
    else
        k_transmittance<1><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, d_out, s->d_flag);
    return cuda_status(cudaGetLastError(), "k_transmittance launch");
}

}  // namespace srt
