// trig64.cu -- "trig64 bridge" mode: the walk with
// the reference's OWN acceptance draw, the trig hash of the fp64 hit position
// (kernels.py:47-60), so GPU output can be compared directly with the
// unmodified reference.  The candidate (kernels.py:139-189) is evaluated in
// fp64 from the scene's fp64 records with explicitly rounded operations in the
// reference's expression order (no FMA contraction), so hit positions -- and
// with them the hash inputs -- are bitwise the reference's.  The remaining
// differences are the device libm: sin/exp/floor here vs glibc on the CPU (a
// 1-ulp sin difference moves the draw by ~1e-5, so ids flip only at
// |u - alpha| < 1e-5 ties).  Traversal reuses the fp32 4-wide tree with
// conservative boxes; slots and the far bound are fp64.
//
// This is a parity mode, not a throughput path: one ray per thread.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "srt_internal.h"
#include "srt_trig64.cuh"

namespace srt {

namespace t64 {

__device__ __forceinline__ float far32(double far) {
    if (far >= 3.0e38) return INFINITY;
    return __double2float_ru(far) * 1.0000002f + 1e-30f;  // conservative
}

// One walk (kernels.py:312-388) with fp64 slots.
// Slot j of the walk is slot slot0 + j of the ray (slot groups of <= 16 for
// multisample N > 16): its draw hashes with slot index slot0 + j.
template <int NS, int MODE>
__device__ void walk(const SceneView &s, const Ray64 &r, double s2, int clip, int nslots, int slot0, double *slot_t,
                     int *slot_id, int *overflow) {
    for (int k = 0; k < NS; ++k) {
        slot_t[k] = k < nslots ? INFINITY : -INFINITY;
        slot_id[k] = -1;
    }
    if (s.num_nodes4 == 0) return;
    RayState rs;
    init_ray(rs, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, r.t_min, r.t_max);
    rs.t_min = __double2float_rd(r.t_min);
    double far = r.t_max;
    int stk[kStackSize];
    int sp = 0;
    int node = 0;
    while (node >= 0) {
        SRT_DCHECK(node >= 0 && node < s.num_nodes4);
        const float4 *np = reinterpret_cast<const float4 *>(s.nodes4 + node);
        float4 lox = __ldg(np), hix = __ldg(np + 1), loy = __ldg(np + 2), hiy = __ldg(np + 3),
               loz = __ldg(np + 4), hiz = __ldg(np + 5);
        int4 kids = __ldg(reinterpret_cast<const int4 *>(np + 6));
        float lx[4] = {lox.x, lox.y, lox.z, lox.w}, hx4[4] = {hix.x, hix.y, hix.z, hix.w};
        float ly[4] = {loy.x, loy.y, loy.z, loy.w}, hy4[4] = {hiy.x, hiy.y, hiy.z, hiy.w};
        float lz[4] = {loz.x, loz.y, loz.z, loz.w}, hz4[4] = {hiz.x, hiz.y, hiz.z, hiz.w};
        int kid[4] = {kids.x, kids.y, kids.z, kids.w};
        node = -1;
        for (int k = 0; k < 4; ++k) {
            if (kid[k] == kLeafEmpty) continue;
            float f = far32(far);
            float xa = fmaf(lx[k], rs.idx, -rs.oidx), xb = fmaf(hx4[k], rs.idx, -rs.oidx);
            float ya = fmaf(ly[k], rs.idy, -rs.oidy), yb = fmaf(hy4[k], rs.idy, -rs.oidy);
            float za = fmaf(lz[k], rs.idz, -rs.oidz), zb = fmaf(hz4[k], rs.idz, -rs.oidz);
            float tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fmaxf(fminf(za, zb), rs.t_min));
            float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), f));
            if (!(tn <= tf)) continue;
            if (kid[k] >= 0) {
                if (sp >= kStackSize) {
                    raise_flag(overflow);
                    return;
                }
                stk[sp++] = kid[k];
                continue;
            }
            int slot = ~kid[k];
            SRT_DCHECK(slot < s.n);
            int pid = __float_as_int(s.geom[slot].b.z);
            double t, resid, px, py, pz;
            if (!candidate<MODE>(r, s.means64 + (int64_t)pid * 3, s.cov64 + (int64_t)pid * 6, s2, t, resid, px, py,
                                 pz))
                continue;
            if (t <= r.t_min || t >= r.t_max) continue;
            double alpha = mul(s.opac64[pid], exp(mul(-0.5, resid)));
            bool improved = false;
            for (int j = 0; j < NS; ++j) {
                bool nearer = t < slot_t[j] || (t == slot_t[j] && pid < slot_id[j]);
                if (nearer && hash_position(px, py, pz, slot0 + j) < alpha) {
                    slot_t[j] = t;
                    slot_id[j] = pid;
                    improved = true;
                }
            }
            if (improved && clip) {
                double worst = slot_t[0];
                for (int j = 1; j < NS; ++j) worst = fmax(worst, slot_t[j]);
                if (worst < far) far = worst;
            }
        }
        if (sp > 0) node = stk[--sp];
    }
}

}  // namespace t64

template <int NS, int MODE>
__global__ void __launch_bounds__(128) k_trace_rays_trig64(SceneView s, const double *__restrict__ rays, int64_t R,
                                                           double t_min, double t_max, double s2, int clip,
                                                           int nslots, int slot0, int ostride, double *out_t,
                                                           int32_t *out_id, int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double *q = rays + i * 6;
    t64::Ray64 r{q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max};
    double st[NS];
    int sid[NS];
    t64::walk<NS, MODE>(s, r, s2, clip, nslots, slot0, st, sid, overflow);
    for (int k = 0; k < nslots && k < NS; ++k) {
        out_t[i * ostride + slot0 + k] = sid[k] >= 0 ? st[k] : INFINITY;
        out_id[i * ostride + slot0 + k] = sid[k];
    }
}

template <int NS, int MODE>
__global__ void __launch_bounds__(128) k_trace_pass_trig64(SceneView s, CamD cam, RenderArgs a, int pass,
                                                           double s2, int slot0, int gslots, int32_t *hits,
                                                           int *overflow) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= a.local_tiles * 256) return;
    int64_t lt = idx >> 8;
    int tid = (int)(idx & 255);
    int64_t gt = lt * a.shard_count + a.shard_index;
    int tx = (int)(gt % a.tiles_x), ty = (int)(gt / a.tiles_x);
    int w = tid >> 5, lane = tid & 31;
    int px = tx * 16 + (w & 1) * 8 + (lane & 7);
    int py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
    if (px >= a.width || py >= a.height) return;
    double dx, dy, dz;
    camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)pass, a.seed, a.width, a.height, dx, dy, dz);
    t64::Ray64 r{cam.e[0], cam.e[1], cam.e[2], dx, dy, dz, 0.0, DBL_MAX};
    double st[NS];
    int sid[NS];
    t64::walk<NS, MODE>(s, r, s2, a.clip, gslots, slot0, st, sid, overflow);
    for (int k = 0; k < gslots && k < NS; ++k) hits[idx * a.nslots + slot0 + k] = sid[k];
}

#define SRT_T64_NS(MACRO) \
    if (nslots <= 1) {    \
        MACRO(1)          \
    } else if (nslots <= 2) { \
        MACRO(2)          \
    } else if (nslots <= 4) { \
        MACRO(4)          \
    } else if (nslots <= 8) { \
        MACRO(8)          \
    } else {              \
        MACRO(16)         \
    }

srt_status launch_trace_rays_trig64(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R,
                                    int nslots, double *d_t, int32_t *d_id, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    SceneView v = s->walk_view();
    const int all = nslots;
    // slot groups of <= 16 (slots are independent; each group hashes its own slot indices)
    for (int g0 = 0; g0 < all; g0 += 16) {
        const int nslots = std::min(16, all - g0);
#define SRT_L(NS)                                                                                             \
    if (p->mode == 0)                                                                                         \
        k_trace_rays_trig64<NS, 0><<<blocks, 128, 0, st>>>(v, d_rays, R, p->t_min, p->t_max, p->s2, p->clip,  \
                                                           nslots, g0, all, d_t, d_id, s->d_flag);            \
    else                                                                                                      \
        k_trace_rays_trig64<NS, 1><<<blocks, 128, 0, st>>>(v, d_rays, R, p->t_min, p->t_max, p->s2, p->clip,  \
                                                           nslots, g0, all, d_t, d_id, s->d_flag);
        SRT_T64_NS(SRT_L)
#undef SRT_L
        srt_status rc = cuda_status(cudaGetLastError(), "k_trace_rays_trig64 launch");
        if (rc) return rc;
    }
    return SRT_OK;
}

srt_status launch_trace_pass_trig64(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, double s2,
                                    int32_t *d_hits, cudaStream_t st) {
    int64_t n = a.local_tiles * 256;
    unsigned blocks = (unsigned)((n + 127) / 128);
    if (blocks == 0) return SRT_OK;
    SceneView v = s->walk_view();
    for (int g0 = 0; g0 < a.nslots; g0 += 16) {
        const int nslots = std::min(16, a.nslots - g0);
#define SRT_L(NS)                                                                                             \
    if (a.mode == 0)                                                                                          \
        k_trace_pass_trig64<NS, 0><<<blocks, 128, 0, st>>>(v, cam, a, pass, s2, g0, nslots, d_hits, s->d_flag); \
    else                                                                                                      \
        k_trace_pass_trig64<NS, 1><<<blocks, 128, 0, st>>>(v, cam, a, pass, s2, g0, nslots, d_hits, s->d_flag);
        SRT_T64_NS(SRT_L)
#undef SRT_L
        srt_status rc = cuda_status(cudaGetLastError(), "k_trace_pass_trig64 launch");
        if (rc) return rc;
    }
    return SRT_OK;
}

}  // namespace srt
