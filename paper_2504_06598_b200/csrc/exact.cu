// exact.cu -- exact sorted compositing: the RNG-free
// converged reference of the estimator, `render(..., reference_mode=True)`.
//
// The reference brute-forces every primitive per ray (kernels.py:441-475).
// Here each ray walks the BVH WITHOUT clipping, collecting every valid
// candidate (the same set: a valid candidate lies inside its ellipsoid, hence
// inside its conservative box), sorts them by (t, prim id) -- the stable
// order of np.argsort(kind="mergesort") over ids appended in increasing order
// -- and composites front to back in fp64: L = sum T_i a_i c_i + T bg.
// Candidates are taken kExactChunk at a time in (t, id) order (NearestK), one
// unclipped walk per chunk, so rays through thousands of candidates need no
// per-ray buffer beyond the chunk.
#include <cfloat>
#include <climits>

#include "srt_internal.h"
#include "srt_trig64.cuh"

namespace srt {

// Every leaf primitive whose conservative box the ray crosses inside
// [t_min, t_max0], in no particular order: visit(slot, gm, ga, gb).
template <class Visit>
__device__ __forceinline__ void for_each_leaf(const SceneView &s, const RayState &r, int *overflow, Visit &&visit,
                                              const float *far = nullptr, float lo = -INFINITY) {
    if (s.num_nodes4 == 0) return;
    int stk[kStackSize];
    int sp = 0, node = 0;
    while (node >= 0) {
        SRT_DCHECK(node >= 0 && node < s.num_nodes4);
        const float4 *np = reinterpret_cast<const float4 *>(s.nodes4 + node);
        float4 lox = __ldg(np), hix = __ldg(np + 1), loy = __ldg(np + 2), hiy = __ldg(np + 3), loz = __ldg(np + 4),
               hiz = __ldg(np + 5);
        int4 kids = __ldg(reinterpret_cast<const int4 *>(np + 6));
        float lx[4] = {lox.x, lox.y, lox.z, lox.w}, hx[4] = {hix.x, hix.y, hix.z, hix.w};
        float ly[4] = {loy.x, loy.y, loy.z, loy.w}, hy[4] = {hiy.x, hiy.y, hiy.z, hiy.w};
        float lz[4] = {loz.x, loz.y, loz.z, loz.w}, hz[4] = {hiz.x, hiz.y, hiz.z, hiz.w};
        int kid[4] = {kids.x, kids.y, kids.z, kids.w};
        node = -1;
        for (int k = 0; k < 4; ++k) {
            if (kid[k] == kLeafEmpty) continue;
            float xa = fmaf(lx[k], r.idx, -r.oidx), xb = fmaf(hx[k], r.idx, -r.oidx);
            float ya = fmaf(ly[k], r.idy, -r.oidy), yb = fmaf(hy[k], r.idy, -r.oidy);
            float za = fmaf(lz[k], r.idz, -r.oidz), zb = fmaf(hz[k], r.idz, -r.oidz);
            float tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fmaxf(fminf(za, zb), r.t_min));
            // optional window [lo, *far] (chunked peeling): a candidate's depth
            // lies in its box's slab interval, so boxes entirely before lo or
            // after *far hold nothing the caller still wants
            float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), far ? *far : r.t_max0));
            if (!(tn <= tf) || tf < lo) continue;
            if (kid[k] >= 0) {
                if (sp >= kStackSize) {
                    raise_flag(overflow);
                    return;
                }
                stk[sp++] = kid[k];
                continue;
            }
            SRT_DCHECK(~kid[k] < s.n);
            const float4 *g = reinterpret_cast<const float4 *>(s.geom + ~kid[k]);
            visit(__ldg(g), __ldg(g + 1), __ldg(g + 2));
        }
        if (sp > 0) node = stk[--sp];
    }
}

// The K nearest (t, prim id) keys offered during one walk, as a bounded
// max-heap (root = farthest kept); sort() leaves them ascending.  Exact and
// biased compositing peel a ray's candidates K at a time with it: each walk
// keeps the K nearest above the last one composited, so any number of
// candidates is handled exactly in ceil(m / K) walks with O(K) state.
template <class T, class A, int K>
struct NearestK {
    T t[K];
    A a[K];
    int id[K];
    int n;
    int cap = K;  // kept entries (<= K)
    __device__ static bool less(T t1, int i1, T t2, int i2) { return t1 < t2 || (t1 == t2 && i1 < i2); }
    __device__ void sift_down(int j, T tt, int ii, A aa, int size) {
        while (true) {
            int c = 2 * j + 1;
            if (c >= size) break;
            if (c + 1 < size && less(t[c], id[c], t[c + 1], id[c + 1])) ++c;
            if (!less(tt, ii, t[c], id[c])) break;
            t[j] = t[c];
            id[j] = id[c];
            a[j] = a[c];
            j = c;
        }
        t[j] = tt;
        id[j] = ii;
        a[j] = aa;
    }
    __device__ void offer(T tt, int ii, A aa) {
        if (n < cap) {
            int j = n++;
            while (j > 0) {
                int p = (j - 1) >> 1;
                if (!less(t[p], id[p], tt, ii)) break;
                t[j] = t[p];
                id[j] = id[p];
                a[j] = a[p];
                j = p;
            }
            t[j] = tt;
            id[j] = ii;
            a[j] = aa;
        } else if (less(tt, ii, t[0], id[0])) {
            sift_down(0, tt, ii, aa, n);
        }
    }
    __device__ void sort() {
        for (int end = n - 1; end > 0; --end) {
            T tt = t[end];
            int ii = id[end];
            A aa = a[end];
            t[end] = t[0];
            id[end] = id[0];
            a[end] = a[0];
            sift_down(0, tt, ii, aa, end);
        }
    }
};

// Window bounds for for_each_leaf, widened so fp32 rounding of a candidate's
// depth against its box's slab interval can never prune it.
__device__ __forceinline__ float window_hi(double t) {
    return t >= 3.0e38 ? INFINITY : __double2float_ru(t + 1e-5 * (fabs(t) + 1.0));
}
__device__ __forceinline__ float window_lo(double t) {
    return t <= -3.0e38 ? -INFINITY : __double2float_rd(t - 1e-5 * (fabs(t) + 1.0));
}

constexpr int kExactChunk = 256;  // candidates composited per walk (exact mode)

template <int MODE>
__device__ void exact_ray(const SceneView &s, const RayState &r, float s2, const float *bg, double out[4],
                          int *overflow) {
    NearestK<float, float, kExactChunk> h;
    float lo_t = -INFINITY;  // exclusive lower bound (lo_t, lo_id) of the next chunk
    int lo_id = INT_MIN;
    double rr = 0.0, gg = 0.0, bb = 0.0, trans = 1.0;
    while (true) {
        h.n = 0;
        float far = INFINITY;  // the chunk's farthest kept depth once it is full
        for_each_leaf(
            s, r, overflow,
            [&](const float4 &gm, const float4 &ga, const float4 &gb) {
                Cand c = candidate<MODE>(r, gm, ga, gb, s2);
                if (!c.valid) return;
                const int id = __float_as_int(gb.z);
                if (!decltype(h)::less(lo_t, lo_id, c.t, id)) return;  // composited by an earlier chunk
                h.offer(c.t, id, c.alpha);
                if (h.n == h.cap) far = window_hi(h.t[0]);
            },
            &far, window_lo(lo_t));
        const int m = h.n;
        h.sort();
        // front to back in (t, prim id) order -- the stable mergesort order of
        // kernels.py:463 over ids appended in increasing order
        for (int i = 0; i < m; ++i) {
            SRT_DCHECK(h.id[i] >= 0 && h.id[i] < s.n);
            float3 col = sh_color(s.sh, s.sh_k, s.sh_deg, h.id[i], r.fdx, r.fdy, r.fdz);
            double w = trans * (double)h.a[i];
            rr += w * col.x;
            gg += w * col.y;
            bb += w * col.z;
            trans *= 1.0 - (double)h.a[i];
        }
        if (m < kExactChunk || trans == 0.0) break;  // all consumed, or nothing further can contribute
        lo_t = h.t[m - 1];
        lo_id = h.id[m - 1];
    }
    out[0] = rr + trans * bg[0];
    out[1] = gg + trans * bg[1];
    out[2] = bb + trans * bg[2];
    out[3] = 1.0 - trans;
}

template <int MODE>
__global__ void __launch_bounds__(128) k_exact_rays(SceneView s, const double *__restrict__ rays, int64_t R,
                                                    double t_min, double t_max, float s2, float3 bg, double *rgb,
                                                    double *op, int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double *q = rays + i * 6;
    RayState r;
    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
    const float b[3] = {bg.x, bg.y, bg.z};
    double o[4];
    exact_ray<MODE>(s, r, s2, b, o, overflow);
    rgb[i * 3] = o[0];
    rgb[i * 3 + 1] = o[1];
    rgb[i * 3 + 2] = o[2];
    op[i] = o[3];
}

// render_exact (kernels.py:677-723): per pixel, the mean over `passes`
// jittered rays of the exact composite.  Row-major fp64 outputs.
template <int MODE>
__global__ void __launch_bounds__(128) k_exact_frame(SceneView s, CamD cam, RenderArgs a, double *rgb, double *op,
                                                     int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)a.width * a.height) return;
    int px = (int)(i % a.width), py = (int)(i / a.width);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int f = 0; f < a.passes; ++f) {
        double dx, dy, dz;
        camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)(a.pass0 + f), a.seed, a.width, a.height, dx, dy, dz);
        RayState r;
        init_ray(r, cam.e[0], cam.e[1], cam.e[2], dx, dy, dz, 0.0, DBL_MAX);
        double o[4];
        exact_ray<MODE>(s, r, a.s2, a.bg, o, overflow);
        for (int c = 0; c < 4; ++c) acc[c] += o[c];
    }
    double inv = 1.0 / (double)a.passes;
    rgb[i * 3] = acc[0] * inv;
    rgb[i * 3 + 1] = acc[1] * inv;
    rgb[i * 3 + 2] = acc[2] * inv;
    op[i] = acc[3] * inv;
}

// ---------------------------------------------------------------------------
// Biased k-nearest composite (kernels.py:479-518, 561-580; tracer.py:305-343):
// every valid candidate in (t_min, t_max) is accepted with ONE draw (slot 0 of
// the ray's stream), and only the kk nearest accepted are composited with
// their original alphas, background behind.  Accepted candidates are peeled
// kBiasedChunk at a time (NearestK), so any kk and any number of accepted
// candidates are handled with O(kBiasedChunk) state.
//   RNG counter: u = counter_u(walk_key(frame_key(seed), ray_id0+i, sample0), pid)
//   RNG table:   u = table[pid * table_slots + 0]
//   RNG trig64:  u = the reference's trig hash of the fp64 hit (kernels.py:55-60)
// ---------------------------------------------------------------------------
constexpr int kBiasedChunk = 128;  // accepted candidates composited per walk (biased mode)

struct BiasedArgs {
    double t_min, t_max, s2;
    int mode, kk;
    float3 bg;
    uint32_t fkey, ray_id0, sample0;
    const double *table;
    int64_t tstride;
};

template <int MODE, int RNG>
__device__ void biased_ray(const SceneView &s, const double *q, uint32_t key, const BiasedArgs &a, double out[3],
                           int *overflow) {
    RayState r;
    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], a.t_min, a.t_max);
    const t64::Ray64 r64{q[0], q[1], q[2], q[3], q[4], q[5], a.t_min, a.t_max};
    const int kk = a.kk < 1 ? 1 : a.kk;
    const float s2f = (float)a.s2;
    NearestK<double, double, kBiasedChunk> h;
    double lo_t = -INFINITY;  // exclusive lower bound (lo_t, lo_id) of the next chunk
    int lo_id = INT_MIN;
    int done = 0;
    double rr = 0.0, gg = 0.0, bb = 0.0, trans = 1.0;
    while (done < kk) {
        h.n = 0;
        h.cap = kk - done < kBiasedChunk ? kk - done : kBiasedChunk;
        float far = INFINITY;
        for_each_leaf(s, r, overflow, [&](const float4 &gm, const float4 &ga, const float4 &gb) {
            const int pid = __float_as_int(gb.z);
            double t, alpha;
            bool acc;
            if (RNG == SRT_RNG_TRIG64) {
                double resid, hx, hy, hz;
                if (!t64::candidate<MODE>(r64, s.means64 + (int64_t)pid * 3, s.cov64 + (int64_t)pid * 6, a.s2, t,
                                          resid, hx, hy, hz))
                    return;
                if (t <= a.t_min || t >= a.t_max) return;
                alpha = t64::mul(s.opac64[pid], exp(t64::mul(-0.5, resid)));
                acc = t64::hash_position(hx, hy, hz, 0) < alpha;
            } else {
                Cand c = candidate<MODE>(r, gm, ga, gb, s2f);
                if (!c.valid) return;
                t = c.t;
                alpha = c.alpha;
                if (RNG == SRT_RNG_TABLE)
                    acc = __ldg(a.table + (int64_t)pid * a.tstride) < alpha;
                else
                    acc = counter_u(key, (uint32_t)pid) < c.alpha;
            }
            if (!acc || !decltype(h)::less(lo_t, lo_id, t, pid)) return;
            h.offer(t, pid, alpha);
            if (h.n == h.cap) far = window_hi(h.t[0]);
        }, &far, window_lo(lo_t));
        const int m = h.n;
        h.sort();
        const int take = m;  // cap <= kk - done
        for (int k = 0; k < take; ++k) {
            SRT_DCHECK(h.id[k] >= 0 && h.id[k] < s.n);
            float3 col = sh_color(s.sh, s.sh_k, s.sh_deg, h.id[k], r.fdx, r.fdy, r.fdz);
            double w = trans * h.a[k];
            rr += w * col.x;
            gg += w * col.y;
            bb += w * col.z;
            trans *= 1.0 - h.a[k];
        }
        done += take;
        if (m < h.cap || trans == 0.0) break;
        lo_t = h.t[m - 1];
        lo_id = h.id[m - 1];
    }
    out[0] = rr + trans * a.bg.x;
    out[1] = gg + trans * a.bg.y;
    out[2] = bb + trans * a.bg.z;
}

template <int MODE, int RNG>
__global__ void __launch_bounds__(128) k_biased_rays(SceneView s, const double *__restrict__ rays, int64_t R,
                                                     BiasedArgs a, double *rgb, int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    biased_ray<MODE, RNG>(s, rays + i * 6, walk_key(a.fkey, a.ray_id0 + (uint32_t)i, a.sample0), a, rgb + i * 3,
                          overflow);
}

// The cli's --compare-biased frame (cli.py:164-203): per pixel, the mean
// over passes of the biased composite of the jittered camera ray of that
// pass; the counter draw of pixel (px,py), pass f is (seed, py*W+px, f).
template <int MODE, int RNG>
__global__ void __launch_bounds__(128) k_biased_frame(SceneView s, CamD cam, BiasedArgs a, int width, int height,
                                                      int passes, int pass0, uint32_t seed, double *rgb,
                                                      int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)width * height) return;
    int px = (int)(i % width), py = (int)(i / width);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int f = 0; f < passes; ++f) {
        double q[6] = {cam.e[0], cam.e[1], cam.e[2], 0.0, 0.0, 0.0};
        camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)(pass0 + f), seed, width, height, q[3], q[4], q[5]);
        double o[3];
        biased_ray<MODE, RNG>(s, q, walk_key(a.fkey, (uint32_t)i, (uint32_t)(pass0 + f)), a, o, overflow);
        for (int c = 0; c < 3; ++c) acc[c] += o[c];
    }
    double inv = 1.0 / (double)passes;
    for (int c = 0; c < 3; ++c) rgb[i * 3 + c] = acc[c] * inv;
}

static BiasedArgs biased_args(double t_min, double t_max, double s2, int mode, int kk, const double *bg,
                              uint32_t seed, uint32_t ray_id0, uint32_t sample0, const double *table,
                              int64_t tstride) {
    BiasedArgs a;
    a.t_min = t_min;
    a.t_max = t_max;
    a.s2 = s2;
    a.mode = mode;
    a.kk = kk;
    a.bg = make_float3((float)bg[0], (float)bg[1], (float)bg[2]);
    uint32_t x = seed ^ 0x9E3779B9u;  // frame_key on the host
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    a.fkey = x;
    a.ray_id0 = ray_id0;
    a.sample0 = sample0;
    a.table = table;
    a.tstride = tstride;
    return a;
}

#define SRT_BIASED_DISPATCH(RNGV, MODEV, LAUNCH)                         \
    if ((RNGV) == SRT_RNG_TRIG64) {                                      \
        if ((MODEV) == 0) LAUNCH(0, SRT_RNG_TRIG64); else LAUNCH(1, SRT_RNG_TRIG64); \
    } else if ((RNGV) == SRT_RNG_TABLE) {                                \
        if ((MODEV) == 0) LAUNCH(0, SRT_RNG_TABLE); else LAUNCH(1, SRT_RNG_TABLE);   \
    } else {                                                             \
        if ((MODEV) == 0) LAUNCH(0, SRT_RNG_COUNTER); else LAUNCH(1, SRT_RNG_COUNTER); \
    }

srt_status launch_biased_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R, int kk,
                              const double *bg, const double *d_table, double *d_rgb, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    BiasedArgs a = biased_args(p->t_min, p->t_max, p->s2, p->mode, kk, bg, p->seed, p->ray_id0, p->sample0, d_table,
                               p->table_slots);
    SceneView v = s->view();
#define SRT_B(M, G) k_biased_rays<M, G><<<blocks, 128, 0, st>>>(v, d_rays, R, a, d_rgb, s->d_flag)
    SRT_BIASED_DISPATCH(p->rng, p->mode, SRT_B)
#undef SRT_B
    return cuda_status(cudaGetLastError(), "k_biased_rays launch");
}

srt_status launch_biased_frame(const SrtScene *s, const CamD &cam, const SrtRenderParams *p, int kk,
                               double *d_rgb, cudaStream_t st) {
    int64_t n = (int64_t)p->width * p->height;
    unsigned blocks = (unsigned)((n + 127) / 128);
    if (blocks == 0) return SRT_OK;
    BiasedArgs a = biased_args(0.0, DBL_MAX, p->s2, p->mode, kk, p->background, p->seed, 0, 0, nullptr, 0);
    SceneView v = s->view();
#define SRT_B(M, G)                                                                                          \
    k_biased_frame<M, G><<<blocks, 128, 0, st>>>(v, cam, a, p->width, p->height, p->passes, p->pass0, p->seed, \
                                                 d_rgb, s->d_flag)
    SRT_BIASED_DISPATCH(p->rng, p->mode, SRT_B)
#undef SRT_B
    return cuda_status(cudaGetLastError(), "k_biased_frame launch");
}

srt_status launch_exact_rays(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max, int mode,
                             double s2, const double *bg, double *d_rgb, double *d_op, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    float3 b = make_float3((float)bg[0], (float)bg[1], (float)bg[2]);
    if (mode == 0)
        k_exact_rays<0><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, b, d_rgb, d_op,
                                                s->d_flag);
    else
        k_exact_rays<1><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, b, d_rgb, d_op,
                                                s->d_flag);
    return cuda_status(cudaGetLastError(), "k_exact_rays launch");
}

srt_status launch_exact_frame(const SrtScene *s, const CamD &cam, const RenderArgs &a, double *d_rgb, double *d_op,
                              cudaStream_t st) {
    int64_t n = (int64_t)a.width * a.height;
    unsigned blocks = (unsigned)((n + 127) / 128);
    if (blocks == 0) return SRT_OK;
    if (a.mode == 0)
        k_exact_frame<0><<<blocks, 128, 0, st>>>(s->view(), cam, a, d_rgb, d_op, s->d_flag);
    else
        k_exact_frame<1><<<blocks, 128, 0, st>>>(s->view(), cam, a, d_rgb, d_op, s->d_flag);
    return cuda_status(cudaGetLastError(), "k_exact_frame launch");
}

}  // namespace srt
