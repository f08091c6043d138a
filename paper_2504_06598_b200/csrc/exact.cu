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
#include <algorithm>
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
                // fp32 screen first: certainly-invalid candidates skip the fp64 stage
                if (!screen<MODE>(r, gm, ga, gb, s2, sqrtf(s2), r.t_max0).maybe) return;
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
                // fp32 screen first: certainly invalid, or a draw above the
                // screen's alpha bound (certainly rejected), skips the fp64 stage
                const Screen sc = screen<MODE>(r, gm, ga, gb, s2f, sqrtf(s2f), r.t_max0);
                if (!sc.maybe) return;
                const float u = RNG == SRT_RNG_TABLE ? (float)__ldg(a.table + (int64_t)pid * a.tstride)
                                                     : counter_u(key, (uint32_t)pid);
                if (RNG != SRT_RNG_TABLE && u >= sc.alpha_hi) return;
                Cand c = candidate<MODE>(r, gm, ga, gb, s2f);
                if (!c.valid) return;
                t = c.t;
                alpha = c.alpha;
                if (RNG == SRT_RNG_TABLE)
                    acc = __ldg(a.table + (int64_t)pid * a.tstride) < alpha;
                else
                    acc = u < c.alpha;
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


// ---------------------------------------------------------------------------
// Exact and biased compositing as warp packets: render(reference_mode=True)
// frames, the --compare-biased frame (cli.py:164-203) and one-hemisphere
// exact_batch / biased_batch rays.  The 32 rays of a packet (an 8x4 pixel
// block, or 32 consecutive rays of a coherence-sorted batch) walk the octant
// tree together; leaf children any lane hits are compacted into a warp job
// queue as in k_trace_packet.  A job screens the owner's ray in fp32
// (certainly-invalid candidates never reach fp64; in biased counter mode a
// draw above the screen's alpha bound is a certain rejection), evaluates
// the exact candidate exactly as the per-lane paths do, and appends a valid
// (biased: accepted) one as (hit key, alpha) to the owner's list in global
// scratch.
//  - exact (kernels.py:441-475): unclipped; every valid candidate counts.
//  - biased (kernels.py:479-518): one draw per candidate (slot 0 of the
//    ray's stream); only the kk nearest accepted are composited, so each
//    owner keeps the kk smallest depths it has accepted (kk <= kBiasedClip)
//    and clips its walk beyond the kk-th (widened, conservative): nodes and
//    candidates past it cannot be among the kk nearest.
// Once the walk ends, the warp sorts each ray's list by (t, prim id) -- the
// stable mergesort order of the reference -- and composites front to back
// in fp64 (composite_ray_warp).  A ray with more than kExactCap list
// entries composites through the per-lane chunked peeling (out of line).
// ---------------------------------------------------------------------------
constexpr int kExactCap = 1024;      // list entries per ray (C3-target: mean 261, max ~720 valid candidates)
constexpr int kExactThreads = 128;
// 6 blocks (80 registers) per SM bound the list scratch: 148 x 6 x 128 lanes x
// 12 KB = 1.4 GB; 7 / 8 blocks were slower (1080p frame 52.6 -> 60.6 / 65.3 ms)
constexpr int kExactBlocksPerSM = 6;
constexpr int kBiasedClip = 8;        // biased walks with kk <= this clip at the kk-th accepted depth

enum { kPacketExact = 0, kPacketBiasedCounter = 1, kPacketBiasedTable = 2 };

// Rays of a packet: camera frames (all passes of an 8x4 pixel block, summed
// in the warp in pass order, mean written once: deterministic).  The
// biased frame's draw of pixel (px, py), pass f is keyed (seed, py*W+px, f)
// (k_biased_frame).
struct ExactFrameSrc {
    CamD cam;
    int width, height, passes, pass0, bw;
    uint32_t seed, fkey;
    double *rgb, *op;
    double t_min, t_max;
    __device__ uint32_t packets() const { return (uint32_t)bw * (uint32_t)((height + 3) / 4); }
    __device__ bool ray(uint32_t p, int lane, int f, double o[3], double d[3]) const {
        const int px = (int)(p % (uint32_t)bw) * 8 + (lane & 7), py = (int)(p / (uint32_t)bw) * 4 + (lane >> 3);
        if (px >= width || py >= height) return false;
        camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)(pass0 + f), seed, width, height, d[0], d[1], d[2]);
        o[0] = cam.e[0], o[1] = cam.e[1], o[2] = cam.e[2];
        return true;
    }
    __device__ uint32_t key(uint32_t p, int lane, int f) const {
        const int px = (int)(p % (uint32_t)bw) * 8 + (lane & 7), py = (int)(p / (uint32_t)bw) * 4 + (lane >> 3);
        return walk_key(fkey, (uint32_t)py * (uint32_t)width + (uint32_t)px, (uint32_t)(pass0 + f));
    }
    __device__ void write(uint32_t p, int lane, const double acc[4]) const {
        const int px = (int)(p % (uint32_t)bw) * 8 + (lane & 7), py = (int)(p / (uint32_t)bw) * 4 + (lane >> 3);
        const int64_t i = (int64_t)py * width + px;
        const double inv = 1.0 / (double)passes;
        rgb[i * 3] = acc[0] * inv;
        rgb[i * 3 + 1] = acc[1] * inv;
        rgb[i * 3 + 2] = acc[2] * inv;
        if (op) op[i] = acc[3] * inv;
    }
};

// Explicit rays (exact_batch kernels.py:584-604, biased_batch 561-580),
// walked in the order of an optional coherence permutation and written in
// the caller's; ray i draws with (seed, ray_id0 + i, sample0).
struct ExactRaySrc {
    const double *rays;
    const uint32_t *perm;
    uint32_t R;
    int passes;
    double *rgb, *op;
    double t_min, t_max;
    uint32_t fkey, ray_id0, sample0;
    __device__ uint32_t packets() const { return (R + 31u) / 32u; }
    __device__ uint32_t index(uint32_t p, int lane) const {
        const uint32_t k = p * 32u + (uint32_t)lane;
        return perm ? __ldg(perm + k) : k;
    }
    __device__ bool ray(uint32_t p, int lane, int, double o[3], double d[3]) const {
        if (p * 32u + (uint32_t)lane >= R) return false;
        const double *q = rays + (int64_t)index(p, lane) * 6;
        o[0] = q[0], o[1] = q[1], o[2] = q[2], d[0] = q[3], d[1] = q[4], d[2] = q[5];
        return true;
    }
    __device__ uint32_t key(uint32_t p, int lane, int) const {
        return walk_key(fkey, ray_id0 + index(p, lane), sample0);
    }
    __device__ void write(uint32_t p, int lane, const double acc[4]) const {
        const int64_t i = index(p, lane);
        rgb[i * 3] = acc[0];
        rgb[i * 3 + 1] = acc[1];
        rgb[i * 3 + 2] = acc[2];
        if (op) op[i] = acc[3];
    }
};

// Per-packet arguments beyond the source.
struct PacketCompositeArgs {
    float s2;
    float3 bg;
    int kk;                 // biased: accepted candidates composited
    const double *table;    // biased table mode: u = table[pid * tstride]
    int64_t tstride;
    BiasedArgs ba;          // biased: the per-lane fallback's arguments
};

template <int MODE>
__device__ __noinline__ void exact_ray_long(const SceneView &s, const RayState &r, float s2, const float *bg,
                                            double out[4], int *overflow) {
    exact_ray<MODE>(s, r, s2, bg, out, overflow);
}
template <int MODE, int RNG>
__device__ __noinline__ void biased_ray_long(const SceneView &s, const double *q, uint32_t key, const BiasedArgs &a,
                                             double out[4], int *overflow) {
    biased_ray<MODE, RNG>(s, q, key, a, out, overflow);
    out[3] = 0.0;
}

// Sort ray o's list (m <= kExactCap entries, key[0..m), alpha[0..m)) and
// composite it front to back, the whole warp on one ray:
//  1. depth range of the list (warp min / max of the orderable keys);
//  2. counting sort into kExactBuckets depth buckets in shared memory
//     (bucket index monotone in t, so bucket order is depth order), keys
//     and list positions scattered into sk / sx;
//  3. insertion sort inside each bucket (a few entries; exact (t, id) order);
//  4. compositing of the first `take` in chunks of 32: lane i of a chunk takes entry c + i, the
//     transmittance before it is the chunk's base times an exclusive warp
//     prefix product of (1 - alpha); sum of T_i alpha_i c_i over the warp.
// Same fp64 terms as exact_ray, products and sums associated differently
// (relative 1e-15).
constexpr int kExactBuckets = 256;
constexpr int kExactSortSmem = 512;  // lists up to this long sort in shared memory, longer ones in global scratch
__device__ __noinline__ void composite_ray_warp(const SceneView &s, const unsigned long long *key,
                                                const float *alpha, int m, int take, float fdx, float fdy,
                                                float fdz, const float *bg, unsigned *sk, uint16_t *sx, int *scn,
                                                double out[4]) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    constexpr int NB = kExactBuckets, PER = kExactBuckets / 32;
    // 1. depth range
    unsigned kmin = 0xffffffffu, kmax = 0u;
    for (int i = lane; i < m; i += 32) {
        const unsigned hi = (unsigned)(key[i] >> 32);
        kmin = min(kmin, hi);
        kmax = max(kmax, hi);
    }
    kmin = __reduce_min_sync(FULL, kmin);
    kmax = __reduce_max_sync(FULL, kmax);
    // buckets linear in the orderable depth bits (monotone in t, and linear in
    // t within one binade): no float decode per entry
    const float scale = (float)NB / ((float)(kmax - kmin) + 1.0f);
    auto bucket = [&](unsigned long long k) {
        const float b = (float)((unsigned)(k >> 32) - kmin) * scale;
        return b >= (float)(NB - 1) ? NB - 1 : (int)b;
    };
    // 2. counting sort: counts, exclusive scan, scatter
#pragma unroll
    for (int j = 0; j < PER; ++j) scn[lane * PER + j] = 0;
    __syncwarp();
    for (int i = lane; i < m; i += 32) atomicAdd(&scn[bucket(key[i])], 1);
    __syncwarp();
    int c[PER], run = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        c[j] = scn[lane * PER + j];
        run += c[j];
    }
    int incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += v;
    }
    int base = incl - run;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        scn[lane * PER + j] = base;
        base += c[j];
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
        const unsigned long long k = key[i];
        const int pos = atomicAdd(&scn[bucket(k)], 1);
        sk[pos] = (unsigned)(k >> 32);  // orderable depth; ties resolved on the list's prim id
        sx[pos] = (uint16_t)i;
    }
    __syncwarp();
    // 3. insertion sort inside each bucket [end of bucket b-1, end of bucket b)
    //    by (t, prim id); lane l sorts buckets l, l + 32, ... so the dense
    //    depth range (neighbouring buckets) spreads over the lanes instead of
    //    serialising on a few (exact 1080p frame 52.0 -> see DESIGN §5)
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int b = j * 32 + lane;
        const int lo = b == 0 ? 0 : scn[b - 1], hi = scn[b];
        for (int i = lo + 1; i < hi; ++i) {
            const unsigned k = sk[i];
            const uint16_t x = sx[i];
            int q = i - 1;
            while (q >= lo && (sk[q] > k || (sk[q] == k && key[sx[q]] > key[x]))) {
                sk[q + 1] = sk[q];
                sx[q + 1] = sx[q];
                --q;
            }
            sk[q + 1] = k;
            sx[q + 1] = x;
        }
    }
    __syncwarp();
    // 4. front-to-back compositing, 32 entries per step
    double T = 1.0, rr = 0.0, gg = 0.0, bb = 0.0;
    for (int c0 = 0; c0 < take; c0 += 32) {
        const int i = c0 + lane;
        double a = 0.0;
        float3 col = make_float3(0.0f, 0.0f, 0.0f);
        if (i < take) {
            const int x = sx[i];
            const int id = (int)(unsigned)key[x];
            SRT_DCHECK(id >= 0 && id < s.n);
            a = (double)alpha[x];
            col = sh_color_v(s.sh, s.sh_k, s.sh_deg, id, fdx, fdy, fdz);
        }
        double p = 1.0 - a;  // inclusive prefix product of (1 - alpha)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double q = __shfl_up_sync(FULL, p, d);
            if (lane >= d) p *= q;
        }
        double ex = __shfl_up_sync(FULL, p, 1);
        if (lane == 0) ex = 1.0;
        const double w = T * ex * a;
        rr += w * col.x;
        gg += w * col.y;
        bb += w * col.z;
        T *= __shfl_sync(FULL, p, 31);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        rr += __shfl_xor_sync(FULL, rr, d);
        gg += __shfl_xor_sync(FULL, gg, d);
        bb += __shfl_xor_sync(FULL, bb, d);
    }
    out[0] = rr + T * bg[0];
    out[1] = gg + T * bg[1];
    out[2] = bb + T * bg[2];
    out[3] = 1.0 - T;
}

template <int MODE, int KIND, class Src>
__global__ void __launch_bounds__(kExactThreads, kExactBlocksPerSM)
    k_composite_packet(SceneView s, Src src, PacketCompositeArgs pa, unsigned long long *lkey, float *lalpha,
                       unsigned *gsort, uint32_t *work, int *overflow) {
    constexpr int W = kExactThreads / 32, PSTACK = 128, BATCH = 32;
    constexpr bool BIASED = KIND != kPacketExact;
    constexpr int KC = BIASED ? kBiasedClip : 1;
    __shared__ double sray[W][32][7];  // fp64 origin, direction, 1/|d|^2 of each lane's ray
    __shared__ int scnt[W][32];        // list entries per ray
    __shared__ uint32_t skey[W][32];   // biased counter mode: walk key of each ray
    __shared__ uint32_t sjob[W][BATCH + 128];
    __shared__ int2 sstk[W][PSTACK];   // (node, warp-min entry key)
    __shared__ unsigned long long stopk[W][KC][32];  // biased: the kk nearest accepted (hit key, alpha) per ray,
    __shared__ float stopa[W][KC][32];               // ascending -- the composite itself when clipping
    __shared__ float sfar[W][32];      // far bound of each ray during a job round
    // one ray's list at a time, bucket-sorted: in shared memory up to
    // kExactSortSmem entries, else in the warp's global sort scratch
    __shared__ unsigned ssk[W][kExactSortSmem];
    __shared__ uint16_t ssx[W][kExactSortSmem];
    __shared__ int sscn[W][kExactBuckets];
    const unsigned FULL = 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const float s2 = pa.s2, sqrt_s2 = sqrtf(s2);
    const float bg[3] = {pa.bg.x, pa.bg.y, pa.bg.z};
    const bool clip = BIASED && pa.kk <= kBiasedClip;
    const size_t lbase = ((size_t)blockIdx.x * W + wid) * 32u * (size_t)kExactCap;
    unsigned long long *wkey = lkey + lbase;
    float *walpha = lalpha + lbase;
    unsigned *gsk = gsort + ((size_t)blockIdx.x * W + wid) * kExactCap * 2;  // u32 keys, then u16 positions
    uint16_t *gsx = reinterpret_cast<uint16_t *>(gsk + kExactCap);
    const RayState r0 = [] {
        RayState z;
        init_ray(z, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0);
        return z;
    }();
    const uint32_t npk = src.packets();
    while (true) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(work, 1u);
        p = __shfl_sync(FULL, p, 0);
        if (p >= npk) break;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        bool any_valid = false;
        for (int f = 0; f < src.passes; ++f) {
            double o[3], d[3];
            const bool valid = src.ray(p, lane, f, o, d);
            any_valid |= valid;
            RayState r = r0;
            float far = -INFINITY;  // idle lanes hit nothing
            int seen = 0, nbest = 0;  // biased clip: list entries ingested, depths kept
            if (valid) {
                init_ray(r, o[0], o[1], o[2], d[0], d[1], d[2], src.t_min, src.t_max);
                far = r.t_max0;
                double *q = sray[wid][lane];
                q[0] = o[0], q[1] = o[1], q[2] = o[2], q[3] = d[0], q[4] = d[1], q[5] = d[2], q[6] = r.inv_dd;
                if (KIND == kPacketBiasedCounter) skey[wid][lane] = src.key(p, lane, f);
            }
            scnt[wid][lane] = 0;
            const unsigned vm = __ballot_sync(FULL, valid);
            const unsigned nx_m = __ballot_sync(FULL, valid && signbit(r.idx));
            const unsigned ny_m = __ballot_sync(FULL, valid && signbit(r.idy));
            const unsigned nz_m = __ballot_sync(FULL, valid && signbit(r.idz));
            const int oct = (nx_m ? 1 : 0) | (ny_m ? 2 : 0) | (nz_m ? 4 : 0);
            const bool mixed = (nx_m && nx_m != vm) || (ny_m && ny_m != vm) || (nz_m && nz_m != vm);
            const uint32_t obase = (uint32_t)oct * (uint32_t)s.num_nodes4;
            int sp = 0, njobs = 0;
            int node = (s.num_nodes4 > 0 && vm) ? 0 : kLeafEmpty;
            auto run_jobs = [&]() {
                if (BIASED) sfar[wid][lane] = far;
                __syncwarp();
                for (int jb = 0; jb < njobs; jb += 32) {
                    const int j = jb + lane;
                    if (j < njobs) {
                        const uint32_t job = sjob[wid][j];
                        const int ow = (int)(job & 31u), slot = (int)(job >> 5);
                        SRT_DCHECK(slot >= 0 && slot < s.n);
                        const double *q = sray[wid][ow];
                        ExactRay er;
                        er.ox = q[0], er.oy = q[1], er.oz = q[2], er.dx = q[3], er.dy = q[4], er.dz = q[5];
                        er.inv_dd = q[6];
                        er.fdx = (float)er.dx, er.fdy = (float)er.dy, er.fdz = (float)er.dz;
                        er.t_min = (float)src.t_min;
                        er.t_max0 = src.t_max >= 3.0e38 ? INFINITY : (float)src.t_max;
                        ScreenRay sr;
                        sr.fox = (float)er.ox, sr.foy = (float)er.oy, sr.foz = (float)er.oz;
                        sr.omag = fmaxf(fabsf(sr.fox), fmaxf(fabsf(sr.foy), fabsf(sr.foz)));
                        sr.fdx = er.fdx, sr.fdy = er.fdy, sr.fdz = er.fdz;
                        sr.inv_dd = er.inv_dd;
                        sr.t_min = er.t_min, sr.t_max0 = er.t_max0;
                        const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
                        const float4 gm = __ldg(g), ga = __ldg(g + 1), gb = __ldg(g + 2);
                        const float ofar = BIASED ? sfar[wid][ow] : er.t_max0;
                        const Screen sc = screen<MODE>(sr, gm, ga, gb, s2, sqrt_s2, ofar);
                        const int pid = __float_as_int(gb.z);
                        float u = 0.0f;
                        bool go = sc.maybe;
                        if (KIND == kPacketBiasedCounter) {
                            u = counter_u(skey[wid][ow], (uint32_t)pid);
                            go = go && u < sc.alpha_hi;  // u >= alpha_hi: certainly rejected
                        }
                        if (go) {
                            const Cand c = candidate<MODE>(er, gm, ga, gb, s2);
                            bool take = c.valid;
                            if (KIND == kPacketBiasedCounter) take = take && u < c.alpha;
                            if (KIND == kPacketBiasedTable)
                                take = take && __ldg(pa.table + (int64_t)pid * pa.tstride) < (double)c.alpha;
                            if (take) {
                                const int pos = atomicAdd(&scnt[wid][ow], 1);
                                if (pos < kExactCap) {
                                    wkey[(size_t)ow * kExactCap + pos] = pack_hit(c.t, pid);
                                    walpha[(size_t)ow * kExactCap + pos] = c.alpha;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                njobs = 0;
                if (clip && valid) {
                    // ingest this batch's accepted candidates into the kk nearest
                    // (by (t, prim id)); clip beyond the kk-th
                    const int m = min(scnt[wid][lane], kExactCap);
                    for (; seen < m; ++seen) {
                        const unsigned long long kk_key = wkey[(size_t)lane * kExactCap + seen];
                        if (nbest == pa.kk && !(kk_key < stopk[wid][nbest - 1][lane])) continue;
                        const float ka = walpha[(size_t)lane * kExactCap + seen];
                        int q = nbest < pa.kk ? nbest++ : nbest - 1;
                        while (q > 0 && stopk[wid][q - 1][lane] > kk_key) {
                            stopk[wid][q][lane] = stopk[wid][q - 1][lane];
                            stopa[wid][q][lane] = stopa[wid][q - 1][lane];
                            --q;
                        }
                        stopk[wid][q][lane] = kk_key;
                        stopa[wid][q][lane] = ka;
                    }
                    if (nbest == pa.kk) far = fminf(far, window_hi((double)unpack_t(stopk[wid][pa.kk - 1][lane])));
                }
            };
            while (true) {
                if (njobs >= BATCH || (node == kLeafEmpty && sp == 0 && njobs)) run_jobs();
                if (node == kLeafEmpty) {
                    if (sp == 0) break;
                    // pop, culling entries beyond every lane's far bound
                    const int maxfar = __reduce_max_sync(FULL, ordered_key(far, 3));
                    while (sp > 0) {
                        const int2 en = sstk[wid][--sp];
                        if (en.y <= maxfar) {
                            node = en.x;
                            break;
                        }
                    }
                    if (node == kLeafEmpty) continue;  // all culled: flush what is queued, then finish
                }
                SRT_DCHECK(node >= 0 && node < s.num_nodes4);
                const float4 *np = reinterpret_cast<const float4 *>(s.nodes8 + (obase + (uint32_t)node));
                const float4 ax = __ldg(np), bx = __ldg(np + 1), ay = __ldg(np + 2), by = __ldg(np + 3),
                             az = __ldg(np + 4), bz = __ldg(np + 5);
                // child codes by shuffle, as in k_trace_packet (lane j holds code j & 3)
                const int mykid = __ldg(reinterpret_cast<const int *>(np + 6) + (lane & 3));
                const unsigned hint = (unsigned)__ldg(reinterpret_cast<const int *>(np + 7));
                const float pax[4] = {ax.x, ax.y, ax.z, ax.w}, pbx[4] = {bx.x, bx.y, bx.z, bx.w};
                const float pay[4] = {ay.x, ay.y, ay.z, ay.w}, pby[4] = {by.x, by.y, by.z, by.w};
                const float paz[4] = {az.x, az.y, az.z, az.w}, pbz[4] = {bz.x, bz.y, bz.z, bz.w};
                unsigned hitm = 0;
                float tn4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float tn, tf;
                    if (!mixed) {
                        tn = fmaxf(fmaxf(fmaf(pax[k], r.idx, -r.oidx), fmaf(pay[k], r.idy, -r.oidy)),
                                   fmaf(paz[k], r.idz, -r.oidz));
                        tf = fminf(fminf(fmaf(pbx[k], r.idx, -r.oidx), fmaf(pby[k], r.idy, -r.oidy)),
                                   fminf(fmaf(pbz[k], r.idz, -r.oidz), far));
                    } else {
                        const float xa = fmaf(pax[k], r.idx, -r.oidx), xb = fmaf(pbx[k], r.idx, -r.oidx);
                        const float ya = fmaf(pay[k], r.idy, -r.oidy), yb = fmaf(pby[k], r.idy, -r.oidy);
                        const float za = fmaf(paz[k], r.idz, -r.oidz), zb = fmaf(pbz[k], r.idz, -r.oidz);
                        tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fminf(za, zb));
                        tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), far));
                    }
                    // closed slab (kernels.py:279,308) clipped to [t_min, far]: boxes
                    // wholly behind the origin are culled here
                    hitm |= fmaxf(tn, r.t_min) <= tf ? (1u << k) : 0u;
                    tn4[k] = tn;
                }
                const unsigned leafm = (hint >> 4) & 15u;
                hitm &= hint & 15u;
                node = kLeafEmpty;
                const unsigned any = __reduce_or_sync(FULL, hitm);
                const unsigned lh = hitm & leafm;
                for (unsigned al = any & leafm; al; al &= al - 1) {
                    const int k = __ffs(al) - 1;
                    const bool h = (lh >> k) & 1u;
                    const unsigned bm = __ballot_sync(FULL, h);
                    const int kc = __shfl_sync(FULL, mykid, k);
                    if (h) {
                        SRT_DCHECK(njobs + __popc(bm & lt) < BATCH + 128);
                        sjob[wid][njobs + __popc(bm & lt)] = ((uint32_t)~kc << 5) | (uint32_t)lane;
                    }
                    njobs += __popc(bm);
                }
                // inner children: nearest (warp-min entry) first -- lists arrive
                // roughly in depth order and the biased clip tightens early; the
                // rest pushed far-to-near with their warp-min entries
                const unsigned ih = hitm & ~leafm;
                const unsigned ai = any & ~leafm;
                if (ai) {
                    if (!(ai & (ai - 1))) {
                        node = __shfl_sync(FULL, mykid, __ffs(ai) - 1);
                    } else {
                        int wk[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            wk[k] = __reduce_min_sync(FULL, ((ih >> k) & 1u) ? ordered_key(tn4[k], k) : 0x7FFFFFFF);
#define SRT_CX(a, b)                  \
    {                                 \
        int lo_ = min(wk[a], wk[b]);  \
        int hi_ = max(wk[a], wk[b]);  \
        wk[a] = lo_;                  \
        wk[b] = hi_;                  \
    }
                        SRT_CX(0, 1) SRT_CX(2, 3) SRT_CX(0, 2) SRT_CX(1, 3) SRT_CX(1, 2)
#undef SRT_CX
                        const int nin = __popc(ai);
                        if (sp + nin - 1 > PSTACK) {
                            if (lane == 0) raise_flag(overflow);
                            break;
                        }
#pragma unroll
                        for (int j = 3; j >= 1; --j)
                            if (j < nin)
                                sstk[wid][sp + nin - 1 - j] = make_int2(__shfl_sync(FULL, mykid, wk[j] & 3), wk[j] & ~3);
                        sp += nin - 1;
                        node = __shfl_sync(FULL, mykid, wk[0] & 3);
                    }
                }
                __syncwarp();
            }
            if (njobs) run_jobs();  // a stack overflow left the loop with jobs queued
            __syncwarp();
            // the warp sorts and composites each ray's list in turn; a clipped
            // biased ray composites its kept kk nearest itself
            const int m = scnt[wid][lane];
            double mine[4] = {0.0, 0.0, 0.0, 0.0};
            if (clip && valid && m <= kExactCap) {
                double rr = 0.0, gg = 0.0, bb = 0.0, trans = 1.0;
                for (int i = 0; i < nbest; ++i) {
                    const int id = (int)(unsigned)stopk[wid][i][lane];
                    SRT_DCHECK(id >= 0 && id < s.n);
                    const double a = (double)stopa[wid][i][lane];
                    const float3 col = sh_color_v(s.sh, s.sh_k, s.sh_deg, id, r.fdx, r.fdy, r.fdz);
                    const double w = trans * a;
                    rr += w * col.x;
                    gg += w * col.y;
                    bb += w * col.z;
                    trans *= 1.0 - a;
                }
                mine[0] = rr + trans * bg[0];
                mine[1] = gg + trans * bg[1];
                mine[2] = bb + trans * bg[2];
                mine[3] = 1.0 - trans;
            }
            for (unsigned todo = __ballot_sync(FULL, valid && m <= kExactCap && !clip); todo; todo &= todo - 1) {
                const int ow = __ffs(todo) - 1;
                const double *q = sray[wid][ow];
                double out[4];
                const int mo = scnt[wid][ow];
                const bool sm = mo <= kExactSortSmem;
                composite_ray_warp(s, wkey + (size_t)ow * kExactCap, walpha + (size_t)ow * kExactCap, mo,
                                   BIASED ? min(mo, pa.kk) : mo, (float)q[3], (float)q[4], (float)q[5], bg,
                                   sm ? ssk[wid] : gsk, sm ? ssx[wid] : gsx, sscn[wid], out);
                if (lane == ow)
                    for (int c = 0; c < 4; ++c) mine[c] = out[c];
            }
            if (valid && m > kExactCap) {
                if constexpr (BIASED) {
                    const double qq[6] = {o[0], o[1], o[2], d[0], d[1], d[2]};
                    biased_ray_long<MODE, KIND == kPacketBiasedTable ? SRT_RNG_TABLE : SRT_RNG_COUNTER>(
                        s, qq, src.key(p, lane, f), pa.ba, mine, overflow);
                } else {
                    exact_ray_long<MODE>(s, r, s2, bg, mine, overflow);
                }
            }
            for (int c = 0; c < 4; ++c) acc[c] += mine[c];
            __syncwarp();
        }
        if (any_valid) src.write(p, lane, acc);
    }
    release_counter(work);
}

// List scratch + work counter for one k_composite_packet launch (stream-ordered).
template <int MODE, int KIND, class Src>
static srt_status launch_composite_packet(const SrtScene *s, const Src &src, const PacketCompositeArgs &pa,
                                          cudaStream_t st) {
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_composite_packet<MODE, KIND, Src>, kExactThreads, 0);
    per_sm = std::max(1, std::min(per_sm, kExactBlocksPerSM));
    const int grid = num_sms * per_sm;
    const size_t entries = (size_t)grid * kExactThreads * kExactCap;
    unsigned long long *lkey = nullptr;
    float *lalpha = nullptr;
    unsigned *gsort = nullptr;
    LaunchCounter work;
    srt_status rc = work.init(s, st);
    if (!rc) rc = cuda_status(cudaMallocAsync((void **)&lkey, entries * sizeof(unsigned long long), st), "list alloc");
    if (!rc) rc = cuda_status(cudaMallocAsync((void **)&lalpha, entries * sizeof(float), st), "list alloc");
    if (!rc)
        rc = cuda_status(
            cudaMallocAsync((void **)&gsort, (size_t)grid * (kExactThreads / 32) * kExactCap * 2 * sizeof(unsigned), st),
            "sort scratch alloc");
    if (!rc) {
        k_composite_packet<MODE, KIND, Src><<<grid, kExactThreads, 0, st>>>(s->view(), src, pa, lkey, lalpha, gsort,
                                                                            work.p, s->d_flag);
        rc = cuda_status(cudaGetLastError(), "k_composite_packet launch");
    }
    if (lkey) cudaFreeAsync(lkey, st);
    if (lalpha) cudaFreeAsync(lalpha, st);
    if (gsort) cudaFreeAsync(gsort, st);
    return rc;
}

template <int KIND, class Src>
static srt_status launch_composite_packet(const SrtScene *s, const Src &src, int mode, const PacketCompositeArgs &pa,
                                          cudaStream_t st) {
    return mode == 0 ? launch_composite_packet<0, KIND>(s, src, pa, st) : launch_composite_packet<1, KIND>(s, src, pa, st);
}

srt_status launch_biased_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R, int kk,
                              const double *bg, const double *d_table, double *d_rgb, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    BiasedArgs a = biased_args(p->t_min, p->t_max, p->s2, p->mode, kk, bg, p->seed, p->ray_id0, p->sample0, d_table,
                               p->table_slots);
    // counter / table draws: one-hemisphere batches walk as packets
    // (coherence-sorted unless one origin), clipped at the kk-th accepted depth
    bool one_origin = false, one_hemisphere = false;
    if (p->rng != SRT_RNG_TRIG64 && R >= 4096 && (uint64_t)R < (1ull << 31)) {
        srt_status rc = probe_rays(d_rays, (uint32_t)R, one_origin, one_hemisphere, st);
        if (rc) return rc;
    }
    if (one_hemisphere) {
        uint32_t *perm = nullptr;
        void *sort_mem = nullptr;
        srt_status rc = SRT_OK;
        if (!one_origin) rc = sort_rays(d_rays, (uint32_t)R, &perm, &sort_mem, st);
        ExactRaySrc src{d_rays, perm, (uint32_t)R, 1, d_rgb, nullptr, p->t_min, p->t_max, a.fkey, a.ray_id0, a.sample0};
        PacketCompositeArgs pa{};
        pa.s2 = (float)p->s2;
        pa.bg = a.bg;
        pa.kk = std::max(1, kk);
        pa.table = d_table;
        pa.tstride = p->table_slots;
        pa.ba = a;
        if (!rc)
            rc = p->rng == SRT_RNG_TABLE ? launch_composite_packet<kPacketBiasedTable>(s, src, p->mode, pa, st)
                                         : launch_composite_packet<kPacketBiasedCounter>(s, src, p->mode, pa, st);
        if (sort_mem) cudaFreeAsync(sort_mem, st);
        return rc;
    }
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
    if (p->rng != SRT_RNG_TRIG64) {
        // counter draws: 8x4 pixel blocks as packets
        ExactFrameSrc src{cam, p->width, p->height, p->passes, p->pass0, (p->width + 7) / 8, p->seed, a.fkey, d_rgb,
                          nullptr, 0.0, DBL_MAX};
        PacketCompositeArgs pa{};
        pa.s2 = (float)p->s2;
        pa.bg = a.bg;
        pa.kk = std::max(1, kk);
        pa.ba = a;
        return launch_composite_packet<kPacketBiasedCounter>(s, src, p->mode, pa, st);
    }
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
    // one-hemisphere batches (camera-like) walk as packets, coherence-sorted
    // unless they share one origin; incoherent ones per lane
    bool one_origin = false, one_hemisphere = false;
    if (R >= 4096 && (uint64_t)R < (1ull << 31)) {
        srt_status rc = probe_rays(d_rays, (uint32_t)R, one_origin, one_hemisphere, st);
        if (rc) return rc;
    }
    if (one_hemisphere) {
        uint32_t *perm = nullptr;
        void *sort_mem = nullptr;
        srt_status rc = SRT_OK;
        if (!one_origin) rc = sort_rays(d_rays, (uint32_t)R, &perm, &sort_mem, st);
        ExactRaySrc src{d_rays, perm, (uint32_t)R, 1, d_rgb, d_op, t_min, t_max, 0u, 0u, 0u};
        PacketCompositeArgs pa{};
        pa.s2 = (float)s2;
        pa.bg = make_float3((float)bg[0], (float)bg[1], (float)bg[2]);
        if (!rc) rc = launch_composite_packet<kPacketExact>(s, src, mode, pa, st);
        if (sort_mem) cudaFreeAsync(sort_mem, st);
        return rc;
    }
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
    if ((int64_t)a.width * a.height == 0) return SRT_OK;
    ExactFrameSrc src{cam, a.width, a.height, a.passes, a.pass0, (a.width + 7) / 8, a.seed, 0u, d_rgb, d_op, 0.0,
                      DBL_MAX};
    PacketCompositeArgs pa{};
    pa.s2 = a.s2;
    pa.bg = make_float3(a.bg[0], a.bg[1], a.bg[2]);
    return launch_composite_packet<kPacketExact>(s, src, a.mode, pa, st);
}

}  // namespace srt
