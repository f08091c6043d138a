// trace.cu -- stochastic BVH walk (kernels.py:312-388) over the 4-wide tree,
// for camera rays (one pass of render_stochastic, kernels.py:644-656) and
// explicit rays (trace_batch, kernels.py:527-540), plus the unclipped
// transmittance walk (kernels.py:392-432).
//
// Execution model: persistent warps.  A grid of
// SMs x resident-blocks warps pulls ray indices from one atomic counter; a
// warp refills its idle lanes (consecutive indices = an 8x4 pixel block, so
// new rays stay coherent with the warp's others) whenever at least kRefill
// lanes are idle.  Per lane the walk is "while-while" (Aila & Laine 2009):
// an inner loop visits 4-wide nodes, pushing hit children (inner nodes AND
// single-primitive leaves) far-to-near on a local stack; a leaf reached at
// the front is postponed while the lane keeps traversing, and the warp
// switches to candidate evaluation once every lane holds a postponed leaf.
// That keeps the expensive candidate code (kernels.py:139-189 + the
// acceptance draw) executing with most lanes converged.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>

#include "srt_internal.h"

namespace srt {

constexpr int kDone = kLeafEmpty;  // "no item" code for the next node / postponed leaf


template <int NS>
struct Slots {
    float t[NS];
    int id[NS];
    uint32_t key[NS];
};

template <int NS>
__device__ __forceinline__ void init_slots(Slots<NS> &sl, int nslots) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        sl.t[k] = k < nslots ? INFINITY : -INFINITY;  // inactive slots never accept, never bind the clip
        sl.id[k] = -1;
        sl.key[k] = 0;
    }
}

// Acceptance draw of slot k (kernels.py:354): counter generator or table.
template <int RNG>
__device__ __forceinline__ bool accepts(uint32_t key, const double *table, int64_t tstride, int pid, int k,
                                        float alpha) {
    if (RNG == SRT_RNG_TABLE) return __ldg(table + (int64_t)pid * tstride + k) < (double)alpha;
    return counter_u(key, (uint32_t)pid) < alpha;
}

struct WalkCfg {
    float s2;
    float sqrt_s2;
    int clip;
    const double *table;
    int64_t tstride;
};

// Optional per-walk work counters (SRT_TRACE_STATS=1): node visits, leaf
// visits, screen passes, exact evaluations, accepted updates, stack pops,
// culled pops, walks.  Accumulated per lane, flushed with one atomic each.
template <bool STATS>
struct Counters {
    __device__ __forceinline__ void add(int, unsigned) {}
    __device__ __forceinline__ void flush(unsigned long long *) {}
};
// Packet-kernel extras (warp-level, counted by lane 0): 8 visits with a leaf
// child hit, 9 leaf children hit (any lane), 10 inner children hit (any lane),
// 11 lanes with a hit per visit, 12 lanes without an accepted hit yet per
// visit, 13 job rounds, 14 visits no lane hits anything.
constexpr int kNumCounters = 16;
template <>
struct Counters<true> {
    unsigned c[kNumCounters] = {};
    __device__ __forceinline__ void add(int i, unsigned v) { c[i] += v; }
    __device__ __forceinline__ void flush(unsigned long long *out) {
        for (int i = 0; i < kNumCounters; ++i)
            if (c[i]) atomicAdd(out + i, (unsigned long long)c[i]);
        for (int i = 0; i < kNumCounters; ++i) c[i] = 0;
    }
};

template <int NS, int MODE, int RNG, bool STATS>
__device__ __forceinline__ void visit_leaf(const SceneView &s, const RayState &r, const WalkCfg &w, int slot,
                                           Slots<NS> &sl, float &far, Counters<STATS> &ct) {
    ct.add(1, 1);
    SRT_DCHECK(slot >= 0 && slot < s.n);
    const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
    float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
    // stage 1: fp32 screen -- can this candidate be accepted by any slot?
    Screen sc = screen<MODE>(r, m, a, b, w.s2, w.sqrt_s2, far);
    if (!sc.maybe) return;
    ct.add(2, 1);
    int pid = __float_as_int(b.z);
    bool need = false, band = false;
    const float alpha_lo = sc.alpha_lo();
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (sc.t_lo <= sl.t[k]) {
            const double u = RNG == SRT_RNG_TABLE ? __ldg(w.table + (int64_t)pid * w.tstride + k)
                                                  : (double)counter_u(sl.key[k], (uint32_t)pid);
            need |= u <= (double)sc.alpha_hi;
            band |= u >= (double)alpha_lo && u <= (double)sc.alpha_hi;
        }
    }
    if (!need) return;
    Cand c;
    if (sc.sure(w.s2, r.t_min, r.t_max0) && !band) {
        // decided by the screen (see packet_job): valid for certain, every
        // relevant draw below alpha_lo or above alpha_hi
        c.t = sc.t;
        c.alpha = alpha_lo;
        c.valid = 1;
    } else {
        ct.add(3, 1);
        // stage 2: exact evaluation (fp64 re-centring, kernels.py:139-189)
        c = candidate<MODE>(r, m, a, b, w.s2);
        if (!c.valid) return;
    }
    bool improved = false;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        // strict t < slot_t (kernels.py:354); an exact tie goes to the
        // smaller primitive id so the result is visit-order independent
        bool nearer = c.t < sl.t[k] || (c.t == sl.t[k] && pid < sl.id[k]);
        if (nearer && accepts<RNG>(sl.key[k], w.table, w.tstride, pid, k, c.alpha)) {
            sl.t[k] = c.t;
            sl.id[k] = pid;
            improved = true;
        }
    }
    ct.add(4, improved ? 1u : 0u);
    if (improved && w.clip) {
        // clip to the farthest slot once every slot holds a hit (kernels.py:358-364);
        // inactive slots hold -inf and never bind
        float worst = sl.t[0];
#pragma unroll
        for (int k = 1; k < NS; ++k) worst = fmaxf(worst, sl.t[k]);
        far = fminf(far, worst);
    }
}


// Per-lane traversal state (registers + a local-memory stack).
struct Walk {
    int next;  // next inner node, or kDone
    int sp;
    float far;
    int2 stk[kStackSize];  // (code, entry distance bits): one 64-bit local-memory word per entry

    float popped_t;  // entry distance of the last popped node

    template <class CT>
    __device__ __forceinline__ int pop(CT &ct) {
        while (sp > 0) {
            --sp;
            ct.add(5, 1);
            const int2 e = stk[sp];
            if (__int_as_float(e.y) <= far) {  // cull beyond the (clipped) far bound
                popped_t = __int_as_float(e.y);
                return e.x;
            }
            ct.add(6, 1);
        }
        return kDone;
    }
};

// Slab test of the 4 children of a node against [t_min, far] (closed,
// kernels.py:266-308): bit k of the result is set when child k is hit;
// key[k] = entry distance (orderable int) with k in the low 2 bits.
template <bool NONNEG = false>
__device__ __forceinline__ unsigned slab4(const RayState &r, const float4 *np, float far, int4 &kids, int key[4]) {
    float4 lox = __ldg(np), hix = __ldg(np + 1), loy = __ldg(np + 2), hiy = __ldg(np + 3), loz = __ldg(np + 4),
           hiz = __ldg(np + 5);
    kids = __ldg(reinterpret_cast<const int4 *>(np + 6));
    float lx[4] = {lox.x, lox.y, lox.z, lox.w}, hx[4] = {hix.x, hix.y, hix.z, hix.w};
    float ly[4] = {loy.x, loy.y, loy.z, loy.w}, hy[4] = {hiy.x, hiy.y, hiy.z, hiy.w};
    float lz[4] = {loz.x, loz.y, loz.z, loz.w}, hz[4] = {hiz.x, hiz.y, hiz.z, hiz.w};
    unsigned hitm = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float xa = fmaf(lx[k], r.idx, -r.oidx), xb = fmaf(hx[k], r.idx, -r.oidx);
        float ya = fmaf(ly[k], r.idy, -r.oidy), yb = fmaf(hy[k], r.idy, -r.oidy);
        float za = fmaf(lz[k], r.idz, -r.oidz), zb = fmaf(hz[k], r.idz, -r.oidz);
        float tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fmaxf(fminf(za, zb), r.t_min));
        float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), far));
        // empty slots carry inverted boxes, which min/max slab tests would see
        // as infinite: mask them by code (deriving the masks from the already
        // loaded codes beats loading the node's hint word here: 161 vs 156
        // Mrays/s on random rays)
        bool hit = tn <= tf && pick(kids, k) != kLeafEmpty;
        key[k] = NONNEG ? ((__float_as_int(tn) & ~3) | k) : ordered_key(tn, k);
        hitm |= hit ? (1u << k) : 0u;
    }
    return hitm;
}

// Visit one 4-wide node: resolve the hit leaf children (single primitives)
// on the spot -- they may clip `far` -- then descend into the nearest hit
// inner child, pushing the others far-to-near.  Returns the next inner node.
template <int NS, int MODE, int RNG, bool STATS>
__device__ __forceinline__ int visit_node(const SceneView &s, const RayState &r, const WalkCfg &w, Walk &wk,
                                          Slots<NS> &sl, int node, int *overflow, Counters<STATS> &ct) {
    ct.add(0, 1);
    int4 kids;
    int key[4];
    SRT_DCHECK(node >= 0 && node < s.num_nodes4);
    unsigned hitm = slab4(r, reinterpret_cast<const float4 *>(s.nodes4 + node), wk.far, kids, key);
    unsigned leafm = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) leafm |= pick(kids, k) < 0 ? (1u << k) : 0u;
    unsigned lm = hitm & leafm;
    while (lm) {
        int k = __ffs(lm) - 1;
        lm &= lm - 1;
        visit_leaf<NS, MODE, RNG, STATS>(s, r, w, ~pick(kids, k), sl, wk.far, ct);
    }
    unsigned im = hitm & ~leafm;
    if (!im) return wk.pop(ct);
    // order the hit inner children by entry distance
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (!(im & (1u << k))) key[k] = 0x7FFFFFFF;
    int ni = __popc(im);
    if (ni > 1) {
#define SRT_CX(a, b)                      \
    {                                     \
        int lo_ = min(key[a], key[b]);    \
        int hi_ = max(key[a], key[b]);    \
        key[a] = lo_;                     \
        key[b] = hi_;                     \
    }
        SRT_CX(0, 1) SRT_CX(2, 3) SRT_CX(0, 2) SRT_CX(1, 3) SRT_CX(1, 2)
#undef SRT_CX
        if (wk.sp + ni - 1 > kStackSize) {
            raise_flag(overflow);
            wk.sp = 0;
            return kDone;
        }
#pragma unroll
        for (int j = 3; j >= 1; --j) {
            if (j < ni) {
                float te = key_t(key[j]);
                if (te <= wk.far) {
                    wk.stk[wk.sp] = make_int2(pick(kids, key[j] & 3), __float_as_int(te));
                    ++wk.sp;
                }
            }
        }
    } else {
        int k = __ffs(im) - 1;
        key[0] = key[k];
    }
    if (key_t(key[0]) <= wk.far) return pick(kids, key[0] & 3);
    return wk.pop(ct);
}


// ---------------------------------------------------------------------------
// ray sources
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_pixel(const RenderArgs &a, int64_t lt, int tid, int &px, int &py) {
    int64_t gt = lt * a.shard_count + a.shard_index;
    int tx = (int)(gt % a.tiles_x), ty = (int)(gt / a.tiles_x);
    int w = tid >> 5, lane = tid & 31;
    px = tx * 16 + (w & 1) * 8 + (lane & 7);
    py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
}

struct CameraSource {
    static constexpr bool kCoherent = true;  // neighbouring indices = neighbouring pixels
    static constexpr bool kRayOrigin = false;  // every ray starts at cam.e
    CamD cam;
    RenderArgs a;
    int pass;
    uint32_t fkey;
    int32_t *hits;
    // Multi-pass launches (npass > 1): work item idx covers pass
    // pass + idx / unit of tile-compact pixel idx % unit; a packet never
    // straddles two passes (unit is a multiple of 256).  Results are summed
    // into acc64 in 2^-32 fixed point with integer atomics, so the sum does
    // not depend on which warp ran which (packet, pass) -- bitwise
    // deterministic -- and the whole frame is one balanced launch.
    unsigned long long *acc64;
    uint32_t npass, unit;
    // Slot group (multisample N > 8 walks as groups of <= 8 slots): this
    // launch walks slots slot0 .. slot0 + gslots - 1 of the a.nslots; slot
    // slot0 + k draws sample pass * N + slot0 + k (kernels.py:353-364 keeps
    // every slot independent, so the split never changes a result).
    uint32_t slot0;
    int gslots;
    __host__ __device__ __forceinline__ uint32_t total() const { return unit * npass; }
    // Work items are packet-major: the npass consecutive 32-item packets of
    // a group walk the same 32 pixels, one pass each, so the group's nodes
    // and primitives are fetched once into L1/L2 for all of its passes.
    __device__ __forceinline__ uint32_t item_pass(uint32_t idx) const { return (idx >> 5) % npass; }
    __device__ __forceinline__ uint32_t item_pixel(uint32_t idx) const {
        return ((idx >> 5) / npass) * 32u + (idx & 31u);
    }
    template <int NS>
    __device__ __forceinline__ bool init(uint32_t idx, RayState &r, Slots<NS> &sl) const {
        uint32_t ps = (uint32_t)pass;
        if (npass > 1) {
            const uint32_t f = item_pass(idx);
            idx = item_pixel(idx);
            ps += f;
        }
        int px, py;
        tile_pixel(a, idx >> 8, idx & 255, px, py);
        if (px >= a.width || py >= a.height) return false;
        double dx, dy, dz;
        camera_ray(cam, (uint32_t)px, (uint32_t)py, ps, a.seed, a.width, a.height, dx, dy, dz);
        init_ray(r, cam.e[0], cam.e[1], cam.e[2], dx, dy, dz, 0.0, DBL_MAX);
        init_slots<NS>(sl, gslots);
        uint32_t ray_id = (uint32_t)py * (uint32_t)a.width + (uint32_t)px;
#pragma unroll
        for (int k = 0; k < NS; ++k) sl.key[k] = walk_key(fkey, ray_id, ps * (uint32_t)a.nslots + slot0 + k);
        return true;
    }
    // fused shading (hits == nullptr): accumulate straight from the walk
    float4 *accum;
    float4 *out;
    double *rgb64, *op64;  // optional final f64 frame (e.g. mapped page-locked host memory)
    int first, last;
    // out is the row-major full frame even for a shard (multi-GPU frames
    // assembled in place: out may be a peer GPU's buffer, CUDA IPC over
    // NVLink), and the kernel ends with a system-scope fence so the stores
    // are visible to the peer before any later signal of this GPU
    int out_rowmajor, sys_fence;
    __device__ __forceinline__ void done() const {
        if (sys_fence) __threadfence_system();
    }
    template <int NS>
    __device__ __forceinline__ void finish(uint32_t idx, const Slots<NS> &sl) const {
        int32_t *h = hits + (int64_t)idx * a.nslots + slot0;
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (k < gslots) h[k] = sl.id[k];
    }
    // Walk result -> either the hit buffer (split trace/shade) or, fused, the
    // SH colour of every slot's hit on this ray's direction plus background
    // for misses, accumulated exactly as k_shade_pass does (kernels.py:657-673).
    // f64v / f64pix (packet kernel): a pixel bound for the f64 frame is
    // returned there instead of stored (store_f64_packet writes the warp's)
    template <int NS>
    __device__ __forceinline__ void finish_shaded(uint32_t idx, const Slots<NS> &sl, const SceneView &s, float fx,
                                                  float fy, float fz, double *f64v = nullptr,
                                                  int64_t *f64pix = nullptr) const {
        if (hits) {
            finish<NS>(idx, sl);
            return;
        }
        float r = 0.f, g = 0.f, b = 0.f, o = 0.f;
        for (int k = 0; k < NS && k < gslots; ++k) {
            int pid = sl.id[k];
            if (pid >= 0) {
                SRT_DCHECK(pid < s.n);
                float3 c = sh_color(s.sh, s.sh_k, s.sh_deg, pid, fx, fy, fz);
                r += c.x;
                g += c.y;
                b += c.z;
                o += 1.0f;
            } else {
                r += a.bg[0];
                g += a.bg[1];
                b += a.bg[2];
            }
        }
        if (acc64) {
            unsigned long long *q = acc64 + (int64_t)item_pixel(idx) * 4;
            atomicAdd(q + 0, __float2ull_rn(r * 4294967296.0f));
            atomicAdd(q + 1, __float2ull_rn(g * 4294967296.0f));
            atomicAdd(q + 2, __float2ull_rn(b * 4294967296.0f));
            atomicAdd(q + 3, (unsigned long long)(unsigned)o << 32);  // hit count in the high word
            return;
        }
        float4 acc = first ? make_float4(0.f, 0.f, 0.f, 0.f) : accum[idx];
        acc.x += r;
        acc.y += g;
        acc.z += b;
        acc.w += o;
        if (last) {
            float inv = 1.0f / ((float)a.passes * (float)a.nslots);
            int px, py;
            tile_pixel(a, idx >> 8, idx & 255, px, py);
            if (rgb64) {
                // the resolved frame straight into its final (H,W,3)+(H,W) f64
                // layout -- over PCIe when it is mapped host memory, so the
                // device->host transfer overlaps the rest of the walk
                int64_t pix = (int64_t)py * a.width + px;
                if (f64v) {  // the packet kernel stores the warp's pixels together
                    f64v[0] = (double)(acc.x * inv);
                    f64v[1] = (double)(acc.y * inv);
                    f64v[2] = (double)(acc.z * inv);
                    f64v[3] = (double)(acc.w * inv);
                    *f64pix = pix;
                    return;
                }
                rgb64[pix * 3 + 0] = (double)(acc.x * inv);
                rgb64[pix * 3 + 1] = (double)(acc.y * inv);
                rgb64[pix * 3 + 2] = (double)(acc.z * inv);
                op64[pix] = (double)(acc.w * inv);
                return;
            }
            int64_t oidx = (a.shard_count > 1 && !out_rowmajor) ? (int64_t)idx : (int64_t)py * a.width + px;
            out[oidx] = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        } else {
            accum[idx] = acc;
        }
    }
};

struct ArraySource {
    static constexpr bool kCoherent = false;
    static constexpr bool kRayOrigin = true;
    const double *rays;  // (R, 6)
    const uint32_t *perm;  // optional processing order (sorted rays); results keyed by the original index
    uint32_t R;
    double t_min, t_max;
    int nslots;
    uint32_t fkey, ray_id0, sample0;
    float *out_t;
    int32_t *out_id;
    int ostride;  // output row length (nslots, or the full slot count of a slot group)
    __host__ __device__ __forceinline__ uint32_t total() const { return R; }
    template <int NS>
    __device__ __forceinline__ bool init(uint32_t idx, RayState &r, Slots<NS> &sl) const {
        if (perm) idx = __ldg(perm + idx);
        const double *q = rays + (int64_t)idx * 6;
        init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
        init_slots<NS>(sl, nslots);
#pragma unroll
        for (int k = 0; k < NS; ++k) sl.key[k] = walk_key(fkey, ray_id0 + idx, sample0 + (uint32_t)k);
        return true;
    }
    template <int NS>
    __device__ __forceinline__ void finish(uint32_t idx, const Slots<NS> &sl) const {
        if (perm) idx = __ldg(perm + idx);
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (k < nslots) {
                out_t[(int64_t)idx * ostride + k] = sl.id[k] >= 0 ? sl.t[k] : INFINITY;
                out_id[(int64_t)idx * ostride + k] = sl.id[k];
            }
    }
    template <int NS>
    __device__ __forceinline__ void finish_shaded(uint32_t idx, const Slots<NS> &sl, const SceneView &, float, float,
                                                  float, double * = nullptr, int64_t * = nullptr) const {
        finish<NS>(idx, sl);
    }
    __device__ __forceinline__ void done() const {}
};

// Explicit rays that point into one hemisphere (camera batches, the
// reference's parallel jittered rays, validate.py:36-43), walked as warp
// packets: neighbouring indices (after the optional sort) share nodes.  The
// per-lane origin and 1/|d|^2 travel through shared memory to the leaf jobs.
struct PacketArraySource : ArraySource {
    static constexpr bool kCoherent = true;
    CamD cam;              // unused (the packet kernel reads per-lane origins)
    float f_tmin, f_tmax;  // the candidate interval as init_ray rounds it
};

// ---------------------------------------------------------------------------
// persistent kernel
// ---------------------------------------------------------------------------
constexpr int kTraceThreads = 128;

// REFILL: refill a warp once this many lanes are idle (32 = whole-warp
// granularity).
template <int NS, int MODE, int RNG, class Src, int REFILL, bool STATS>
__global__ void __launch_bounds__(kTraceThreads) k_trace(SceneView s, Src src, WalkCfg w, uint32_t *work,
                                                          int *overflow, unsigned long long *stats) {
    Counters<STATS> ct;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t total = src.total();
    RayState r;
    Slots<NS> sl;
    Walk wk;
    bool active = false;
    bool exhausted = false;
    uint32_t idx = 0;
    while (true) {
        unsigned idle = __ballot_sync(FULL, !active);
        if (!exhausted && __popc(idle) >= REFILL) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(work, (uint32_t)__popc(idle));
            base = __shfl_sync(FULL, base, 0);
            if (base + (uint32_t)__popc(idle) >= total) exhausted = true;
            if (!active) {
                uint32_t my = base + (uint32_t)__popc(idle & ((1u << lane) - 1u));
                if (my < total && src.template init<NS>(my, r, sl)) {
                    idx = my;
                    active = true;
                    wk.sp = 0;
                    wk.far = r.t_max0;
                    wk.next = s.num_nodes4 > 0 ? 0 : kDone;
                }
            }
        } else if (exhausted && idle == FULL) {
            ct.flush(stats);
            break;
        }
        if (active) {
            // one node visit per round, so finished lanes are refilled while
            // the rest of the warp keeps walking
            if (wk.next >= 0) wk.next = visit_node<NS, MODE, RNG, STATS>(s, r, w, wk, sl, wk.next, overflow, ct);
            if (wk.next < 0) {
                ct.add(7, 1);
                src.template finish_shaded<NS>(idx, sl, s, r.fdx, r.fdy, r.fdz);
                active = false;
            }
        }
    }
    release_counter(work);
}

// ---------------------------------------------------------------------------
// Warp-cooperative kernel.  Each lane walks its own ray through the inner
// nodes, but leaf work is compacted across the warp: every round, the hit
// leaf children of all 32 lanes go into a warp queue in shared memory and
// are screened by all 32 lanes together (ballot/prefix-sum compaction), with
// the owner's ray read from shared memory.  Slot updates are 64-bit
// shared-memory atomicMin of (orderable t, prim id): the closest accepted
// hit, ties to the smaller id -- exactly the order-free semantics of
// kernels.py:353-357.
// ---------------------------------------------------------------------------

template <int NS, int MODE, int RNG, bool STATS>
__device__ __forceinline__ void leaf_job(const SceneView &s, const RayState &r, const WalkCfg &w, int slot,
                                         unsigned long long *best, const uint32_t *keys, float far,
                                         Counters<STATS> &ct) {
    ct.add(1, 1);
    SRT_DCHECK(slot >= 0 && slot < s.n);
    const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
    float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
    Screen sc = screen<MODE>(r, m, a, b, w.s2, w.sqrt_s2, far);
    if (!sc.maybe) return;
    ct.add(2, 1);
    int pid = __float_as_int(b.z);
    bool need = false, band = false;
    const float alpha_lo = sc.alpha_lo();
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (sc.t_lo <= unpack_t(best[k])) {
            const double u = RNG == SRT_RNG_TABLE ? __ldg(w.table + (int64_t)pid * w.tstride + k)
                                                  : (double)counter_u(keys[k], (uint32_t)pid);
            need |= u <= (double)sc.alpha_hi;
            band |= u >= (double)alpha_lo && u <= (double)sc.alpha_hi;
        }
    }
    if (!need) return;
    Cand c;
    if (sc.sure(w.s2, r.t_min, r.t_max0) && !band) {
        c.t = sc.t;  // decided by the screen (see packet_job)
        c.alpha = alpha_lo;
        c.valid = 1;
    } else {
        ct.add(3, 1);
        c = candidate<MODE>(r, m, a, b, w.s2);
        if (!c.valid) return;
    }
    unsigned long long key = pack_hit(c.t, pid);
#pragma unroll
    for (int k = 0; k < NS; ++k)
        if (key < best[k] && accepts<RNG>(keys[k], w.table, w.tstride, pid, k, c.alpha)) {
            atomicMin(best + k, key);
            ct.add(4, 1);
        }
}


// Leaf job of the packet kernel: screen on the owner's fp32 direction and
// the shared camera origin; the exact fp64 stage rebuilds the owner's ray
// from its fp64 direction only when the screen cannot decide.
// RO (explicit-ray packets): the owner's fp64 origin and 1/|d|^2 come from
// ro[0..3] and the candidate interval from sr, instead of the camera's.
template <int NS, int MODE, bool STATS, bool RO = false>
__device__ __forceinline__ void packet_job(const SceneView &s, const CamD &cam, const ScreenRay &sr, const double *dd,
                                           const WalkCfg &w, int slot, unsigned long long *best,
                                           const uint32_t *keys, float far, Counters<STATS> &ct,
                                           const double *ro = nullptr) {
    ct.add(1, 1);
    SRT_DCHECK(slot >= 0 && slot < s.n);
    const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
    float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
    Screen sc = screen<MODE>(sr, m, a, b, w.s2, w.sqrt_s2, far);
    if (!sc.maybe) return;
    ct.add(2, 1);
    int pid = __float_as_int(b.z);
    // single-slot walks draw once and reuse the draw in the exact stage
    const float u0 = NS == 1 ? counter_u(keys[0], (uint32_t)pid) : 0.0f;
    bool need = false;
#pragma unroll
    for (int k = 0; k < NS; ++k)
        if (sc.t_lo <= unpack_t(best[k]))
            need |= (NS == 1 ? u0 : counter_u(keys[k], (uint32_t)pid)) <= sc.alpha_hi;
    if (!need) return;
    if (sc.sure(w.s2, sr.t_min, sr.t_max0)) {
        const float alpha_lo = sc.alpha_lo();
        // Valid for certain and every draw outside [alpha_lo, alpha_hi]: the
        // screen decides (u < alpha_lo <= alpha: accepted, at the screen's
        // depth, ~1e-6 from the exact one).  Only draws inside the error band
        // -- a few in 1e4 -- need the exact stage, which keeps the divergent
        // fp64 code off the common path.
        const unsigned long long key = pack_hit(sc.t, pid);
        bool band = false;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const float u = NS == 1 ? u0 : counter_u(keys[k], (uint32_t)pid);
            if (u < alpha_lo) {
                if (key < best[k]) {
                    atomicMin(best + k, key);
                    ct.add(4, 1);
                }
            } else {
                band |= u <= sc.alpha_hi;
            }
        }
        if (!band) return;
    }
    ct.add(3, 1);
    // the camera ray's fields the exact candidate reads; camera directions are
    // unit in fp64 to an ulp, and 1/|d|^2 only sets the re-centring point,
    // so inv_dd = 1 (as in the screen) changes the fp32 result by < 1e-15
    ExactRay r;
    r.dx = dd[0], r.dy = dd[1], r.dz = dd[2];
    r.fdx = (float)r.dx, r.fdy = (float)r.dy, r.fdz = (float)r.dz;
    if constexpr (RO) {
        r.ox = ro[0], r.oy = ro[1], r.oz = ro[2];
        r.inv_dd = ro[3];
        r.t_min = sr.t_min, r.t_max0 = sr.t_max0;
    } else {
        r.ox = cam.e[0], r.oy = cam.e[1], r.oz = cam.e[2];
        r.inv_dd = 1.0;
        r.t_min = 0.0f, r.t_max0 = INFINITY;
    }
    // one re-centring: the second (peak) re-centring only matters for extreme
    // anisotropy and would raise this loop's register count by ~10
    Cand c = candidate<MODE, ExactRay, false>(r, m, a, b, w.s2);
    if (!c.valid) return;
    unsigned long long key = pack_hit(c.t, pid);
#pragma unroll
    for (int k = 0; k < NS; ++k)
        if (key < best[k] && (NS == 1 ? u0 : counter_u(keys[k], (uint32_t)pid)) < c.alpha) {
            atomicMin(best + k, key);
            ct.add(4, 1);
        }
}

// Inner children of a visited node: descend into the nearest hit one, push
// the others far-to-near.  Returns the next node (or a popped one).
template <bool STATS>
__device__ __forceinline__ int descend(Walk &wk, const int4 &kids, int key[4], unsigned im, float &next_t,
                                       int *overflow, Counters<STATS> &ct) {
    if (!im) {
        int n = wk.pop(ct);
        next_t = wk.popped_t;
        return n;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (!(im & (1u << k))) key[k] = 0x7FFFFFFF;
    int ni = __popc(im);
    if (ni > 1) {
#define SRT_CX(a, b)                      \
    {                                     \
        int lo_ = min(key[a], key[b]);    \
        int hi_ = max(key[a], key[b]);    \
        key[a] = lo_;                     \
        key[b] = hi_;                     \
    }
        SRT_CX(0, 1) SRT_CX(2, 3) SRT_CX(0, 2) SRT_CX(1, 3) SRT_CX(1, 2)
#undef SRT_CX
        if (wk.sp + ni - 1 > kStackSize) {
            raise_flag(overflow);
            wk.sp = 0;
            return kDone;
        }
#pragma unroll
        for (int j = 3; j >= 1; --j) {
            if (j < ni) {
                wk.stk[wk.sp] = make_int2(pick(kids, key[j] & 3), __float_as_int(key_t(key[j])));
                ++wk.sp;
            }
        }
    } else {
        key[0] = key[__ffs(im) - 1];
    }
    next_t = key_t(key[0]);
    return pick(kids, key[0] & 3);
}

template <int NS, int MODE, int RNG, class Src, bool STATS, int REFILL = 32>
__global__ void __launch_bounds__(kTraceThreads) k_trace_coop(SceneView s, Src src, WalkCfg w, uint32_t *work,
                                                               int *overflow, unsigned long long *stats) {
    constexpr int W = kTraceThreads / 32;
    __shared__ RayState sray[W][32];
    __shared__ unsigned long long sbest[W][32][NS];
    __shared__ uint32_t skey[W][32][NS];
    __shared__ float sfar[W][32];
    __shared__ int sjob[W][128];
    __shared__ unsigned char sown[W][128];
    const unsigned FULL = 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t total = src.total();
    Counters<STATS> ct;
    RayState r;
    Slots<NS> sl;
    Walk wk;
    float next_t = 0.f;
    bool active = false;
    bool exhausted = false;
    uint32_t idx = 0;
    const unsigned lt = (1u << lane) - 1u;
    while (true) {
        const unsigned idle = __ballot_sync(FULL, !active);
        if (exhausted && idle == FULL) break;
        // refill the idle lanes once REFILL of them are free (32: whole-warp refills)
        if (!exhausted && __popc(idle) >= REFILL) {
            const uint32_t nidle = (uint32_t)__popc(idle);
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(work, nidle);
            base = __shfl_sync(FULL, base, 0);
            if (base + nidle >= total) exhausted = true;
            const uint32_t my = base + (uint32_t)__popc(idle & lt);
            if (!active && my < total && src.template init<NS>(my, r, sl)) {
                idx = my;
                active = true;
                wk.sp = 0;
                wk.far = r.t_max0;
                wk.next = s.num_nodes4 > 0 ? 0 : kDone;
                next_t = r.t_min;
                sray[wid][lane] = r;
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    sbest[wid][lane][k] = pack_hit(sl.t[k], -1);
                    skey[wid][lane][k] = sl.key[k];
                }
            }
            if (__ballot_sync(FULL, active) == 0) continue;
        }
        // ---- inner traversal step (per lane) ----
        unsigned lm = 0;
        int4 kids = make_int4(kDone, kDone, kDone, kDone);
        if (active && wk.next >= 0) {
            ct.add(0, 1);
            int key[4];
            unsigned hitm = slab4(r, reinterpret_cast<const float4 *>(s.nodes4 + wk.next), wk.far, kids, key);
            unsigned leafm = (kids.x < 0 ? 1u : 0u) | (kids.y < 0 ? 2u : 0u) | (kids.z < 0 ? 4u : 0u) |
                             (kids.w < 0 ? 8u : 0u);
            lm = hitm & leafm;
            wk.next = descend<STATS>(wk, kids, key, hitm & ~leafm, next_t, overflow, ct);
        }
        // ---- warp-compacted leaf jobs ----
        int cnt = __popc(lm);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        int njobs = __shfl_sync(FULL, incl, 31);
        if (njobs) {
            int off = incl - cnt;
            if (lm & 1u) { sjob[wid][off] = ~kids.x; sown[wid][off] = (unsigned char)lane; ++off; }
            if (lm & 2u) { sjob[wid][off] = ~kids.y; sown[wid][off] = (unsigned char)lane; ++off; }
            if (lm & 4u) { sjob[wid][off] = ~kids.z; sown[wid][off] = (unsigned char)lane; ++off; }
            if (lm & 8u) { sjob[wid][off] = ~kids.w; sown[wid][off] = (unsigned char)lane; ++off; }
            sfar[wid][lane] = wk.far;
            __syncwarp();
            for (int jb = 0; jb < njobs; jb += 32) {
                int j = jb + lane;
                if (j < njobs) {
                    int o = sown[wid][j];
                    leaf_job<NS, MODE, RNG, STATS>(s, sray[wid][o], w, sjob[wid][j], sbest[wid][o], skey[wid][o],
                                                    sfar[wid][o], ct);
                }
            }
            __syncwarp();
            if (active && w.clip) {
                // clip to the farthest slot once every slot holds a hit (kernels.py:358-364)
                float worst = unpack_t(sbest[wid][lane][0]);
#pragma unroll
                for (int k = 1; k < NS; ++k) worst = fmaxf(worst, unpack_t(sbest[wid][lane][k]));
                wk.far = fminf(wk.far, worst);
            }
        }
        if (active) {
            if (wk.next >= 0 && next_t > wk.far) {
                wk.next = wk.pop(ct);
                next_t = wk.popped_t;
            }
            if (wk.next < 0) {
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    unsigned long long v = sbest[wid][lane][k];
                    sl.id[k] = (int)(unsigned)v;
                    sl.t[k] = unpack_t(v);
                }
                src.template finish_shaded<NS>(idx, sl, s, r.fdx, r.fdy, r.fdz);
                ct.add(7, 1);
                active = false;
            }
        }
    }
    ct.flush(stats);
    release_counter(work);
}

// ---------------------------------------------------------------------------
// Warp-packet kernel (camera rays): the 32 rays of an 8x4 pixel block walk
// the tree TOGETHER.  Node addresses, the stack and the visit order are
// warp-uniform (one 128-B node fetch serves the warp); every lane slab-tests
// the node's children against its own ray and far bound; the warp descends
// into every child that any lane hits, nearest (warp-min entry) first, and
// culls a popped node when its warp-min entry lies beyond every lane's far.
// Leaf work is compacted across the warp exactly as in k_trace_coop.
//
// The packet reads the copy of the tree laid out for its direction octant
// (SceneView::nodes8): per axis the near planes of the 4 children first, the
// far planes second, so a lane's slab test is 6 FMAs, a 3-way max and a 3-way
// min -- no per-axis min/max to sort the two planes.  A packet whose lanes do
// not all share the octant (a pixel block straddling an axis of the view)
// takes the order-agnostic min/max slab on the same record.  Child handling
// is driven by warp-uniform masks: one OR-reduction of the lanes' hit masks,
// one ballot per hit leaf child, one min-reduction per inner child when more
// than one must be ordered.
// ---------------------------------------------------------------------------
// BATCH: leaf jobs are run once at least BATCH are queued; MINB: minimum
// resident blocks per SM requested from the register allocator.
// The f64 frame pixels of a packet (an 8x4 block when the packet is whole):
// staged in shared memory and written as 16-byte words, each row's 8 pixels
// one contiguous 192 B (rgb) + 64 B (opacity) run -- full PCIe write
// payloads into mapped host memory instead of 8-byte stores at a 24-byte
// stride.  Partial or unaligned packets store per lane.
template <class Src>
__device__ __forceinline__ void store_f64_packet(const Src &src, bool f64, const double v[4], int64_t pix,
                                                 double *stage_rgb, double *stage_op) {
    if constexpr (!Src::kRayOrigin) {
        const unsigned FULL = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const unsigned m = __ballot_sync(FULL, f64);
        if (!m) return;
        double *rgb = src.rgb64, *op = src.op64;
        const int64_t W = src.a.width;
        const int64_t pix0 = __shfl_sync(FULL, pix, 0);
        const bool block = m == FULL && pix == pix0 + (int64_t)(lane >> 3) * W + (lane & 7);
        const bool aligned = ((((uintptr_t)rgb | (uintptr_t)op) & 15u) == 0) && !((pix0 | W) & 1);
        if (__all_sync(FULL, block) && aligned) {
            stage_rgb[lane * 3] = v[0];
            stage_rgb[lane * 3 + 1] = v[1];
            stage_rgb[lane * 3 + 2] = v[2];
            stage_op[lane] = v[3];
            __syncwarp();
            for (int g = lane; g < 48; g += 32) {  // 4 rows x 12 double2 of rgb
                const int r = g / 12, q = g - r * 12;
                const double2 w = *reinterpret_cast<const double2 *>(stage_rgb + r * 24 + 2 * q);
                *reinterpret_cast<double2 *>(rgb + (pix0 + r * W) * 3 + 2 * q) = w;
            }
            if (lane < 16) {  // 4 rows x 4 double2 of opacity
                const int r = lane >> 2, q = lane & 3;
                const double2 w = *reinterpret_cast<const double2 *>(stage_op + r * 8 + 2 * q);
                *reinterpret_cast<double2 *>(op + pix0 + r * W + 2 * q) = w;
            }
            __syncwarp();
        } else if (f64) {
            rgb[pix * 3] = v[0];
            rgb[pix * 3 + 1] = v[1];
            rgb[pix * 3 + 2] = v[2];
            op[pix] = v[3];
        }
    }
}

#ifdef SRT_PACKET_CLOCKS
// Per-packet timing (experiments only, -DSRT_PACKET_CLOCKS via
// tools/build_variant.sh): start (globaltimer ns) and duration | smid << 48
// of work packet base/32 of the last k_trace_packet launch.
constexpr uint32_t kClockSlots = 1u << 20;
__device__ uint64_t g_packet_clk[2 * kClockSlots];
__device__ uint32_t g_packet_cnt[4 * kClockSlots];  // node visits, leaf jobs, pops, mixed | lanes hit << 1
}  // namespace srt
extern "C" int srt_exp_packet_clocks(uint64_t *out, int n) {
    if (n > (int)srt::kClockSlots) n = (int)srt::kClockSlots;
    return (int)cudaMemcpyFromSymbol(out, srt::g_packet_clk, sizeof(uint64_t) * 2 * (size_t)n);
}
extern "C" int srt_exp_packet_counts(uint32_t *out, int n) {
    if (n > (int)srt::kClockSlots) n = (int)srt::kClockSlots;
    return (int)cudaMemcpyFromSymbol(out, srt::g_packet_cnt, sizeof(uint32_t) * 4 * (size_t)n);
}
namespace srt {
#endif
template <int NS, int MODE, int RNG, class Src, bool STATS, int BATCH = 32, int MINB = 1>
__global__ void __launch_bounds__(kTraceThreads, MINB) k_trace_packet(SceneView s, Src src, WalkCfg w, uint32_t *work,
                                                                       int *overflow, unsigned long long *stats) {
    constexpr int W = kTraceThreads / 32;
    constexpr int PSTACK = 128;
    __shared__ float4 sdir[W][32];      // fp32 direction + far bound of each lane's ray
    __shared__ __align__(16) double sdd[W][32][3];  // fp64 direction (exact stage); f64 pixel staging
    __shared__ __align__(16) unsigned long long sbest[W][32][NS];
    __shared__ uint32_t skey[W][32][NS];
    __shared__ uint32_t sjob[W][BATCH + 128];  // leaf job: (slot << 5) | owner lane
    __shared__ int2 sstk[W][PSTACK];  // (node, warp-min entry key): one 64-bit word per entry
    // explicit-ray packets (Src::kRayOrigin): each lane's own origin
    constexpr bool RO = Src::kRayOrigin;
    __shared__ float4 sorg[RO ? W : 1][32];    // fp32 origin + max |o_i|
    __shared__ double sdo[RO ? W : 1][32][4];  // fp64 origin + 1/|d|^2 (exact stage)
    const unsigned FULL = 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t total = src.total();
    const float cfox = (float)src.cam.e[0], cfoy = (float)src.cam.e[1], cfoz = (float)src.cam.e[2];
    const float comag = fmaxf(fabsf(cfox), fmaxf(fabsf(cfoy), fabsf(cfoz)));
    Counters<STATS> ct;
    RayState r;
    Slots<NS> sl;
    while (true) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(work, 32u);
        base = __shfl_sync(FULL, base, 0);
        if (base >= total) break;
#ifdef SRT_PACKET_CLOCKS
        uint64_t clk_t0 = 0;
        uint32_t pk_visits = 0, pk_jobs = 0, pk_pops = 0;
        if (lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk_t0));
#endif
        uint32_t idx = base + (uint32_t)lane;
        bool valid = idx < total && src.template init<NS>(idx, r, sl);
        float far;
        if (valid) {
            far = r.t_max0;
            sdd[wid][lane][0] = r.dx;
            sdd[wid][lane][1] = r.dy;
            sdd[wid][lane][2] = r.dz;
            if constexpr (RO) {
                sorg[wid][lane] = make_float4(r.fox, r.foy, r.foz, r.omag);
                sdo[wid][lane][0] = r.ox;
                sdo[wid][lane][1] = r.oy;
                sdo[wid][lane][2] = r.oz;
                sdo[wid][lane][3] = r.inv_dd;
            }
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                sbest[wid][lane][k] = pack_hit(sl.t[k], -1);
                skey[wid][lane][k] = sl.key[k];
            }
            ct.add(7, 1);
        } else {
            init_ray(r, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0);
            far = -INFINITY;  // hits nothing
        }
        // direction octant of the packet, from the signs of the reciprocal
        // directions the slab uses (a -0 component counts as negative)
        const unsigned vm = __ballot_sync(FULL, valid);
        const unsigned nx_m = __ballot_sync(FULL, valid && signbit(r.idx));
        const unsigned ny_m = __ballot_sync(FULL, valid && signbit(r.idy));
        const unsigned nz_m = __ballot_sync(FULL, valid && signbit(r.idz));
        const int oct = (nx_m ? 1 : 0) | (ny_m ? 2 : 0) | (nz_m ? 4 : 0);
        const bool mixed = (nx_m && nx_m != vm) || (ny_m && ny_m != vm) || (nz_m && nz_m != vm);
        // node records addressed as one unsigned 32-bit index from the octant
        // copies' base (8 x num_nodes4 < 2^32): one wide multiply-add per visit
        // (seed mean 1.692 -> 1.654 ms over 64-bit pointer arithmetic)
        const uint32_t obase = (uint32_t)oct * (uint32_t)s.num_nodes4;
        int sp = 0;
        int njobs = 0;  // leaf jobs queued for the warp (processed in batches of >= BATCH)
        int node = (s.num_nodes4 > 0 && vm) ? 0 : kDone;
        auto run_jobs = [&]() {
            sdir[wid][lane] = make_float4(r.fdx, r.fdy, r.fdz, far);
            __syncwarp();
            // N <= 2: mid-walk flushes run whole rounds of 32 jobs only; the
            // rest stay queued (moved to the front) for the next flush or the
            // walk's end (rounds 84% -> ~100% full; N=1 seed mean 1.678 ->
            // 1.648 ms at 32-job batches, N=2 +1.7%; N=4 / N=8 lose 1.4 / 1.7%:
            // their clip waits on more slots, so they flush everything)
            constexpr bool kFullRounds = NS <= 2;
            const bool walk_end = node == kDone && sp == 0;
            const int nrun = (walk_end || !kFullRounds) ? njobs : (njobs & ~31);
            for (int jb = 0; jb < nrun; jb += 32) {
                if (lane == 0) ct.add(13, 1);
                int j = jb + lane;
                if (j < nrun) {
                    const uint32_t job = sjob[wid][j];
                    const int o = (int)(job & 31u), slot = (int)(job >> 5);
                    float4 dv = sdir[wid][o];
                    ScreenRay sr;
                    sr.fdx = dv.x; sr.fdy = dv.y; sr.fdz = dv.z;
                    if constexpr (RO) {
                        float4 og = sorg[wid][o];
                        sr.fox = og.x; sr.foy = og.y; sr.foz = og.z; sr.omag = og.w;
                        sr.inv_dd = sdo[wid][o][3];
                        sr.t_min = src.f_tmin;
                        sr.t_max0 = src.f_tmax;
                        packet_job<NS, MODE, STATS, true>(s, src.cam, sr, sdd[wid][o], w, slot, sbest[wid][o],
                                                          skey[wid][o], dv.w, ct, sdo[wid][o]);
                    } else {
                        sr.fox = cfox; sr.foy = cfoy; sr.foz = cfoz; sr.omag = comag;
                        sr.inv_dd = 1.0;  // camera directions are unit in fp64
                        sr.t_min = 0.0f;
                        sr.t_max0 = INFINITY;
                        packet_job<NS, MODE, STATS>(s, src.cam, sr, sdd[wid][o], w, slot, sbest[wid][o], skey[wid][o],
                                                    dv.w, ct);
                    }
                }
            }
            __syncwarp();
            {
                const int left = njobs - nrun;  // < 32
                const uint32_t v = lane < left ? sjob[wid][nrun + lane] : 0u;
                __syncwarp();
                if (lane < left) sjob[wid][lane] = v;
                __syncwarp();
                njobs = left;
            }
            if (valid && w.clip) {
                // clip to the farthest slot once every slot holds a hit (kernels.py:358-364)
                float worst = unpack_t(sbest[wid][lane][0]);
#pragma unroll
                for (int k = 1; k < NS; ++k) worst = fmaxf(worst, unpack_t(sbest[wid][lane][k]));
                far = fminf(far, worst);
            }
        };
        while (true) {
            // the one job-flush site (a single inlined copy of the job code): a
            // full batch, or the end of the walk
            if (njobs >= BATCH || (node == kDone && sp == 0 && njobs)) run_jobs();
            if (node == kDone) {
                if (sp == 0) break;
                // pop, culling entries beyond every lane's far bound
                int maxfar = __reduce_max_sync(FULL, __float_as_int(far));  // far >= 0, or -inf when idle
                __syncwarp();
                while (sp > 0) {
                    --sp;
                    if (lane == 0) ct.add(5, 1);
#ifdef SRT_PACKET_CLOCKS
                    ++pk_pops;
#endif
                    const int2 e = sstk[wid][sp];
                    if (e.y <= maxfar) {
                        node = e.x;
                        SRT_DCHECK(node >= 0 && node < s.num_nodes4);
                        break;
                    }
                    if (lane == 0) ct.add(6, 1);
                }
                if (node == kDone) continue;  // all culled: flush what is queued, then finish
            }
            if (lane == 0) ct.add(0, 1);
#ifdef SRT_PACKET_CLOCKS
            ++pk_visits;
#endif
            SRT_DCHECK(node >= 0 && node < s.num_nodes4);
            const float4 *np = reinterpret_cast<const float4 *>(s.nodes8 + (obase + (uint32_t)node));
            // near / far planes of the 4 children along the packet's octant
            const float4 ax = __ldg(np), bx = __ldg(np + 1), ay = __ldg(np + 2), by = __ldg(np + 3),
                         az = __ldg(np + 4), bz = __ldg(np + 5);
            // lane j holds child code j & 3 (one 4-byte load per lane); a child
            // code for a warp-uniform k is then one shuffle instead of the
            // three selects of sel4 (seed mean 1.453 -> 1.422 ms)
            const int mykid = __ldg(reinterpret_cast<const int *>(np + 6) + (lane & 3));
#define SRT_KID(k) __shfl_sync(FULL, mykid, (k))
            const unsigned hint = (unsigned)__ldg(reinterpret_cast<const int *>(np + 7));
            const float pax[4] = {ax.x, ax.y, ax.z, ax.w}, pbx[4] = {bx.x, bx.y, bx.z, bx.w};
            const float pay[4] = {ay.x, ay.y, ay.z, ay.w}, pby[4] = {by.x, by.y, by.z, by.w};
            const float paz[4] = {az.x, az.y, az.z, az.w}, pbz[4] = {bz.x, bz.y, bz.z, bz.w};
            unsigned hitm = 0;
            float tn4[4];  // entry distances (ordering keys are built only when inner children compete)
            if (!mixed) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // entry not clamped to t_min: a box wholly before t_min may
                    // pass (conservative), keys of boxes behind the origin sort first
                    const float tn = fmaxf(fmaxf(fmaf(pax[k], r.idx, -r.oidx), fmaf(pay[k], r.idy, -r.oidy)),
                                           fmaf(paz[k], r.idz, -r.oidz));
                    const float tf = fminf(fminf(fminf(fmaf(pbx[k], r.idx, -r.oidx), fmaf(pby[k], r.idy, -r.oidy)),
                                                 fmaf(pbz[k], r.idz, -r.oidz)), far);
                    hitm |= tn <= tf ? (1u << k) : 0u;
                    tn4[k] = tn;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float xa = fmaf(pax[k], r.idx, -r.oidx), xb = fmaf(pbx[k], r.idx, -r.oidx);
                    const float ya = fmaf(pay[k], r.idy, -r.oidy), yb = fmaf(pby[k], r.idy, -r.oidy);
                    const float za = fmaf(paz[k], r.idz, -r.oidz), zb = fmaf(pbz[k], r.idz, -r.oidz);
                    const float tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fmaxf(fminf(za, zb), r.t_min));
                    const float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), far));
                    hitm |= tn <= tf ? (1u << k) : 0u;
                    tn4[k] = tn;
                }
            }
            const unsigned validm = hint & 15u, leafm = (hint >> 4) & 15u;
            hitm &= validm;  // empty slots: inverted boxes
            node = kDone;
            if constexpr (STATS) {
                const unsigned anyh = __reduce_or_sync(FULL, hitm);
                const unsigned hl = __ballot_sync(FULL, hitm != 0u);
                const unsigned nohit = __ballot_sync(FULL, valid && far == r.t_max0);
                if (lane == 0) {
                    ct.add(8, (anyh & leafm) ? 1u : 0u);
                    ct.add(9, __popc(anyh & leafm));
                    ct.add(10, __popc(anyh & ~leafm));
                    ct.add(11, __popc(hl));
                    ct.add(12, __popc(nohit));
                    ct.add(14, anyh ? 0u : 1u);
                }
            }
            // leaf children any lane hits: one ballot each compacts the hitting
            // lanes into the job queue (jobs run in batches at the loop top:
            // deferring them only delays the far-bound clip, never a result)
            const unsigned any = __reduce_or_sync(FULL, hitm);
            const unsigned lh = hitm & leafm;
            for (unsigned al = any & leafm; al; al &= al - 1) {
                const int k = __ffs(al) - 1;
                const bool h = (lh >> k) & 1u;
                const unsigned bm = __ballot_sync(FULL, h);
                {
                    // predicated shared store (no divergent branch to reconverge):
                    // 1.787 -> 1.762 ms seed mean
                    const uint32_t code = ((uint32_t)~SRT_KID(k) << 5) | (uint32_t)lane;
                    SRT_DCHECK(!h || njobs + __popc(bm & lt) < BATCH + 128);
                    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(&sjob[wid][njobs + __popc(bm & lt)]);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}"
                                 :: "r"(addr), "r"(code), "r"((uint32_t)h) : "memory");
                }
                njobs += __popc(bm);
#ifdef SRT_PACKET_CLOCKS
                pk_jobs += __popc(bm);
#endif
            }
            // inner children any lane hits: descend into the nearest (warp-min
            // entry), push the others far-to-near with their warp-min entries
            const unsigned ih = hitm & ~leafm;
            const unsigned ai = any & ~leafm;
            if (ai) {
                if (!(ai & (ai - 1))) {
                    node = SRT_KID(__ffs(ai) - 1);  // one: nothing to order or push
                } else {
                    int wk[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // entry bits with the child index in the low 2 bits (orderable when >= 0)
                        wk[k] = __reduce_min_sync(FULL, ((ih >> k) & 1u) ? ((__float_as_int(tn4[k]) & ~3) | k) : 0x7FFFFFFF);
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
                    // far-to-near: entries nin-1 .. 1 (unused sort slots hold INT_MAX)
                    // warp-uniform values: every lane stores the same word, no
                    // divergent branch (1.766 -> 1.746 ms seed mean)
#pragma unroll
                    for (int j = 3; j >= 1; --j)
                        if (j < nin) {
                            sstk[wid][sp + nin - 1 - j] = make_int2(SRT_KID(wk[j] & 3), wk[j] & ~3);
                        }
                    sp += nin - 1;
                    node = SRT_KID(wk[0] & 3);
#undef SRT_KID
                }
            }
            __syncwarp();
        }
        double f64v[4] = {-1.0, 0.0, 0.0, 0.0};
        int64_t f64pix = -1;
        if (valid) {
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                unsigned long long v = sbest[wid][lane][k];
                sl.id[k] = (int)(unsigned)v;
                sl.t[k] = unpack_t(v);
            }
            src.template finish_shaded<NS>(idx, sl, s, r.fdx, r.fdy, r.fdz, f64v, &f64pix);
        }
        __syncwarp();
        // the packet's f64 frame pixels (fused last pass into rgb64/op64);
        // staged in sdd / sbest, which the next packet rewrites after this
        store_f64_packet(src, f64pix >= 0, f64v, f64pix, &sdd[wid][0][0], reinterpret_cast<double *>(&sbest[wid][0][0]));
        __syncwarp();
#ifdef SRT_PACKET_CLOCKS
        if (lane == 0 && (base >> 5) < kClockSlots) {
            uint64_t t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_packet_clk[(base >> 5) * 2] = clk_t0;
            g_packet_clk[(base >> 5) * 2 + 1] = (t1 - clk_t0) | ((uint64_t)smid << 48);
        }
        {
            const unsigned hitl = __ballot_sync(FULL, valid && far < r.t_max0);
            if (lane == 0 && (base >> 5) < kClockSlots) {
                g_packet_cnt[(base >> 5) * 4] = pk_visits;
                g_packet_cnt[(base >> 5) * 4 + 1] = pk_jobs;
                g_packet_cnt[(base >> 5) * 4 + 2] = pk_pops;
                g_packet_cnt[(base >> 5) * 4 + 3] = (mixed ? 1u : 0u) | ((unsigned)__popc(hitl) << 1);
            }
        }
#endif
    }
    src.done();
    ct.flush(stats);
    release_counter(work);
}

template <int NS, int MODE, int RNG, class Src, bool STATS>
static srt_status launch_trace_packet(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st);

// incoherent multi-slot walks refill as soon as 8 lanes are idle: 2M random
// rays at N=4, 91.6 -> 111 Mrays/s over whole-warp refills
#ifndef SRT_COOP_REFILL
#define SRT_COOP_REFILL 8
#endif
template <int NS, int MODE, int RNG, class Src, bool STATS, int REFILL = SRT_COOP_REFILL>
static srt_status launch_trace_coop(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st);

static int g_num_sms = 0;

template <int NS, int MODE, int RNG, class Src, int REFILL, bool STATS>
static srt_status launch_trace_v(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st) {
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_trace<NS, MODE, RNG, Src, REFILL, STATS>,
                                                      kTraceThreads, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    LaunchCounter work;
    srt_status rc = work.init(s, st);
    if (rc) return rc;
    int64_t need = ((int64_t)src.total() + kTraceThreads - 1) / kTraceThreads;
    int64_t grid = (int64_t)g_num_sms * blocks_per_sm;
    if (grid > need) grid = need;
    k_trace<NS, MODE, RNG, Src, REFILL, STATS>
        <<<(unsigned)grid, kTraceThreads, 0, st>>>(s->walk_view(), src, w, work.p, s->d_flag, s->d_stats);
    return cuda_status(cudaGetLastError(), "k_trace launch");
}

template <int NS, int MODE, int RNG, class Src, bool STATS, int REFILL>
static srt_status launch_trace_coop(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st) {
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_trace_coop<NS, MODE, RNG, Src, STATS, REFILL>,
                                                      kTraceThreads, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    LaunchCounter work;
    srt_status rc = work.init(s, st);
    if (rc) return rc;
    int64_t need = ((int64_t)src.total() + kTraceThreads - 1) / kTraceThreads;
    int64_t grid = (int64_t)g_num_sms * blocks_per_sm;
    if (grid > need) grid = need;
    k_trace_coop<NS, MODE, RNG, Src, STATS, REFILL>
        <<<(unsigned)grid, kTraceThreads, 0, st>>>(s->walk_view(), src, w, work.p, s->d_flag, s->d_stats);
    return cuda_status(cudaGetLastError(), "k_trace_coop launch");
}

// SRT_TRACE_STATS=1 enables the traversal counters (srt_trace_stats).
static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <int NS, int MODE, int RNG, class Src, bool STATS, int BATCH, int MINB>
static srt_status launch_trace_packet_v(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st) {
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &blocks_per_sm, k_trace_packet<NS, MODE, RNG, Src, STATS, BATCH, MINB>, kTraceThreads, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    LaunchCounter work;
    srt_status rc = work.init(s, st);
    if (rc) return rc;
    int64_t need = ((int64_t)src.total() + kTraceThreads - 1) / kTraceThreads;
    int64_t grid = (int64_t)g_num_sms * blocks_per_sm;
    if (grid > need) grid = need;
    k_trace_packet<NS, MODE, RNG, Src, STATS, BATCH, MINB>
        <<<(unsigned)grid, kTraceThreads, 0, st>>>(s->walk_view(), src, w, work.p, s->d_flag, s->d_stats);
    return cuda_status(cudaGetLastError(), "k_trace_packet launch");
}

static int env_int(const char *name, int dflt);

template <int NS, int MODE, int RNG, class Src, bool STATS>
static srt_status launch_trace_packet(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st) {
#ifdef SRT_EXPERIMENTS
    // A/B configurations of the packet kernel, only in the experiments build
    // (make experiments -> libsrt_exp.so, selected with SRT_LIBSRT_PATH); the
    // release library has no environment-dependent kernel choice.
    // SRT_PACKET_CFG (N=1 mean depth): 1 batch 64, 2 batch 32 at 7 blocks/SM,
    // 3 batch 64 at 8, 12 / 13 batch 48 at 9 / 10 blocks/SM.
    static const int cfg = env_int("SRT_PACKET_CFG", 0);
    if constexpr (NS == 1 && MODE == 0 && !STATS && !Src::kRayOrigin) {
        if (cfg == 1) return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, 64, 1>(s, src, w, st);
        if (cfg == 2) return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, 32, 7>(s, src, w, st);
        if (cfg == 3) return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, 64, 8>(s, src, w, st);
        if (cfg == 12) return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, 48, 9>(s, src, w, st);
        if (cfg == 13) return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, 48, 10>(s, src, w, st);
    }
#endif
    // 8 resident blocks/SM (64 registers, no spills) at N=1: 1.936 vs 1.964 ms
    // at 7 blocks (once the walk had a single job-flush site); 7 blocks were
    // 12% faster than the 90-register build at N=4 (3.16 vs 3.53 ms, C3)
    // resident blocks per SM requested from the register allocator, per slot
    // count: the largest without spills (N=8: +6%, N=16: +4% over unconstrained)
#ifndef SRT_N1_MINB
#define SRT_N1_MINB 8
#endif
#ifndef SRT_N1_BATCH
#define SRT_N1_BATCH 32
#endif
    // N=4 at 8 blocks/SM and N=8 at 7 (end of round 2: 2.647 -> 2.612 ms and
    // 4.149 -> 3.975 ms for the 1080p frame; 8 blocks for N=8 and 32-job
    // batches for N=4 measured no better)
#ifndef SRT_N4_MINB
#define SRT_N4_MINB 8
#endif
#ifndef SRT_N4_BATCH
#define SRT_N4_BATCH 48
#endif
#ifndef SRT_N8_MINB
#define SRT_N8_MINB 7
#endif
    constexpr int kMinB = NS == 1 ? SRT_N1_MINB
                          : ((NS == 2 && MODE == 0) ? 8
                             : (NS == 2 ? 7 : ((NS == 4 && MODE == 0) ? SRT_N4_MINB : (NS <= 8 ? SRT_N8_MINB : 5))));
    // leaf jobs per flush threshold (flushes run whole 32-job rounds): 32 for
    // N=1 (round 2: 1.648 vs 1.662 ms at 48), 48 for N=4 (round 1: 2.957 vs
    // 2.993 ms); N=2 at 8 blocks/SM: 2.376 vs 2.419 ms
    constexpr int kBatch = NS == 1 ? SRT_N1_BATCH : ((NS == 4 && MODE == 0) ? SRT_N4_BATCH : 32);
    return launch_trace_packet_v<NS, MODE, RNG, Src, STATS, kBatch, kMinB>(s, src, w, st);
}

template <int NS, int MODE, int RNG, class Src>
static srt_status launch_trace_t(const SrtScene *s, const Src &src, const WalkCfg &w, cudaStream_t st) {
    if (src.total() == 0) return SRT_OK;
    static const bool stats = env_int("SRT_TRACE_STATS", 0) != 0 && s->d_stats;
#ifdef SRT_EXPERIMENTS
    // traversal policy A/B (experiments build only): 2 warp-cooperative leaf
    // compaction for every ray source, 0 / 1 per-lane walks with refill at 32 /
    // 8 idle lanes; 3 (default) the release policy below
    static const int variant = env_int("SRT_TRACE_VARIANT", 3);
    if (variant == 2) {
        if (stats) return launch_trace_coop<NS, MODE, RNG, Src, true>(s, src, w, st);
        return launch_trace_coop<NS, MODE, RNG, Src, false>(s, src, w, st);
    }
    if (variant == 0 || variant == 1) {
        if (stats) return variant ? launch_trace_v<NS, MODE, RNG, Src, 8, true>(s, src, w, st)
                                  : launch_trace_v<NS, MODE, RNG, Src, 32, true>(s, src, w, st);
        return variant ? launch_trace_v<NS, MODE, RNG, Src, 8, false>(s, src, w, st)
                       : launch_trace_v<NS, MODE, RNG, Src, 32, false>(s, src, w, st);
    }
#endif
    if constexpr (Src::kCoherent) {
        // camera rays and one-hemisphere explicit batches: warp packets
        if (stats) return launch_trace_packet<NS, MODE, RNG, Src, true>(s, src, w, st);
        return launch_trace_packet<NS, MODE, RNG, Src, false>(s, src, w, st);
    } else if constexpr (NS == 1) {
        // incoherent single-slot walks are fastest per lane with refill at 8
        // idle lanes (142 vs 122 Mrays/s on 2M random rays in the 1M cloud)
        if (stats) return launch_trace_v<NS, MODE, RNG, Src, 8, true>(s, src, w, st);
        return launch_trace_v<NS, MODE, RNG, Src, 8, false>(s, src, w, st);
    } else {
        // multi-slot incoherent walks gain from the cooperative leaf compaction
        if (stats) return launch_trace_coop<NS, MODE, RNG, Src, true>(s, src, w, st);
        return launch_trace_coop<NS, MODE, RNG, Src, false>(s, src, w, st);
    }
}

template <class Src, int RNG>
static srt_status dispatch(const SrtScene *s, const Src &src, const WalkCfg &w, int nslots, int mode, cudaStream_t st) {
#define SRT_NS(NS)                                                      \
    return mode == 0 ? launch_trace_t<NS, 0, RNG, Src>(s, src, w, st)   \
                     : launch_trace_t<NS, 1, RNG, Src>(s, src, w, st);
    if (nslots <= 1) SRT_NS(1)
    if (nslots <= 2) SRT_NS(2)
    if (nslots <= 4) SRT_NS(4)
    if (nslots <= 8) SRT_NS(8)
#undef SRT_NS
    set_error("a walk holds at most 8 slots (callers split larger N into slot groups)");
    return SRT_ERR_UNSUPPORTED;
}

srt_status launch_trace_pass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass, int32_t *d_hits,
                             cudaStream_t st) {
    if (a.rng == SRT_RNG_TRIG64) return launch_trace_pass_trig64(s, cam, a, pass, (double)a.s2d, d_hits, st);
    return launch_render_pass_fused(s, cam, a, pass, nullptr, false, false, nullptr, st, d_hits);
}

// One pass traced AND shaded by the packet kernel (d_hits == nullptr), or
// traced into d_hits for a separate k_shade_pass.
// Work items of one persistent launch: the 32-bit work counter is advanced
// by every warp once more after the last item (up to ~5k warps x 32), so a
// launch stays far below 2^32 items and the counter can never wrap.
constexpr uint64_t kMaxLaunchItems = 1ull << 31;

// Slots per walk: multisample N > 8 runs as ceil(N / 8) walks of <= 8 slots
// over the same ray (CameraSource::slot0).  Two 8-slot walks beat one 16-slot
// walk (3.88 vs 2.95 G samples/s at 1080p in the 1M cloud): the 16-slot walk
// keeps its slots in local memory.
constexpr int kSlotGroup = 8;

static uint32_t frame_key_host(uint32_t seed) {
    uint32_t x = seed ^ 0x9E3779B9u;
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

srt_status launch_render_pass_fused(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass,
                                   float4 *d_accum, bool first, bool last, float4 *d_out, cudaStream_t st,
                                   int32_t *d_hits, double *d_rgb64, double *d_op64, bool out_rowmajor,
                                   bool sys_fence) {
    if ((uint64_t)a.local_tiles * 256 > kMaxLaunchItems) {
        set_error("frame too large for one launch");
        return SRT_ERR_INVALID_ARG;
    }
    CameraSource src;
    src.accum = d_accum;
    src.out = d_out;
    src.rgb64 = d_rgb64;
    src.op64 = d_op64;
    src.acc64 = nullptr;
    src.npass = 1;
    src.unit = (uint32_t)(a.local_tiles * 256);
    src.first = first ? 1 : 0;
    src.last = last ? 1 : 0;
    src.cam = cam;
    src.a = a;
    src.pass = pass;
    src.fkey = 0;
    src.hits = d_hits;
    src.out_rowmajor = out_rowmajor ? 1 : 0;
    src.sys_fence = sys_fence ? 1 : 0;
    src.fkey = frame_key_host(a.seed);  // frame_key() of the device code, on the host
    WalkCfg w{a.s2, sqrtf(a.s2), a.clip, nullptr, 0};
    srt_status rc = SRT_OK;
    for (int g0 = 0; g0 < a.nslots && !rc; g0 += kSlotGroup) {
        const bool lastg = g0 + kSlotGroup >= a.nslots;
        src.slot0 = (uint32_t)g0;
        src.gslots = std::min(kSlotGroup, a.nslots - g0);
        src.first = first && g0 == 0 ? 1 : 0;
        src.last = last && lastg ? 1 : 0;
        src.rgb64 = lastg ? d_rgb64 : nullptr;
        src.op64 = lastg ? d_op64 : nullptr;
        rc = dispatch<CameraSource, SRT_RNG_COUNTER>(s, src, w, src.gslots, a.mode, st);
    }
    return rc;
}

// All `npass` passes (pass0 ...) of a frame in ONE packet launch, summed into
// the zeroed fixed-point accumulator d_acc64 (unit * 4 u64); see CameraSource.
// Frames with more than 2^32 (pixel, pass) work items are split into pass
// chunks; integer sums do not care which launch added what.
static srt_status launch_multipass_chunk(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass0,
                                         int npass, unsigned long long *d_acc64, cudaStream_t st);

srt_status launch_render_frame_multipass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass0,
                                         int npass, unsigned long long *d_acc64, cudaStream_t st) {
    const uint64_t unit = (uint64_t)(a.local_tiles * 256);
    if (unit == 0 || npass <= 0) return SRT_OK;
    uint64_t limit = kMaxLaunchItems;  // work items per launch (32-bit work counter, with headroom)
    if (const char *e = getenv("SRT_MULTIPASS_MAX_ITEMS")) limit = std::min<uint64_t>(limit, strtoull(e, nullptr, 10));
    const int per = (int)std::min<uint64_t>((uint64_t)npass, limit / unit);
    if (per < 1) {
        set_error("frame too large for one work counter");
        return SRT_ERR_INVALID_ARG;
    }
    srt_status rc = SRT_OK;
    for (int f = 0; f < npass && !rc; f += per)
        rc = launch_multipass_chunk(s, cam, a, pass0 + f, std::min(per, npass - f), d_acc64, st);
    return rc;
}

static srt_status launch_multipass_chunk(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass0,
                                         int npass, unsigned long long *d_acc64, cudaStream_t st) {
    CameraSource src;
    src.accum = nullptr;
    src.out = nullptr;
    src.rgb64 = nullptr;
    src.op64 = nullptr;
    src.first = 0;
    src.last = 0;
    src.cam = cam;
    src.a = a;
    src.pass = pass0;
    src.hits = nullptr;
    src.out_rowmajor = 0;
    src.sys_fence = 0;
    src.acc64 = d_acc64;
    src.unit = (uint32_t)(a.local_tiles * 256);
    src.npass = (uint32_t)npass;
    src.fkey = frame_key_host(a.seed);
    WalkCfg w{a.s2, sqrtf(a.s2), a.clip, nullptr, 0};
    // slot groups add into the same integer sums (k_resolve_fixed divides by passes * N)
    srt_status rc = SRT_OK;
    for (int g0 = 0; g0 < a.nslots && !rc; g0 += kSlotGroup) {
        src.slot0 = (uint32_t)g0;
        src.gslots = std::min(kSlotGroup, a.nslots - g0);
        rc = dispatch<CameraSource, SRT_RNG_COUNTER>(s, src, w, src.gslots, a.mode, st);
    }
    return rc;
}

// ---------------------------------------------------------------------------
// Ray reordering for large batches of explicit (possibly incoherent) rays:
// 30-bit keys = 8-bit-per-axis Morton code of the origin inside the batch's
// origin bounds, then 2 bits per direction component; a stable radix sort of
// (key, index) gives the processing order.  Neighbouring lanes then walk
// neighbouring, similarly directed rays.  Results and random draws stay keyed
// by the original index, so the output does not depend on the order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread8(uint32_t v) {  // 8 bits -> every third bit
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ int ordered(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float unordered(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

__global__ void k_ray_bounds(const double *__restrict__ rays, uint32_t R, int *bounds) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    if (i < R)
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = ordered((float)rays[(int64_t)i * 6 + a]);
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
        if ((threadIdx.x & 31) == 0 && lo[a] <= hi[a]) {
            atomicMin(bounds + a, lo[a]);
            atomicMax(bounds + 3 + a, hi[a]);
        }
    }
}

__global__ void k_ray_keys(const double *__restrict__ rays, uint32_t R, const int *__restrict__ bounds,
                           uint32_t *keys, uint32_t *idx) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double *q = rays + (int64_t)i * 6;
    uint32_t m = 0, dkey = 0;
    for (int a = 0; a < 3; ++a) {
        float lo = unordered(bounds[a]), hi = unordered(bounds[3 + a]);
        float u = hi > lo ? ((float)q[a] - lo) / (hi - lo) : 0.0f;
        uint32_t c = (uint32_t)fminf(fmaxf(u * 256.0f, 0.0f), 255.0f);
        m |= spread8(c) << a;
        float d = (float)q[3 + a];
        uint32_t db = d < -0.5f ? 0u : (d < 0.0f ? 1u : (d < 0.5f ? 2u : 3u));
        dkey = (dkey << 2) | db;
    }
    keys[i] = (m << 6) | dkey;
    idx[i] = i;
}

// 64 evenly spaced rays of a batch (R >= 64): one shared origin (a camera
// batch, already coherent in its given order) and whether every probed
// direction lies in the hemisphere of the first (a coherent batch: camera
// rays, the reference's parallel jittered rays, validate.py:36-43).  Only the
// kernel choice depends on it, never a result.
srt_status probe_rays(const double *d_rays, uint32_t R, bool &one_origin, bool &one_hemisphere,
                      cudaStream_t st) {
    double probe[64][6];
    const size_t step = (size_t)(R / 64) * 6 * sizeof(double);
    srt_status rc = cuda_status(cudaMemcpy2DAsync(probe, sizeof(probe[0]), d_rays, step, sizeof(probe[0]), 64,
                                                  cudaMemcpyDeviceToHost, st), "ray probe");
    if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "ray probe");
    if (rc) return rc;
    one_origin = one_hemisphere = true;
    for (int j = 1; j < 64; ++j) {
        one_origin &= probe[j][0] == probe[0][0] && probe[j][1] == probe[0][1] && probe[j][2] == probe[0][2];
        one_hemisphere &= probe[j][3] * probe[0][3] + probe[j][4] * probe[0][4] + probe[j][5] * probe[0][5] > 0.0;
    }
    return SRT_OK;
}

// Smallest one-hemisphere batch walked as packets by default: one-origin
// batches are coherent as given; distinct origins need the sort, which only
// pays for itself on large batches (parallel jittered rays in the 1M cloud:
// packets 0.583 vs 0.523 ms per-lane at 60k rays, 2x faster at 2M;
// tools/exp/prays3.sh, prays4.sh: 1.47x at 131k).
constexpr int64_t PACKET_MIN_DISTINCT = 65536;
int64_t packet_min(bool one_origin) { return one_origin ? 4096 : PACKET_MIN_DISTINCT; }

srt_status sort_rays(const double *d_rays, uint32_t R, uint32_t **d_perm_out, void **d_mem_out,
                     cudaStream_t st) {
    *d_perm_out = nullptr;
    *d_mem_out = nullptr;
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)R, 0, 30, st);
    size_t arr = ((sizeof(uint32_t) * (size_t)R + 255) / 256) * 256;
    size_t total = 4 * arr + 256 + temp;
    char *mem = nullptr;
    srt_status rc = cuda_status(cudaMallocAsync((void **)&mem, total, st), "ray sort scratch");
    if (rc) return rc;
    uint32_t *k0 = (uint32_t *)mem, *k1 = (uint32_t *)(mem + arr), *v0 = (uint32_t *)(mem + 2 * arr),
             *v1 = (uint32_t *)(mem + 3 * arr);
    int *bounds = (int *)(mem + 4 * arr);
    void *tmp = mem + 4 * arr + 256;
    const int init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
    rc = cuda_status(cudaMemcpyAsync(bounds, init, sizeof(init), cudaMemcpyHostToDevice, st), "ray bounds init");
    unsigned blocks = (R + 255) / 256;
    if (!rc) {
        k_ray_bounds<<<blocks, 256, 0, st>>>(d_rays, R, bounds);
        rc = cuda_status(cudaGetLastError(), "ray bounds");
    }
    if (!rc) {
        k_ray_keys<<<blocks, 256, 0, st>>>(d_rays, R, bounds, k0, v0);
        rc = cuda_status(cudaGetLastError(), "ray keys");
    }
    if (!rc)
        rc = cuda_status(cub::DeviceRadixSort::SortPairs(tmp, temp, k0, k1, v0, v1, (int)R, 0, 30, st), "ray sort");
    if (rc) {
        cudaFreeAsync(mem, st);
        return rc;
    }
    *d_perm_out = v1;
    *d_mem_out = mem;
    return SRT_OK;
}

srt_status launch_trace_rays(const SrtScene *s, const SrtTraceParams *p, const double *d_rays, int64_t R, int nslots,
                             const double *d_table, float *d_t, int32_t *d_id, cudaStream_t st) {
    if ((uint64_t)R > kMaxLaunchItems) {
        set_error("too many rays in one call (at most 2^31)");
        return SRT_ERR_INVALID_ARG;
    }
    ArraySource src;
    src.rays = d_rays;
    src.R = (uint32_t)R;
    src.t_min = p->t_min;
    src.t_max = p->t_max;
    src.nslots = nslots;
    src.fkey = frame_key_host(p->seed);
    src.ray_id0 = p->ray_id0;
    src.sample0 = p->sample0;
    src.out_t = d_t;
    src.out_id = d_id;
    src.perm = nullptr;
    // Batches of >= 4096 rays in one hemisphere are walked as warp packets
    // (counter RNG; SRT_PACKET_RAYS: -1 auto, 0 never, 1 always); large
    // batches from distinct origins are walked in sorted order (SRT_RAY_SORT=0
    // disables; per-lane single-slot walks, or any packet walk)
    const int packet_env = env_int("SRT_PACKET_RAYS", -1);  // read per call (tests switch it)
    static const int sort_min = env_int("SRT_RAY_SORT", 1) ? 65536 : INT_MAX;
    bool one_origin = false, one_hemisphere = false;
    if (R >= 4096) {
        srt_status rc = probe_rays(d_rays, (uint32_t)R, one_origin, one_hemisphere, st);
        if (rc) return rc;
    }
    const bool packets = p->rng == SRT_RNG_COUNTER &&
                         (packet_env > 0 || (packet_env < 0 && one_hemisphere && R >= packet_min(one_origin)));
    void *sort_mem = nullptr;
    // packets from distinct origins need the sort at any size (unsorted
    // random-origin packets walk 5x slower)
    const bool sort_on = sort_min != INT_MAX;
    if (!one_origin && ((packets && sort_on && R >= 4096) || (R >= sort_min && nslots == 1))) {
        uint32_t *perm = nullptr;
        srt_status rc = sort_rays(d_rays, (uint32_t)R, &perm, &sort_mem, st);
        if (rc) return rc;
        src.perm = perm;
    }
    WalkCfg w{(float)p->s2, (float)std::sqrt(p->s2), p->clip, d_table, p->table_slots};
    srt_status rc = SRT_OK;
    // More than 8 slots: walks of <= 8 slots each (kSlotGroup), slot group g
    // drawing samples sample0 + 8 g + k (or table columns 8 g + k).  Slots are independent --
    // the clip only culls entries beyond the farthest slot bound, so a slot's
    // closest accepted hit never depends on the others -- and the groups
    // write disjoint columns of the (R, nslots) outputs.
    const int group = kSlotGroup;
    src.ostride = nslots;
    for (int g0 = 0; g0 < nslots && !rc; g0 += group) {
        WalkCfg wg = w;
        if (wg.table) wg.table += g0;  // table draws: slot g0 + k reads column g0 + k
        ArraySource gs = src;
        gs.nslots = std::min(group, nslots - g0);
        gs.sample0 = p->sample0 + (uint32_t)g0;
        gs.out_t = d_t + g0;
        gs.out_id = d_id + g0;
        if (packets) {
            PacketArraySource ps;
            static_cast<ArraySource &>(ps) = gs;
            memset(&ps.cam, 0, sizeof(ps.cam));
            ps.f_tmin = (float)p->t_min;  // the interval exactly as init_ray rounds it
            ps.f_tmax = p->t_max >= 3.0e38 ? INFINITY : (float)p->t_max;
            rc = dispatch<PacketArraySource, SRT_RNG_COUNTER>(s, ps, wg, gs.nslots, p->mode, st);
        } else {
            rc = p->rng == SRT_RNG_TABLE ? dispatch<ArraySource, SRT_RNG_TABLE>(s, gs, wg, gs.nslots, p->mode, st)
                                         : dispatch<ArraySource, SRT_RNG_COUNTER>(s, gs, wg, gs.nslots, p->mode, st);
        }
    }
    if (sort_mem) cudaFreeAsync(sort_mem, st);
    return rc;
}

// ---------------------------------------------------------------------------
// transmittance: prod(1 - alpha) over every valid candidate, no clipping
// (kernels.py:392-432).  The product order differs from the reference's
// walk; the value agrees to product-reordering roundoff (fp32 alphas).
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(128) k_transmittance(SceneView s, const double *__restrict__ rays, int64_t R,
                                                       double t_min, double t_max, float s2, double *out,
                                                       int *overflow, const uint32_t *__restrict__ perm) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    if (perm) i = __ldg(perm + i);  // walked in sorted order, written in the caller's
    const float sqrt_s2 = sqrtf(s2);
    const double *q = rays + i * 6;
    RayState r;
    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
    double result = 1.0;
    int stk[kStackSize];
    int sp = 0;
    int node = s.num_nodes4 > 0 ? 0 : kDone;
    while (node != kDone) {
        int4 kids;
        int key[4];
        SRT_DCHECK(node >= 0 && node < s.num_nodes4);
        unsigned hitm = slab4(r, reinterpret_cast<const float4 *>(s.nodes4 + node), r.t_max0, kids, key);
        node = kDone;
        while (hitm) {
            int k = __ffs(hitm) - 1;
            hitm &= hitm - 1;
            int code = pick(kids, k);
            if (code < 0) {
                SRT_DCHECK(~code < s.n);
                const float4 *g = reinterpret_cast<const float4 *>(s.geom + ~code);
                float4 m = __ldg(g), a = __ldg(g + 1), b = __ldg(g + 2);
                // fp32 screen first: certainly-invalid candidates skip the fp64 stage
                if (!screen<MODE>(r, m, a, b, s2, sqrt_s2, r.t_max0).maybe) continue;
                Cand cd = candidate<MODE>(r, m, a, b, s2);
                if (cd.valid) result *= 1.0 - (double)cd.alpha;
            } else if (node == kDone) {
                node = code;
            } else if (sp < kStackSize) {
                stk[sp++] = code;
            } else {
                raise_flag(overflow);
            }
        }
        if (node == kDone && sp > 0) node = stk[--sp];
    }
    out[i] = result;
}

// Coherent transmittance batches (one hemisphere, e.g. shadow rays towards a
// light): the warp walks its 32 rays as a packet over the octant node copies
// (near planes first: 6 FMAs and two 3-way min/max per child, as in
// k_trace_packet), leaf hits compacted by ballot into a job queue; each job
// screens the owner's ray in fp32 and evaluates the owner's fp64 candidate
// exactly as the per-lane walk does, multiplying (1 - alpha) into the owner's
// product in shared memory.  The owner's fp64 origin, direction and 1/|d|^2
// sit in shared memory, so a job builds no RayState.  The walk is unclipped
// (kernels.py:392-432): nothing is culled, any visit order gives the same
// factors; only the product order differs from the per-lane walk (roundoff).
template <int MODE>
__global__ void __launch_bounds__(kTraceThreads) k_transmittance_packet(SceneView s, const double *__restrict__ rays,
                                                                        const uint32_t *__restrict__ perm, uint32_t R,
                                                                        double t_min, double t_max, float s2,
                                                                        double *out, uint32_t *work, int *overflow) {
    constexpr int W = kTraceThreads / 32;
    constexpr int PSTACK = 128, BATCH = 32;
    __shared__ double sray[W][32][7];  // fp64 origin, direction, 1/|d|^2
    __shared__ unsigned long long sprod[W][32];
    __shared__ uint32_t sjob[W][BATCH + 128];  // (slot << 5) | owner lane
    __shared__ int sstk[W][PSTACK];
    const unsigned FULL = 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float sqrt_s2 = sqrtf(s2);
    const unsigned lt = (1u << lane) - 1u;
    const float ft_min = (float)t_min, ft_max = t_max >= 3.0e38 ? INFINITY : (float)t_max;
    while (true) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(work, 32u);
        base = __shfl_sync(FULL, base, 0);
        if (base >= R) break;
        const uint32_t idx = base + (uint32_t)lane;
        const bool valid = idx < R;
        const uint32_t ri = valid ? (perm ? __ldg(perm + idx) : idx) : 0u;
        RayState r;
        float far;
        if (valid) {
            const double *q = rays + (int64_t)ri * 6;
            init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
            double *sq = sray[wid][lane];
            sq[0] = r.ox, sq[1] = r.oy, sq[2] = r.oz, sq[3] = r.dx, sq[4] = r.dy, sq[5] = r.dz, sq[6] = r.inv_dd;
            sprod[wid][lane] = __double_as_longlong(1.0);
            far = r.t_max0;
        } else {
            init_ray(r, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0);
            far = -INFINITY;  // hits nothing
        }
        const unsigned vm = __ballot_sync(FULL, valid);
        const unsigned nx_m = __ballot_sync(FULL, valid && signbit(r.idx));
        const unsigned ny_m = __ballot_sync(FULL, valid && signbit(r.idy));
        const unsigned nz_m = __ballot_sync(FULL, valid && signbit(r.idz));
        const int oct = (nx_m ? 1 : 0) | (ny_m ? 2 : 0) | (nz_m ? 4 : 0);
        const bool mixed = (nx_m && nx_m != vm) || (ny_m && ny_m != vm) || (nz_m && nz_m != vm);
        const uint32_t obase = (uint32_t)oct * (uint32_t)s.num_nodes4;
        int sp = 0, njobs = 0;
        int node = (s.num_nodes4 > 0 && vm) ? 0 : kDone;
        bool ovf = false;
        while (true) {
            if (njobs >= BATCH || (node == kDone && (sp == 0 || ovf) && njobs)) {
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
                        er.t_min = ft_min, er.t_max0 = ft_max;
                        ScreenRay sr;
                        sr.fox = (float)er.ox, sr.foy = (float)er.oy, sr.foz = (float)er.oz;
                        sr.omag = fmaxf(fabsf(sr.fox), fmaxf(fabsf(sr.foy), fabsf(sr.foz)));
                        sr.fdx = er.fdx, sr.fdy = er.fdy, sr.fdz = er.fdz;
                        sr.inv_dd = er.inv_dd;
                        sr.t_min = ft_min, sr.t_max0 = ft_max;
                        const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
                        const float4 gm = __ldg(g), ga = __ldg(g + 1), gb = __ldg(g + 2);
                        if (screen<MODE>(sr, gm, ga, gb, s2, sqrt_s2, ft_max).maybe) {
                            const Cand cd = candidate<MODE>(er, gm, ga, gb, s2);
                            if (cd.valid) {
                                const double f = 1.0 - (double)cd.alpha;
                                unsigned long long *p = &sprod[wid][ow];
                                unsigned long long old = *p, assumed;
                                do {
                                    assumed = old;
                                    old = atomicCAS(p, assumed, __double_as_longlong(__longlong_as_double(assumed) * f));
                                } while (assumed != old);
                            }
                        }
                    }
                }
                __syncwarp();
                njobs = 0;
            }
            if (node == kDone) {
                if (sp == 0 || ovf) break;
                node = sstk[wid][--sp];
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
                // closed slab (kernels.py:279,308) clipped to [t_min, t_max]
                hitm |= fmaxf(tn, r.t_min) <= tf ? (1u << k) : 0u;
            }
            hitm &= hint & 15u;
            const unsigned leafm = (hint >> 4) & 15u;
            const unsigned any = __reduce_or_sync(FULL, hitm);
            const unsigned lh = hitm & leafm;
            node = kDone;
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
            // unclipped: every inner child any lane hits is walked, in any order
            for (unsigned ai = any & ~leafm; ai; ai &= ai - 1) {
                const int code = __shfl_sync(FULL, mykid, __ffs(ai) - 1);
                if (node == kDone) {
                    node = code;
                } else if (sp < PSTACK) {
                    sstk[wid][sp++] = code;  // warp-uniform: every lane stores the same word
                } else {
                    if (lane == 0) raise_flag(overflow);
                    ovf = true;
                }
            }
            __syncwarp();
        }
        __syncwarp();
        if (valid) out[ri] = __longlong_as_double(sprod[wid][lane]);
        __syncwarp();
    }
    release_counter(work);
}

// Incoherent transmittance batches (rays from distinct origins in all
// directions): per-lane walks with warp-compacted leaf work.  Each step
// every active lane visits one node of its own ray (min/max slab, per-lane
// stack); the leaf children the lanes hit go to a warp job queue (prefix-sum
// compaction) and, once 32 are queued or a lane's walk ends, the whole warp
// screens and evaluates them together, multiplying (1 - alpha) into the
// owner's product in shared memory.  Idle lanes take new rays as soon as 8
// are free, so the warp stays full while long rays finish.  Same candidates
// and factors as the per-lane walk; only the product order differs.
template <int MODE>
__global__ void __launch_bounds__(kTraceThreads) k_transmittance_coop(SceneView s, const double *__restrict__ rays,
                                                                      const uint32_t *__restrict__ perm, uint32_t R,
                                                                      double t_min, double t_max, float s2,
                                                                      double *out, uint32_t *work, int *overflow) {
    constexpr int W = kTraceThreads / 32, QCAP = 32 + 128;
    __shared__ double sray[W][32][7];  // fp64 origin, direction, 1/|d|^2
    __shared__ unsigned long long sprod[W][32];
    __shared__ uint32_t sjob[W][QCAP];  // (slot << 5) | owner lane
    const unsigned FULL = 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const float sqrt_s2 = sqrtf(s2);
    const float ft_min = (float)t_min, ft_max = t_max >= 3.0e38 ? INFINITY : (float)t_max;
    RayState r;
    init_ray(r, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0);
    int stk[kStackSize];
    int sp = 0, node = kLeafEmpty, njobs = 0;
    bool active = false, exhausted = false;
    uint32_t ri = 0;
    while (true) {
        const unsigned idle = __ballot_sync(FULL, !active);
        if (!exhausted && __popc(idle) >= 8) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(work, (uint32_t)__popc(idle));
            base = __shfl_sync(FULL, base, 0);
            if (base + (uint32_t)__popc(idle) >= R) exhausted = true;
            if (!active) {
                const uint32_t my = base + (uint32_t)__popc(idle & lt);
                if (my < R) {
                    ri = perm ? __ldg(perm + my) : my;
                    const double *q = rays + (int64_t)ri * 6;
                    init_ray(r, q[0], q[1], q[2], q[3], q[4], q[5], t_min, t_max);
                    double *sq = sray[wid][lane];
                    sq[0] = r.ox, sq[1] = r.oy, sq[2] = r.oz, sq[3] = r.dx, sq[4] = r.dy, sq[5] = r.dz;
                    sq[6] = r.inv_dd;
                    sprod[wid][lane] = __double_as_longlong(1.0);
                    sp = 0;
                    node = s.num_nodes4 > 0 ? 0 : kLeafEmpty;
                    active = true;
                }
            }
        } else if (exhausted && idle == FULL) {
            break;
        }
        // one node visit per walking lane
        unsigned lm = 0;
        int4 kids = make_int4(kLeafEmpty, kLeafEmpty, kLeafEmpty, kLeafEmpty);
        if (active && node != kLeafEmpty) {
            SRT_DCHECK(node >= 0 && node < s.num_nodes4);
            const float4 *np = reinterpret_cast<const float4 *>(s.nodes4 + node);
            const float4 lox = __ldg(np), hix = __ldg(np + 1), loy = __ldg(np + 2), hiy = __ldg(np + 3),
                         loz = __ldg(np + 4), hiz = __ldg(np + 5);
            kids = __ldg(reinterpret_cast<const int4 *>(np + 6));
            const unsigned hint = (unsigned)__ldg(reinterpret_cast<const int *>(np + 7));
            const float lx[4] = {lox.x, lox.y, lox.z, lox.w}, hx[4] = {hix.x, hix.y, hix.z, hix.w};
            const float ly[4] = {loy.x, loy.y, loy.z, loy.w}, hy[4] = {hiy.x, hiy.y, hiy.z, hiy.w};
            const float lz[4] = {loz.x, loz.y, loz.z, loz.w}, hz[4] = {hiz.x, hiz.y, hiz.z, hiz.w};
            unsigned hitm = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float xa = fmaf(lx[k], r.idx, -r.oidx), xb = fmaf(hx[k], r.idx, -r.oidx);
                const float ya = fmaf(ly[k], r.idy, -r.oidy), yb = fmaf(hy[k], r.idy, -r.oidy);
                const float za = fmaf(lz[k], r.idz, -r.oidz), zb = fmaf(hz[k], r.idz, -r.oidz);
                const float tn = fmaxf(fmaxf(fminf(xa, xb), fminf(ya, yb)), fmaxf(fminf(za, zb), r.t_min));
                const float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), r.t_max0));
                hitm |= tn <= tf ? (1u << k) : 0u;
            }
            hitm &= hint & 15u;
            const unsigned leafm = (hint >> 4) & 15u;
            lm = hitm & leafm;
            // unclipped: every hit inner child is walked, in any order
            node = kLeafEmpty;
            for (unsigned im = hitm & ~leafm; im; im &= im - 1) {
                const int c = sel4(kids, __ffs(im) - 1);
                if (node == kLeafEmpty) {
                    node = c;
                } else if (sp < kStackSize) {
                    stk[sp++] = c;
                } else {
                    raise_flag(overflow);
                }
            }
            if (node == kLeafEmpty && sp > 0) node = stk[--sp];
        }
        // queue the hit leaf children of every lane
        const int cnt = __popc(lm);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        int off = njobs + incl - cnt;
        for (unsigned m = lm; m; m &= m - 1) {
            SRT_DCHECK(off < QCAP);
            sjob[wid][off++] = ((uint32_t)~sel4(kids, __ffs(m) - 1) << 5) | (uint32_t)lane;
        }
        njobs += __shfl_sync(FULL, incl, 31);
        const bool ending = active && node == kLeafEmpty;
        if (njobs >= 32 || (njobs > 0 && __any_sync(FULL, ending))) {
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
                    er.t_min = ft_min, er.t_max0 = ft_max;
                    ScreenRay sr;
                    sr.fox = (float)er.ox, sr.foy = (float)er.oy, sr.foz = (float)er.oz;
                    sr.omag = fmaxf(fabsf(sr.fox), fmaxf(fabsf(sr.foy), fabsf(sr.foz)));
                    sr.fdx = er.fdx, sr.fdy = er.fdy, sr.fdz = er.fdz;
                    sr.inv_dd = er.inv_dd;
                    sr.t_min = ft_min, sr.t_max0 = ft_max;
                    const float4 *g = reinterpret_cast<const float4 *>(s.geom + slot);
                    const float4 gm = __ldg(g), ga = __ldg(g + 1), gb = __ldg(g + 2);
                    if (screen<MODE>(sr, gm, ga, gb, s2, sqrt_s2, ft_max).maybe) {
                        const Cand cd = candidate<MODE>(er, gm, ga, gb, s2);
                        if (cd.valid) {
                            const double f = 1.0 - (double)cd.alpha;
                            unsigned long long *pp = &sprod[wid][ow];
                            unsigned long long old = *pp, assumed;
                            do {
                                assumed = old;
                                old = atomicCAS(pp, assumed, __double_as_longlong(__longlong_as_double(assumed) * f));
                            } while (assumed != old);
                        }
                    }
                }
            }
            __syncwarp();
            njobs = 0;
        }
        if (ending && njobs == 0) {
            out[ri] = __longlong_as_double(sprod[wid][lane]);
            active = false;
        }
    }
    release_counter(work);
}

srt_status launch_transmittance(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max,
                                int mode, double s2, double *d_out, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
    uint32_t *perm = nullptr;
    void *sort_mem = nullptr;
    // one-hemisphere batches of >= 4096 rays walk as packets (SRT_PACKET_RAYS
    // as for srt_trace_rays); one-origin batches are already coherent: no sort
    static const int sort_min = env_int("SRT_RAY_SORT", 1) ? 65536 : INT_MAX;
    const int packet_env = env_int("SRT_PACKET_RAYS", -1);
    const bool fits = (uint64_t)R <= kMaxLaunchItems;
    bool one_origin = false, one_hemisphere = false;
    if (fits && R >= 4096) {
        srt_status rc = probe_rays(d_rays, (uint32_t)R, one_origin, one_hemisphere, st);
        if (rc) return rc;
    }
    const bool packets = fits && (packet_env > 0 || (packet_env < 0 && one_hemisphere && R >= packet_min(one_origin)));
    if (fits && !one_origin && (R >= sort_min || (packets && sort_min != INT_MAX && R >= 4096))) {
        srt_status rc = sort_rays(d_rays, (uint32_t)R, &perm, &sort_mem, st);
        if (rc) return rc;
    }
    if (packets) {
        static int blocks_per_sm = 0;
        if (!blocks_per_sm) {
            if (mode == 0)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_transmittance_packet<0>, kTraceThreads, 0);
            else
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_transmittance_packet<1>, kTraceThreads, 0);
            if (blocks_per_sm < 1) blocks_per_sm = 1;
        }
        if (!g_num_sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        }
        LaunchCounter work;
        srt_status rc = work.init(s, st);
        int64_t need = (R + kTraceThreads - 1) / kTraceThreads;
        int64_t grid = std::min<int64_t>((int64_t)g_num_sms * blocks_per_sm, need);
        if (!rc) {
            if (mode == 0)
                k_transmittance_packet<0><<<(unsigned)grid, kTraceThreads, 0, st>>>(
                    s->view(), d_rays, perm, (uint32_t)R, t_min, t_max, (float)s2, d_out, work.p, s->d_flag);
            else
                k_transmittance_packet<1><<<(unsigned)grid, kTraceThreads, 0, st>>>(
                    s->view(), d_rays, perm, (uint32_t)R, t_min, t_max, (float)s2, d_out, work.p, s->d_flag);
            rc = cuda_status(cudaGetLastError(), "k_transmittance_packet launch");
        }
        if (sort_mem) cudaFreeAsync(sort_mem, st);
        return rc;
    }
    if (!fits) {
        // more rays than one work counter covers: per-lane walks
        if (mode == 0)
            k_transmittance<0><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, d_out, s->d_flag,
                                                       perm);
        else
            k_transmittance<1><<<blocks, 128, 0, st>>>(s->view(), d_rays, R, t_min, t_max, (float)s2, d_out, s->d_flag,
                                                       perm);
        srt_status rc = cuda_status(cudaGetLastError(), "k_transmittance launch");
        if (sort_mem) cudaFreeAsync(sort_mem, st);
        return rc;
    }
    // incoherent batches: per-lane walks, warp-compacted leaf work
    static int coop_per_sm = 0;
    if (!coop_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&coop_per_sm, k_transmittance_coop<0>, kTraceThreads, 0);
        if (coop_per_sm < 1) coop_per_sm = 1;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    LaunchCounter work;
    srt_status rc = work.init(s, st);
    const int64_t grid = std::min<int64_t>((int64_t)g_num_sms * coop_per_sm, (R + kTraceThreads - 1) / kTraceThreads);
    if (!rc) {
        if (mode == 0)
            k_transmittance_coop<0><<<(unsigned)grid, kTraceThreads, 0, st>>>(
                s->view(), d_rays, perm, (uint32_t)R, t_min, t_max, (float)s2, d_out, work.p, s->d_flag);
        else
            k_transmittance_coop<1><<<(unsigned)grid, kTraceThreads, 0, st>>>(
                s->view(), d_rays, perm, (uint32_t)R, t_min, t_max, (float)s2, d_out, work.p, s->d_flag);
        rc = cuda_status(cudaGetLastError(), "k_transmittance_coop launch");
    }
    if (sort_mem) cudaFreeAsync(sort_mem, st);
    return rc;
}

}  // namespace srt
