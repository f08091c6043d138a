// srt_device.cuh -- device-side records and per-primitive math of libsrt.
//
// Layout in HBM:
//   Node2  64 B  binary BVH node holding BOTH children's fp32 boxes (one
//                visit = four 128-bit loads).  Leaves have exactly one
//                primitive, so a leaf child's box IS the primitive box
//                (the reference's separate prim-box test, kernels.py:344,
//                is folded into the parent visit).
//   Geom   48 B  per primitive in leaf ("slot") order: mean + opacity,
//                six inverse-covariance entries, original primitive id.
//   SH     K*12 B per primitive in ORIGINAL id order, channel major, fp32.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace srt {

constexpr int kLeafEmpty = INT32_MIN;  // child slot with no content
constexpr int kStackSize = 128;        // kernels.py:26

struct __align__(16) Node2 {
    float4 xy0;  // child0 lo.x hi.x lo.y hi.y
    float4 xy1;  // child1 lo.x hi.x lo.y hi.y
    float4 z01;  // child0 lo.z hi.z, child1 lo.z hi.z
    int4 kids;   // child0, child1 (>=0 inner node, <0 leaf ~slot, kLeafEmpty), pad
};

// 4-wide node, one 128-B line: child boxes SoA + child codes.  Produced by
// collapsing the binary tree (greedy largest-area expansion); unused slots
// have an empty box and code kLeafEmpty.  The octant copies (nodes8) hold
// the same record with, per axis whose direction sign is negative in that
// octant, the lo and hi plane arrays swapped: the first array of each axis is
// then the near planes of a ray in that octant.  pad.x = valid child mask |
// leaf child mask << 4.
struct __align__(128) Node4 {
    float4 lox, hix, loy, hiy, loz, hiz;
    int4 kids;
    int4 pad;
};

struct __align__(16) Geom {
    float4 m;  // mean.xyz, opacity
    float4 a;  // a00 a01 a02 a11
    float4 b;  // a12 a22, prim id (int bits), sqrt(sum |a_ij|) (screen error bound)
};

// Device-side invariant checks, compiled in only for the bounds-checked
// debug library (make debug): a failed check prints and traps the context.
#ifdef SRT_DEBUG
#define SRT_DCHECK(c)                                                              \
    do {                                                                           \
        if (!(c)) {                                                                \
            printf("SRT_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);       \
            __trap();                                                              \
        }                                                                          \
    } while (0)
#else
#define SRT_DCHECK(c) \
    do {              \
    } while (0)
#endif

// Device error flag (traversal stack overflow): one int in mapped page-locked
// host memory, set with a plain store (idempotent), read by the host after
// the stream synchronises -- no device->host copy, no memset on the stream.
__device__ __forceinline__ void raise_flag(int *flag) { *(volatile int *)flag = 1; }

struct SceneView {
    const double *means64;  // fp64 records in original id order (trig64 bridge mode)
    const double *cov64;
    const double *opac64;
    const Node2 *nodes;
    const Node4 *nodes4;
    const Node4 *nodes8;  // 8 x num_nodes4: the tree laid out per direction octant (packet kernel)
    int32_t num_nodes4;
    const Geom *geom;
    const float *sh;  // (n, 3, K) fp32, original id order
    int32_t num_nodes;
    int32_t root;      // 0, or a leaf code (~slot) when the tree is a single leaf
    int32_t sh_k;      // (deg + 1)^2
    int32_t sh_deg;
    int64_t n;
};

// End of a persistent launch: the last block out zeroes the (work, done)
// counter pair, so a counter reused by the next launch on the same stream
// needs no memset (LaunchCounter).
__device__ __forceinline__ void release_counter(uint32_t *work) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {
            work[0] = 0u;
            work[1] = 0u;
            __threadfence();
        }
    }
}

// Hit key (orderable fp32 depth << 32 | prim id): integer order = (t, id)
// order, so a 64-bit atomicMin keeps the closest hit with ties to the
// smaller id (kernels.py:353-357) and a sort of keys is the stable
// (t, id) order of np.argsort(kind="mergesort") (kernels.py:463).
__device__ __forceinline__ unsigned long long pack_hit(float t, int pid) {
    unsigned u = __float_as_uint(t);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (unsigned)pid;
}
__device__ __forceinline__ float unpack_t(unsigned long long v) {
    unsigned u = (unsigned)(v >> 32);
    u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
    return __uint_as_float(u);
}

// Child ordering keys: an fp32 entry distance as an orderable int with the
// child index in the low 2 bits.
__device__ __forceinline__ int ordered_key(float t, int k) {
    int i = __float_as_int(t);
    i = i >= 0 ? i : i ^ 0x7FFFFFFF;
    return (i & ~3) | k;
}
__device__ __forceinline__ float key_t(int key) {
    int ki = key & ~3;
    return __int_as_float(ki >= 0 ? ki : ki ^ 0x7FFFFFFF);
}

__device__ __forceinline__ int pick(const int4 &v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
// pick() for a run-time k as three selects (no branches)
__device__ __forceinline__ int sel4(const int4 &v, int k) {
    const int a = (k & 1) ? v.y : v.x;
    const int b = (k & 1) ? v.w : v.z;
    return (k & 2) ? b : a;
}

// ---------------------------------------------------------------------------
// counter RNG -- bitwise identical to oracle/srt_oracle.c
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t frame_key(uint32_t seed) { return mix32(seed ^ 0x9E3779B9u); }
__device__ __forceinline__ uint32_t walk_key(uint32_t fkey, uint32_t ray_id, uint32_t sample) {
    return mix32(mix32(fkey ^ ray_id) ^ sample);
}
// u in [0,1) with 24 bits; returned as the exact integer 0..2^24-1 scaled.
__device__ __forceinline__ float counter_u(uint32_t key, uint32_t prim) {
    uint32_t h = mix32(mix32(key ^ prim) ^ 0x68E31DA4u);
    return (float)(h >> 8) * (1.0f / 16777216.0f);
}

// ---------------------------------------------------------------------------
// Sobol pixel jitter (kernels.py:64-116), integer exact.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t wang32(uint32_t x) {
    x = (x ^ 61u) ^ (x >> 16);
    x = x * 9u;
    x = x ^ (x >> 4);
    x = x * 0x27D4EB2Du;
    x = x ^ (x >> 15);
    return x;
}
__device__ __forceinline__ uint32_t sobol_dim1(uint32_t index) {
    // direction numbers of x^2+x+1 generated on the fly (kernels.py:74-84)
    uint32_t y = 0, m = 1;
    for (int k = 0; index != 0; ++k, index >>= 1) {
        if (index & 1u) y ^= m << (31 - k);
        m = (m ^ (m << 1)) & (uint32_t)((2ull << (k + 1)) - 1ull);
    }
    return y;
}
// Returns the jitter (jx, jy) as exact doubles (32-bit fixed point).
__device__ __forceinline__ void pixel_jitter(uint32_t px, uint32_t py, uint32_t frame, uint32_t seed,
                                             double &jx, double &jy) {
    uint32_t base = wang32((px * 0x9E3779B1u) ^ (py * 0x85EBCA77u) ^ (seed * 0xC2B2AE3Du));
    uint32_t sx = wang32(base ^ 0x68E31DA4u);
    uint32_t sy = wang32(base ^ 0xB5297A4Du);
    uint32_t bx = __brev(frame);
    uint32_t by = sobol_dim1(frame);
    jx = (double)(bx ^ sx) * (1.0 / 4294967296.0);
    jy = (double)(by ^ sy) * (1.0 / 4294967296.0);
}

// Camera ray (kernels.py:613-618, 646-647) in fp64 with explicit IEEE
// rounding at every step (no FMA contraction), so the direction is bitwise
// equal to the oracle's.
struct CamD {
    double e[3], r[3], u[3], f[3];
    double half_w, half_h;
};
__device__ __forceinline__ void camera_ray(const CamD &c, uint32_t px, uint32_t py, uint32_t frame,
                                           uint32_t seed, int width, int height, double &dx, double &dy,
                                           double &dz) {
    double jx, jy;
    pixel_jitter(px, py, frame, seed, jx, jy);
    double u = __dsub_rn(__ddiv_rn(__dmul_rn(2.0, __dadd_rn((double)px, jx)), (double)width), 1.0);
    double v = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dadd_rn((double)py, jy)), (double)height));
    double uw = __dmul_rn(u, c.half_w), vh = __dmul_rn(v, c.half_h);
    double ddx = __dadd_rn(__dadd_rn(c.f[0], __dmul_rn(uw, c.r[0])), __dmul_rn(vh, c.u[0]));
    double ddy = __dadd_rn(__dadd_rn(c.f[1], __dmul_rn(uw, c.r[1])), __dmul_rn(vh, c.u[1]));
    double ddz = __dadd_rn(__dadd_rn(c.f[2], __dmul_rn(uw, c.r[2])), __dmul_rn(vh, c.u[2]));
    double nn = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)), __dmul_rn(ddz, ddz));
    double inv = __ddiv_rn(1.0, __dsqrt_rn(nn));
    dx = __dmul_rn(ddx, inv);
    dy = __dmul_rn(ddy, inv);
    dz = __dmul_rn(ddz, inv);
}

// ---------------------------------------------------------------------------
// Per-ray state for the traversal.
// ---------------------------------------------------------------------------
struct RayState {
    float fox, foy, foz;   // fp32 origin (stage-1 screen)
    float omag;            // max |o_i| (screen error model)
    double ox, oy, oz;     // origin (fp64, used by the candidate re-centring)
    double dx, dy, dz;     // direction (fp64)
    double inv_dd;         // 1 / |d|^2
    float fdx, fdy, fdz;   // fp32 direction (quadratic form)
    float idx, idy, idz;   // fp32 reciprocal direction (slab tests)
    float oidx, oidy, oidz;  // o * idir (slab tests as one FMA per plane)
    float t_min, t_max0;
};

__device__ __forceinline__ float safe_rcp(float d) {
    // zero direction components: a huge finite reciprocal keeps the slab
    // test exact-enough (kernels.py:276-279 treats d == 0 as 'inside slab')
    const float tiny = 1e-30f;
    if (fabsf(d) < tiny) d = copysignf(tiny, d);
    return 1.0f / d;
}

__device__ __forceinline__ void init_ray(RayState &r, double ox, double oy, double oz, double dx, double dy,
                                         double dz, double t_min, double t_max) {
    r.ox = ox; r.oy = oy; r.oz = oz;
    r.fox = (float)ox; r.foy = (float)oy; r.foz = (float)oz;
    r.omag = fmaxf(fabsf(r.fox), fmaxf(fabsf(r.foy), fabsf(r.foz)));
    r.dx = dx; r.dy = dy; r.dz = dz;
    r.inv_dd = 1.0 / (dx * dx + dy * dy + dz * dz);
    r.fdx = (float)dx; r.fdy = (float)dy; r.fdz = (float)dz;
    r.idx = safe_rcp(r.fdx); r.idy = safe_rcp(r.fdy); r.idz = safe_rcp(r.fdz);
    r.oidx = (float)ox * r.idx; r.oidy = (float)oy * r.idy; r.oidz = (float)oz * r.idz;
    // the candidate interval (t_min, t_max0) is open (kernels.py:349); fp32
    // bounds are rounded so they never exclude what fp64 would include
    r.t_min = (float)t_min;
    r.t_max0 = t_max >= 3.0e38 ? INFINITY : (float)t_max;
}

// Slab entry of both children of a node against [t_min, far] (closed,
// kernels.py:266-308).  Boxes are outward-rounded and inflated at build time.
__device__ __forceinline__ void slab2(const RayState &r, const float4 &xy0, const float4 &xy1, const float4 &z01,
                                      float far, float &e0, float &e1, bool &h0, bool &h1) {
    float x0a = fmaf(xy0.x, r.idx, -r.oidx), x0b = fmaf(xy0.y, r.idx, -r.oidx);
    float y0a = fmaf(xy0.z, r.idy, -r.oidy), y0b = fmaf(xy0.w, r.idy, -r.oidy);
    float z0a = fmaf(z01.x, r.idz, -r.oidz), z0b = fmaf(z01.y, r.idz, -r.oidz);
    float x1a = fmaf(xy1.x, r.idx, -r.oidx), x1b = fmaf(xy1.y, r.idx, -r.oidx);
    float y1a = fmaf(xy1.z, r.idy, -r.oidy), y1b = fmaf(xy1.w, r.idy, -r.oidy);
    float z1a = fmaf(z01.z, r.idz, -r.oidz), z1b = fmaf(z01.w, r.idz, -r.oidz);
    float n0 = fmaxf(fmaxf(fminf(x0a, x0b), fminf(y0a, y0b)), fmaxf(fminf(z0a, z0b), r.t_min));
    float f0 = fminf(fminf(fmaxf(x0a, x0b), fmaxf(y0a, y0b)), fminf(fmaxf(z0a, z0b), far));
    float n1 = fmaxf(fmaxf(fminf(x1a, x1b), fminf(y1a, y1b)), fmaxf(fminf(z1a, z1b), r.t_min));
    float f1 = fminf(fminf(fmaxf(x1a, x1b), fmaxf(y1a, y1b)), fminf(fmaxf(z1a, z1b), far));
    h0 = n0 <= f0;
    h1 = n1 <= f1;
    e0 = n0;
    e1 = n1;
}

// ---------------------------------------------------------------------------
// Candidate (kernels.py:139-189), re-centred: the ray is re-expressed from
// p = o + t0 d, t0 = (mu - o).d / |d|^2, the point nearest the mean, so the
// quadratic form is evaluated on a SMALL vector w = p - mu and fp32 keeps
// its accuracy.  t0 and w are formed in fp64 (the ray is fp64
// end to end); the 3x3 quadratic form runs in fp32.
// ---------------------------------------------------------------------------
struct Cand {
    float t;
    float alpha;
    int valid;
};

template <int MODE, class R, bool REFINE = true>
__device__ __forceinline__ Cand candidate(const R &r, const float4 &m, const float4 &a, const float4 &b,
                                          float s2) {
    Cand c;
    double vx = (double)m.x - r.ox, vy = (double)m.y - r.oy, vz = (double)m.z - r.oz;  // mu - o
    double tc = vx * r.dx + vy * r.dy + vz * r.dz;  // (mu - o).d  == center depth (mode 1)
    double t0 = tc * r.inv_dd;
    float wx = (float)(t0 * r.dx - vx), wy = (float)(t0 * r.dy - vy), wz = (float)(t0 * r.dz - vz);
    float a00 = a.x, a01 = a.y, a02 = a.z, a11 = a.w, a12 = b.x, a22 = b.y;
    float adx = a00 * r.fdx + a01 * r.fdy + a02 * r.fdz;
    float ady = a01 * r.fdx + a11 * r.fdy + a12 * r.fdz;
    float adz = a02 * r.fdx + a12 * r.fdy + a22 * r.fdz;
    float dad = r.fdx * adx + r.fdy * ady + r.fdz * adz;
    float awx = a00 * wx + a01 * wy + a02 * wz;
    float awy = a01 * wx + a11 * wy + a12 * wz;
    float awz = a02 * wx + a12 * wy + a22 * wz;
    float daw = r.fdx * awx + r.fdy * awy + r.fdz * awz;
    float waw = wx * awx + wy * awy + wz * awz;
    if (REFINE) {
        // second re-centring, at the estimated peak: there d.A.w vanishes and
        // w.A.w carries no cancellation even for very anisotropic A
        t0 = t0 - (double)(daw / dad);
        wx = (float)(t0 * r.dx - vx);
        wy = (float)(t0 * r.dy - vy);
        wz = (float)(t0 * r.dz - vz);
        awx = a00 * wx + a01 * wy + a02 * wz;
        awy = a01 * wx + a11 * wy + a12 * wz;
        awz = a02 * wx + a12 * wy + a22 * wz;
        daw = r.fdx * awx + r.fdy * awy + r.fdz * awz;
        waw = wx * awx + wy * awy + wz * awz;
    }
    float resid = fmaxf(waw - daw * daw / dad, 0.0f);
    float mah, t;
    if (MODE == 0) {
        t = (float)(t0 - (double)(daw / dad));
        mah = resid;
    } else {
        t = (float)tc;
        float s = (float)(tc - t0);
        float qx = wx + s * r.fdx, qy = wy + s * r.fdy, qz = wz + s * r.fdz;
        mah = qx * (a00 * qx + a01 * qy + a02 * qz) + qy * (a01 * qx + a11 * qy + a12 * qz) +
              qz * (a02 * qx + a12 * qy + a22 * qz);
    }
    // dad <= 0 or non-finite -> invalid (kernels.py:167-168); mah > s2 ->
    // outside the cutoff (kernels.py:187); open range (kernels.py:349)
    c.valid = (dad > 0.0f) && isfinite(dad) && isfinite(t) && (mah <= s2) && (t > r.t_min) && (t < r.t_max0);
    c.t = t;
    c.alpha = m.w * __expf(-0.5f * resid);
    return c;
}

// The fields of a ray the exact candidate reads (a light RayState).
struct ExactRay {
    double ox, oy, oz, dx, dy, dz, inv_dd;
    float fdx, fdy, fdz, t_min, t_max0;
};

// The screen's transcendentals without denormal handling (MUFU directly):
// exp2 flushes results below 2^-126 to 0 and rsqrt treats a denormal input
// as 0.  Both keep the screen's bounds conservative -- alpha_hi >= 1e-7 bounds
// any flushed alpha from above, a flushed alpha_lo only loosens the lower
// bound -- and a denormal d.A.d (an eigenvalue of A below 1e-38 along the ray,
// i.e. a primitive scale above 1e18) is the only input they change.
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float exp_ftz(float x) { return ex2_ftz(x * 1.4426950408889634f); }
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Stage-1 screen: the same quantities as `candidate` in plain fp32 (no
// fp64), with a conservative bound on their rounding error.  A candidate the
// screen rejects is certainly invalid or beyond `far`; `alpha_hi` bounds
// alpha from above, so a draw u >= alpha_hi is certainly a rejection and the
// exact fp64 evaluation can be skipped (it runs for ~1 candidate in 10).
struct Screen {
    float t_lo;      // lower bound of the candidate depth
    float alpha_hi;  // upper bound of alpha
    bool maybe;      // could be a valid candidate inside (t_min, far]
    float t;         // the screen's depth estimate
    // the bounds behind the decision below
    float mt, mah, mr, dad, alpha_base;  // alpha_base = opacity * exp(-max(resid - mr, 0) / 2)
    // Decided by the screen alone (no exact stage)?  True when the candidate
    // is valid for certain (dAd > 0, mah + error <= s^2, t +- error inside the
    // open interval); alpha_lo then bounds alpha from below.  Evaluated only
    // for the few candidates whose draw passed alpha_hi.
    __device__ __forceinline__ bool sure(float s2, float t_min, float t_max0) const {
        return (dad > 0.0f) && isfinite(dad) && (mah + mr <= s2) && (t - mt > t_min) && (t + mt < t_max0);
    }
    __device__ __forceinline__ float alpha_lo() const { return alpha_base * exp_ftz(-mr) * 0.9999f - 1e-7f; }
};

// Minimal fp32 ray for the screen (camera rays share one origin).
struct ScreenRay {
    float fox, foy, foz, omag;
    float fdx, fdy, fdz;
    double inv_dd;
    float t_min, t_max0;
};

template <int MODE, class R>
__device__ __forceinline__ Screen screen(const R &r, const float4 &m, const float4 &a, const float4 &b,
                                         float s2, float sqrt_s2, float far) {
    Screen sc;
    float vx = m.x - r.fox, vy = m.y - r.foy, vz = m.z - r.foz;
    float tc = vx * r.fdx + vy * r.fdy + vz * r.fdz;
    float t0 = tc * (float)r.inv_dd;
    float wx = fmaf(t0, r.fdx, -vx), wy = fmaf(t0, r.fdy, -vy), wz = fmaf(t0, r.fdz, -vz);
    float a00 = a.x, a01 = a.y, a02 = a.z, a11 = a.w, a12 = b.x, a22 = b.y;
    float adx = a00 * r.fdx + a01 * r.fdy + a02 * r.fdz;
    float ady = a01 * r.fdx + a11 * r.fdy + a12 * r.fdz;
    float adz = a02 * r.fdx + a12 * r.fdy + a22 * r.fdz;
    float dad = r.fdx * adx + r.fdy * ady + r.fdz * adz;
    float awx = a00 * wx + a01 * wy + a02 * wz;
    float awy = a01 * wx + a11 * wy + a12 * wz;
    float awz = a02 * wx + a12 * wy + a22 * wz;
    float daw = r.fdx * awx + r.fdy * awy + r.fdz * awz;
    float waw = wx * awx + wy * awy + wz * awz;
    float rs = rsqrt_ftz(dad);
    float inv_dad = rs * rs;
    float resid = waw - daw * daw * inv_dad;
    float mah, t;
    // absolute error of w: roundings of |o|-, |mu|- and |t0|-sized terms
    // (|mu| <= |mu - o| + |o|); sqrt_tr = sqrt(sum |a_ij|) bounds sqrt(lambda_max)
    float sqrt_tr = b.w;
    float e = 4.0e-7f * (fabsf(t0) + 2.0f * r.omag + fabsf(vx) + fabsf(vy) + fabsf(vz)) + 1e-30f;
    float es = e * sqrt_tr;
    float mr = es * (4.0f * sqrt_s2 + 4.0f * es) + 2.0e-5f * (fabsf(waw) + 1e-6f);
    if (MODE == 0) {
        t = t0 - daw * inv_dad;
        mah = resid;
    } else {
        t = tc;
        float sd = tc - t0;
        float qx = fmaf(sd, r.fdx, wx), qy = fmaf(sd, r.fdy, wy), qz = fmaf(sd, r.fdz, wz);
        mah = qx * (a00 * qx + a01 * qy + a02 * qz) + qy * (a01 * qx + a11 * qy + a12 * qz) +
              qz * (a02 * qx + a12 * qy + a22 * qz);
        mr += 2.0e-5f * fabsf(mah);
    }
    float mt = e + es * rs + 2.0e-6f * (fabsf(t) + 1.0f);
    sc.t_lo = t - mt;
    sc.maybe = (dad > 0.0f) && (mah - mr <= s2) && (t - mt <= far) && (t + mt > r.t_min) && (t - mt < r.t_max0);
    sc.alpha_base = m.w * exp_ftz(-0.5f * fmaxf(resid - mr, 0.0f));
    sc.alpha_hi = sc.alpha_base * 1.0001f + 1e-7f;
    // alpha_lo(): the same error terms the other way (exp(-mr) widens the
    // band by the residual's bound; the opacity is fp32-rounded)
    sc.t = t;
    sc.mt = mt;
    sc.mah = mah;
    sc.mr = mr;
    sc.dad = dad;
    return sc;
}

// SH colour (kernels.py:193-257) in fp32 on the ray direction.
__device__ __forceinline__ float3 sh_color(const float *__restrict__ sh, int K, int deg, int pid, float x, float y,
                                           float z) {
    const float SH_C0 = 0.28209479177387814f, SH_C1 = 0.4886025119029199f;
    const float C2_0 = 1.0925484305920792f, C2_1 = -1.0925484305920792f, C2_2 = 0.31539156525252005f,
                C2_3 = -1.0925484305920792f, C2_4 = 0.5462742152960396f;
    const float C3_0 = -0.5900435899266435f, C3_1 = 2.890611442640554f, C3_2 = -0.4570457994644658f,
                C3_3 = 0.3731763325901154f, C3_4 = -0.4570457994644658f, C3_5 = 1.445305721320277f,
                C3_6 = -0.5900435899266435f;
    const float *s = sh + (int64_t)pid * 3 * K;
    float out[3];
    float xx = x * x, yy = y * y, zz = z * z;
    float b0 = x * y, b1 = y * z, b2 = 2.0f * zz - xx - yy, b3 = x * z, b4 = xx - yy;
    float c0 = y * (3.0f * xx - yy), c1 = b0 * z, c2 = y * (4.0f * zz - xx - yy),
          c3 = z * (2.0f * zz - 3.0f * xx - 3.0f * yy), c4 = x * (4.0f * zz - xx - yy), c5 = z * b4,
          c6 = x * (xx - 3.0f * yy);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float *q = s + ch * K;
        float v = SH_C0 * __ldg(q);
        if (deg >= 1) v = v - SH_C1 * y * __ldg(q + 1) + SH_C1 * z * __ldg(q + 2) - SH_C1 * x * __ldg(q + 3);
        if (deg >= 2)
            v += C2_0 * b0 * __ldg(q + 4) + C2_1 * b1 * __ldg(q + 5) + C2_2 * b2 * __ldg(q + 6) +
                 C2_3 * b3 * __ldg(q + 7) + C2_4 * b4 * __ldg(q + 8);
        if (deg >= 3)
            v += C3_0 * c0 * __ldg(q + 9) + C3_1 * c1 * __ldg(q + 10) + C3_2 * c2 * __ldg(q + 11) +
                 C3_3 * c3 * __ldg(q + 12) + C3_4 * c4 * __ldg(q + 13) + C3_5 * c5 * __ldg(q + 14) +
                 C3_6 * c6 * __ldg(q + 15);
        out[ch] = fmaxf(v + 0.5f, 0.0f);
    }
    return make_float3(out[0], out[1], out[2]);
}

// sh_color for degree 3 with the 48 coefficients fetched as 12 128-bit loads
// (a record is 192 B, 16-B aligned); the same expressions, so the same
// result bit for bit.  Other degrees take sh_color.
__device__ __forceinline__ float3 sh_color_v(const float *__restrict__ sh, int K, int deg, int pid, float x, float y,
                                             float z) {
    if (deg != 3) return sh_color(sh, K, deg, pid, x, y, z);
    const float SH_C0 = 0.28209479177387814f, SH_C1 = 0.4886025119029199f;
    const float C2_0 = 1.0925484305920792f, C2_1 = -1.0925484305920792f, C2_2 = 0.31539156525252005f,
                C2_3 = -1.0925484305920792f, C2_4 = 0.5462742152960396f;
    const float C3_0 = -0.5900435899266435f, C3_1 = 2.890611442640554f, C3_2 = -0.4570457994644658f,
                C3_3 = 0.3731763325901154f, C3_4 = -0.4570457994644658f, C3_5 = 1.445305721320277f,
                C3_6 = -0.5900435899266435f;
    const float4 *s4 = reinterpret_cast<const float4 *>(sh + (int64_t)pid * 48);
    float f[48];
#pragma unroll
    for (int j = 0; j < 12; ++j) {
        const float4 v = __ldg(s4 + j);
        f[4 * j] = v.x, f[4 * j + 1] = v.y, f[4 * j + 2] = v.z, f[4 * j + 3] = v.w;
    }
    float out[3];
    float xx = x * x, yy = y * y, zz = z * z;
    float b0 = x * y, b1 = y * z, b2 = 2.0f * zz - xx - yy, b3 = x * z, b4 = xx - yy;
    float c0 = y * (3.0f * xx - yy), c1 = b0 * z, c2 = y * (4.0f * zz - xx - yy),
          c3 = z * (2.0f * zz - 3.0f * xx - 3.0f * yy), c4 = x * (4.0f * zz - xx - yy), c5 = z * b4,
          c6 = x * (xx - 3.0f * yy);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float *q = f + ch * 16;
        float v = SH_C0 * q[0];
        v = v - SH_C1 * y * q[1] + SH_C1 * z * q[2] - SH_C1 * x * q[3];
        v += C2_0 * b0 * q[4] + C2_1 * b1 * q[5] + C2_2 * b2 * q[6] + C2_3 * b3 * q[7] + C2_4 * b4 * q[8];
        v += C3_0 * c0 * q[9] + C3_1 * c1 * q[10] + C3_2 * c2 * q[11] + C3_3 * c3 * q[12] + C3_4 * c4 * q[13] +
             C3_5 * c5 * q[14] + C3_6 * c6 * q[15];
        out[ch] = fmaxf(v + 0.5f, 0.0f);
    }
    return make_float3(out[0], out[1], out[2]);
}

}  // namespace srt
