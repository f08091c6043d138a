// lbvh.cu -- GPU LBVH build (north-star subsystem 1), replacing the
// reference's single-threaded Python binned-SAH build (bvh.py:87-193).
//
//   1. k_prim_boxes   per-primitive AABB of the cutoff ellipsoid
//                     {x : (x-mu)^T A (x-mu) <= s^2}: half extent_i =
//                     s*sqrt(Sigma_ii), Sigma = A^-1 (fp64), rounded outward
//                     to fp32 and inflated (conservative slab tests).  Any
//                     superset of the ellipsoid is correct: a valid candidate
//                     peaks inside the ellipsoid (kernels.py:187), hence
//                     inside its box.  Also the centroid bounds (atomics).
//   2. k_morton       63-bit Morton code of the box centroid (21 bits/axis).
//   3. CUB radix sort of (code, prim) pairs.
//   4. k_karras       Karras (HPG 2012) binary radix tree over the sorted
//                     codes; duplicate codes are disambiguated by index.
//   5. k_refit        bottom-up: the second thread to reach a node writes
//                     the node's Node2 (both children's boxes) and its union.
//   6. k_geom         primitive records permuted into leaf ("slot") order.
// With method SRT_BVH_PLOC, steps 4-5 are replaced by agglomerative PLOC
// clustering over the same Morton order (ploc.cu).
#include <functional>
#include <vector>
#include <cstring>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cub/device/device_radix_sort.cuh>

#include "srt_internal.h"

namespace srt {

__device__ __forceinline__ int ordered_int(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float from_ordered(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

__device__ __forceinline__ float lo32(double x) {
    float f = __double2float_rd(x);
    return f - (fabsf(f) * 9.5367431640625e-07f + 1e-30f);  // 2^-20 relative inflation
}
__device__ __forceinline__ float hi32(double x) {
    float f = __double2float_ru(x);
    return f + (fabsf(f) * 9.5367431640625e-07f + 1e-30f);
}

__global__ void k_prim_boxes(int64_t n, const double *__restrict__ means, const double *__restrict__ cov6, double s,
                             float *lo, float *hi, int *cbounds) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (i < n) {
        const double *c = cov6 + i * 6;
        double a00 = c[0], a01 = c[1], a02 = c[2], a11 = c[3], a12 = c[4], a22 = c[5];
        // Sigma = adj(A) / det(A); only the diagonal is needed
        double c00 = a11 * a22 - a12 * a12;
        double c11 = a00 * a22 - a02 * a02;
        double c22 = a00 * a11 - a01 * a01;
        double det = a00 * c00 - a01 * (a01 * a22 - a12 * a02) + a02 * (a01 * a12 - a11 * a02);
        double sd[3] = {c00 / det, c11 / det, c22 / det};
        for (int k = 0; k < 3; ++k) {
            double m = means[i * 3 + k];
            double h = s * sqrt(sd[k]);
            float l, u;
            if (!(h >= 0.0) || !isfinite(h)) {
                // degenerate: the box must not reject anything; the candidate
                // test (dAd <= 0 etc.) decides
                l = -3.0e38f;
                u = 3.0e38f;
            } else {
                l = lo32(m - h);
                u = hi32(m + h);
            }
            lo[i * 3 + k] = l;
            hi[i * 3 + k] = u;
            cmin[k] = (float)m;  // Morton codes use the mean (the box centre)
            cmax[k] = (float)m;
        }
    }
    // block reduce via warp shuffles then one atomic per warp
    for (int k = 0; k < 3; ++k) {
        float a = cmin[k], b = cmax[k];
        for (int o = 16; o > 0; o >>= 1) {
            a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0 && a <= b) {
            atomicMin(cbounds + k, ordered_int(a));
            atomicMax(cbounds + 3 + k, ordered_int(b));
        }
    }
}

__device__ __forceinline__ uint64_t spread21(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

__global__ void k_morton(int64_t n, const double *__restrict__ means, const int *cbounds, uint64_t *keys,
                         uint32_t *vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t code = 0;
    for (int k = 0; k < 3; ++k) {
        float lo = from_ordered(cbounds[k]), hi = from_ordered(cbounds[3 + k]);
        float ext = hi - lo;
        float c = (float)means[i * 3 + k];
        float u = ext > 0.f ? (c - lo) / ext : 0.5f;
        u = fminf(fmaxf(u, 0.f), 1.f);
        uint64_t q = (uint64_t)fminf(u * 2097152.0f, 2097151.0f);
        code |= spread21(q) << (2 - k);
    }
    keys[i] = code;
    vals[i] = (uint32_t)i;
}

__device__ __forceinline__ int delta(const uint64_t *keys, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = keys[i], b = keys[j];
    if (a == b) return 64 + __clzll((unsigned long long)(i ^ j));
    return __clzll((unsigned long long)(a ^ b));
}

// internal node i in [0, n-2]; children: >=0 internal, <0 leaf ~slot
__global__ void k_karras(int64_t n, const uint64_t *__restrict__ keys, int2 *children, int *parent_int,
                         int *parent_leaf) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int64_t lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int64_t j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int64_t s = 0;
    int64_t t = l;
    do {
        t = (t + 1) / 2;
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
    int64_t first = i < j ? i : j, last = i < j ? j : i;
    int left, right;
    if (first == gamma) {
        left = ~(int)gamma;
        parent_leaf[gamma] = (int)i;
    } else {
        left = (int)gamma;
        parent_int[gamma] = (int)i;
    }
    if (last == gamma + 1) {
        right = ~(int)(gamma + 1);
        parent_leaf[gamma + 1] = (int)i;
    } else {
        right = (int)(gamma + 1);
        parent_int[gamma + 1] = (int)i;
    }
    children[i] = make_int2(left, right);
}

struct Box6 {
    float lo[3], hi[3];
};

__device__ __forceinline__ Box6 load_child_box(int code, const float *plo, const float *phi,
                                               const uint32_t *slot_prim, const float *ibox) {
    Box6 b;
    if (code < 0) {
        int64_t p = slot_prim[~code];
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = plo[p * 3 + k];
            b.hi[k] = phi[p * 3 + k];
        }
    } else {
        // written by another thread of this kernel: bypass L1
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = __ldcg(ibox + (int64_t)code * 6 + k);
            b.hi[k] = __ldcg(ibox + (int64_t)code * 6 + 3 + k);
        }
    }
    return b;
}

__global__ void k_refit(int64_t n, const int2 *__restrict__ children, const int *__restrict__ parent_int,
                        const int *__restrict__ parent_leaf, const float *__restrict__ plo,
                        const float *__restrict__ phi, const uint32_t *__restrict__ slot_prim, float *ibox,
                        int *flags, Node2 *nodes) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int node = parent_leaf[j];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(flags + node, 1) == 0) return;  // sibling subtree not finished yet
        __threadfence();
        int2 ch = children[node];
        Box6 a = load_child_box(ch.x, plo, phi, slot_prim, ibox);
        Box6 b = load_child_box(ch.y, plo, phi, slot_prim, ibox);
        Node2 nd;
        nd.xy0 = make_float4(a.lo[0], a.hi[0], a.lo[1], a.hi[1]);
        nd.xy1 = make_float4(b.lo[0], b.hi[0], b.lo[1], b.hi[1]);
        nd.z01 = make_float4(a.lo[2], a.hi[2], b.lo[2], b.hi[2]);
        nd.kids = make_int4(ch.x, ch.y, 0, 0);
        nodes[node] = nd;
        for (int k = 0; k < 3; ++k) {
            __stcg(ibox + (int64_t)node * 6 + k, fminf(a.lo[k], b.lo[k]));
            __stcg(ibox + (int64_t)node * 6 + 3 + k, fmaxf(a.hi[k], b.hi[k]));
        }
        node = parent_int[node];  // root's parent is -1
    }
}

// tree depth in nodes (leaf level included): max over leaves of the path length
__global__ void k_depth(int64_t n, const int *__restrict__ parent_int, const int *__restrict__ parent_leaf,
                        int *depth_out) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int d = 1;
    for (int node = parent_leaf[j]; node >= 0; node = parent_int[node]) ++d;
    atomicMax(depth_out, d);
}

// geometry records in slot order; fp64 -> fp32
__global__ void k_geom(int64_t n, const uint32_t *__restrict__ slot_prim, const double *__restrict__ means,
                       const double *__restrict__ cov6, const double *__restrict__ opac, Geom *geom) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int64_t p = slot_prim[j];
    Geom g;
    g.m = make_float4((float)means[p * 3], (float)means[p * 3 + 1], (float)means[p * 3 + 2], (float)opac[p]);
    const double *c = cov6 + p * 6;
    g.a = make_float4((float)c[0], (float)c[1], (float)c[2], (float)c[3]);
    double tr = fabs(c[0]) + fabs(c[3]) + fabs(c[5]) + 2.0 * (fabs(c[1]) + fabs(c[2]) + fabs(c[4]));
    g.b = make_float4((float)c[4], (float)c[5], __int_as_float((int)p), (float)(sqrt(tr) * 1.0000002));
    geom[j] = g;
}

// single-primitive tree: one node, child0 = leaf 0, child1 = empty
__global__ void k_single(const float *plo, const float *phi, Node2 *nodes) {
    Node2 nd;
    nd.xy0 = make_float4(plo[0], phi[0], plo[1], phi[1]);
    nd.xy1 = make_float4(3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f);
    nd.z01 = make_float4(plo[2], phi[2], 3.0e38f, -3.0e38f);
    nd.kids = make_int4(~0, kLeafEmpty, 0, 0);
    nodes[0] = nd;
}

srt_status launch_geom(int64_t n, const uint32_t *slot_prim, const SrtScene *s, Geom *out, cudaStream_t st) {
    if (n <= 0) return SRT_OK;
    k_geom<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, slot_prim, s->d_means, s->d_cov6, s->d_opac, out);
    return cuda_status(cudaGetLastError(), "k_geom");
}

template <typename T>
static srt_status dalloc(T **p, size_t count, const char *what) {
    cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (count ? count : 1));
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc failed for ") + what + ": " + cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SRT_ERR_OOM : SRT_ERR_CUDA;
    }
    return SRT_OK;
}

srt_status lbvh_build(SrtScene *s, double cutoff_s, int method) {
    const int64_t n = s->n;
    cudaStream_t st = s->stream;
    free_split(s);
    if (s->d_nodes) cudaFree(s->d_nodes);
    if (s->d_geom) cudaFree(s->d_geom);
    s->d_nodes = nullptr;
    s->d_geom = nullptr;
    s->has_bvh = false;
    s->num_nodes = 0;
    s->depth = 0;
    if (n == 0) {
        s->has_bvh = true;
        return SRT_OK;
    }
    if (n > (int64_t)INT32_MAX / 2) {
        set_error("too many primitives for 32-bit node indices");
        return SRT_ERR_INVALID_ARG;
    }
    float *plo = nullptr, *phi = nullptr, *ibox = nullptr;
    int *cb = nullptr, *parent_int = nullptr, *parent_leaf = nullptr, *flags = nullptr, *ddepth = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    uint32_t *vals = nullptr, *vals2 = nullptr;
    int2 *children = nullptr;
    void *temp = nullptr;
    size_t temp_bytes = 0;
    srt_status rc = SRT_OK;
    const unsigned B = 256;
    const unsigned G = (unsigned)((n + B - 1) / B);
    int cb_init[6];
    int h_depth = 0;
#define SRT_TRY(x)          \
    do {                    \
        rc = (x);           \
        if (rc) goto done;  \
    } while (0)
    SRT_TRY(dalloc(&plo, n * 3, "prim lo"));
    SRT_TRY(dalloc(&phi, n * 3, "prim hi"));
    SRT_TRY(dalloc(&cb, 6, "bounds"));
    SRT_TRY(dalloc(&keys, n, "keys"));
    SRT_TRY(dalloc(&keys2, n, "keys"));
    SRT_TRY(dalloc(&vals, n, "vals"));
    SRT_TRY(dalloc(&vals2, n, "vals"));
    SRT_TRY(dalloc(&s->d_geom, n, "geom"));
    SRT_TRY(dalloc(&ddepth, 1, "depth"));
    for (int k = 0; k < 3; ++k) {
        cb_init[k] = 0x7FFFFFFF;       // ordered +max
        cb_init[3 + k] = (int)0x80000000;  // ordered -max
    }
    SRT_TRY(cuda_status(cudaMemcpyAsync(cb, cb_init, sizeof(cb_init), cudaMemcpyHostToDevice, st), "bounds init"));
    k_prim_boxes<<<G, B, 0, st>>>(n, s->d_means, s->d_cov6, cutoff_s, plo, phi, cb);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_prim_boxes"));
    k_morton<<<G, B, 0, st>>>(n, s->d_means, cb, keys, vals);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_morton"));
    SRT_TRY(cuda_status(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, keys2, vals, vals2, (int)n, 0, 63, st),
                        "radix sort sizing"));
    SRT_TRY(dalloc((char **)&temp, temp_bytes, "sort temp"));
    SRT_TRY(cuda_status(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys2, vals, vals2, (int)n, 0, 63, st),
                        "radix sort"));
    k_geom<<<G, B, 0, st>>>(n, vals2, s->d_means, s->d_cov6, s->d_opac, s->d_geom);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_geom"));
    if (n == 1) {
        SRT_TRY(dalloc(&s->d_nodes, 1, "nodes"));
        k_single<<<1, 1, 0, st>>>(plo, phi, s->d_nodes);
        SRT_TRY(cuda_status(cudaGetLastError(), "k_single"));
        s->num_nodes = 1;
        s->depth = 2;
    } else {
        const int64_t m = n - 1;
        SRT_TRY(dalloc(&s->d_nodes, m, "nodes"));
        SRT_TRY(dalloc(&children, m, "children"));
        SRT_TRY(dalloc(&parent_int, m, "parents"));
        SRT_TRY(dalloc(&parent_leaf, n, "parents"));
        SRT_TRY(dalloc(&flags, m, "flags"));
        SRT_TRY(dalloc(&ibox, m * 6, "internal boxes"));
        SRT_TRY(cuda_status(cudaMemsetAsync(flags, 0, sizeof(int) * m, st), "flags"));
        SRT_TRY(cuda_status(cudaMemsetAsync(ddepth, 0, sizeof(int), st), "depth"));
        SRT_TRY(cuda_status(cudaMemsetAsync(parent_int, 0xFF, sizeof(int) * m, st), "parents"));
        if (method == SRT_BVH_PLOC) {
            SRT_TRY(ploc_build(s, n, vals2, plo, phi, parent_int, parent_leaf, st, s->d_nodes));
        } else {
            k_karras<<<(unsigned)((m + B - 1) / B), B, 0, st>>>(n, keys2, children, parent_int, parent_leaf);
            SRT_TRY(cuda_status(cudaGetLastError(), "k_karras"));
            k_refit<<<G, B, 0, st>>>(n, children, parent_int, parent_leaf, plo, phi, vals2, ibox, flags, s->d_nodes);
            SRT_TRY(cuda_status(cudaGetLastError(), "k_refit"));
        }
        k_depth<<<G, B, 0, st>>>(n, parent_int, parent_leaf, ddepth);
        SRT_TRY(cuda_status(cudaGetLastError(), "k_depth"));
        SRT_TRY(cuda_status(cudaMemcpyAsync(&h_depth, ddepth, sizeof(int), cudaMemcpyDeviceToHost, st), "depth"));
        SRT_TRY(cuda_status(cudaStreamSynchronize(st), "lbvh build"));
        s->num_nodes = (int32_t)m;
        s->depth = h_depth;
    }
    SRT_TRY(cuda_status(cudaStreamSynchronize(st), "lbvh build"));
    SRT_TRY(collapse4(s));
    // the packet walk's spatially split copy (PLOC builds of large scenes)
    free_split(s);
    if (method == SRT_BVH_PLOC) SRT_TRY(split_build(s, plo, phi, cb, st));
    s->has_bvh = true;
done:
#undef SRT_TRY
    cudaFree(plo);
    cudaFree(phi);
    cudaFree(cb);
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(vals);
    cudaFree(vals2);
    cudaFree(children);
    cudaFree(parent_int);
    cudaFree(parent_leaf);
    cudaFree(flags);
    cudaFree(ibox);
    cudaFree(ddepth);
    cudaFree(temp);
    return rc;
}

}  // namespace srt

// ---------------------------------------------------------------------------
// Binary -> 4-wide collapse.  Each 4-wide node starts from a binary node's two
// children and repeatedly opens the inner child with the largest surface
// area until it holds 4 children (or only leaves remain).  Breadth-first
// waves over a device worklist; boxes come from the parents' Node2 records.
// ---------------------------------------------------------------------------
namespace srt {

struct Entry4 {
    int code;
    float lo[3], hi[3];
};

__host__ __device__ __forceinline__ void node2_child(const Node2 &nd, int c, Entry4 &e) {
    if (c == 0) {
        e.code = nd.kids.x;
        e.lo[0] = nd.xy0.x; e.hi[0] = nd.xy0.y; e.lo[1] = nd.xy0.z; e.hi[1] = nd.xy0.w;
        e.lo[2] = nd.z01.x; e.hi[2] = nd.z01.y;
    } else {
        e.code = nd.kids.y;
        e.lo[0] = nd.xy1.x; e.hi[0] = nd.xy1.y; e.lo[1] = nd.xy1.z; e.hi[1] = nd.xy1.w;
        e.lo[2] = nd.z01.z; e.hi[2] = nd.z01.w;
    }
}

__host__ __device__ __forceinline__ float area(const Entry4 &e) {
    float dx = e.hi[0] - e.lo[0], dy = e.hi[1] - e.lo[1], dz = e.hi[2] - e.lo[2];
    return dx * dy + dy * dz + dz * dx;
}

// Node4 record from up to 4 child entries (boxes) and their final codes (inner
// node4 index, leaf ~slot, kLeafEmpty), with the traversal hints: valid / leaf
// child masks and, for each of the 8 ray direction octants, the children
// ordered near-to-far along that octant's diagonal (2 bits per child).
__host__ __device__ inline void make_node4(Node4 &o, const Entry4 *e, int cnt, const int *kids) {
    float lo[3][4], hi[3][4];
    for (int k = 0; k < 4; ++k)
        for (int a = 0; a < 3; ++a) {
            lo[a][k] = k < cnt ? e[k].lo[a] : 3.0e38f;
            hi[a][k] = k < cnt ? e[k].hi[a] : -3.0e38f;
        }
    o.lox = make_float4(lo[0][0], lo[0][1], lo[0][2], lo[0][3]);
    o.hix = make_float4(hi[0][0], hi[0][1], hi[0][2], hi[0][3]);
    o.loy = make_float4(lo[1][0], lo[1][1], lo[1][2], lo[1][3]);
    o.hiy = make_float4(hi[1][0], hi[1][1], hi[1][2], hi[1][3]);
    o.loz = make_float4(lo[2][0], lo[2][1], lo[2][2], lo[2][3]);
    o.hiz = make_float4(hi[2][0], hi[2][1], hi[2][2], hi[2][3]);
    o.kids = make_int4(kids[0], kids[1], kids[2], kids[3]);
    unsigned validm = 0, leafm = 0;
    float ctr[4][3];
    for (int k = 0; k < 4; ++k) {
        if (kids[k] != kLeafEmpty) validm |= 1u << k;
        if (kids[k] < 0 && kids[k] != kLeafEmpty) leafm |= 1u << k;
        for (int a = 0; a < 3; ++a) ctr[k][a] = 0.5f * (lo[a][k] + hi[a][k]);
    }
    unsigned ord[2] = {0, 0};
    for (int oc = 0; oc < 8; ++oc) {
        float dir[3] = {(oc & 1) ? -1.f : 1.f, (oc & 2) ? -1.f : 1.f, (oc & 4) ? -1.f : 1.f};
        float key[4];
        int idx[4] = {0, 1, 2, 3};
        for (int k = 0; k < 4; ++k)
            key[k] = (validm >> k) & 1u ? ctr[k][0] * dir[0] + ctr[k][1] * dir[1] + ctr[k][2] * dir[2] : 3.0e38f;
        for (int i = 1; i < 4; ++i)  // insertion sort of 4
            for (int j = i; j > 0 && key[idx[j]] < key[idx[j - 1]]; --j) {
                int t = idx[j];
                idx[j] = idx[j - 1];
                idx[j - 1] = t;
            }
        unsigned byte = idx[0] | (idx[1] << 2) | (idx[2] << 4) | (idx[3] << 6);
        ord[oc >> 2] |= byte << ((oc & 3) * 8);
    }
    o.pad = make_int4((int)(validm | (leafm << 4)), (int)ord[0], (int)ord[1], cnt);
}

// work item: (binary node id, 4-wide node index)
__global__ void k_collapse4(const Node2 *__restrict__ n2, const int2 *__restrict__ work_in, int n_in,
                            int2 *work_out, int *n_out, int *n4_count, Node4 *n4) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_in) return;
    int2 w = work_in[i];
    Entry4 e[4];
    int cnt = 0;
    Node2 root = n2[w.x];
    for (int c = 0; c < 2; ++c) {
        node2_child(root, c, e[cnt]);
        if (e[cnt].code != kLeafEmpty) ++cnt;
    }
    while (cnt < 4) {
        int best = -1;
        float ba = -1.f;
        for (int k = 0; k < cnt; ++k)
            if (e[k].code >= 0 && area(e[k]) > ba) {
                ba = area(e[k]);
                best = k;
            }
        if (best < 0) break;
        Node2 nd = n2[e[best].code];
        Entry4 a, b;
        node2_child(nd, 0, a);
        node2_child(nd, 1, b);
        if (a.code == kLeafEmpty) {
            e[best] = b;
        } else if (b.code == kLeafEmpty) {
            e[best] = a;
        } else {
            e[best] = a;
            e[cnt++] = b;
        }
    }
    int ninner = 0;
    for (int k = 0; k < cnt; ++k) ninner += e[k].code >= 0;
    int base4 = ninner ? atomicAdd(n4_count, ninner) : 0;
    int basew = ninner ? atomicAdd(n_out, ninner) : 0;
    int kids[4];
    int j = 0;
    for (int k = 0; k < 4; ++k) {
        if (k < cnt && e[k].code >= 0) {
            kids[k] = base4 + j;
            work_out[basew + j] = make_int2(e[k].code, base4 + j);
            ++j;
        } else {
            kids[k] = k < cnt ? e[k].code : kLeafEmpty;
        }
    }
    Node4 o;
    make_node4(o, e, cnt, kids);
    n4[w.y] = o;
}

// ---------------------------------------------------------------------------
// Cost-optimal collapse (host dynamic programme over the binary tree, after
// Ylitie et al. 2017's wide-BVH collapse).  For binary node x with children
// a, b and slot counts j = 1..4:
//   F(x, 1) = T(x)  (x becomes a 4-wide node)      F(leaf, 1) = A(leaf) * cj
//   F(x, j) = G(x, j) = min_{j1 + j2 = j} F(a, j1) + F(b, j2)   (x opened)
//   T(x)    = A(x) * cv + min_{j = 2..4} [A(x) * ct * j + G(x, j)]
// with A the box surface area (visit probability), cv the cost of visiting a
// node, ct of testing one child box, cj of one leaf job.  The 4-wide tree is
// then emitted top-down (breadth first) following the argmins.
// ---------------------------------------------------------------------------
[[maybe_unused]] static srt_status collapse4_dp(SrtScene *s, float cv, float ct, float cj) {
    const int m2 = s->num_nodes;
    std::vector<Node2> n2(m2);
    srt_status rc = cuda_status(cudaMemcpy(n2.data(), s->d_nodes, sizeof(Node2) * m2, cudaMemcpyDeviceToHost),
                                "node download");
    if (rc) return rc;
    const float INF = INFINITY;
    std::vector<float> F((size_t)m2 * 4, INF);
    std::vector<signed char> split((size_t)m2 * 4, 1), bestj(m2, 2);
    auto childF = [&](const Entry4 &e, int j) -> float {  // j = 1..4
        if (e.code == kLeafEmpty) return INF;
        if (e.code < 0) return j == 1 ? area(e) * cj : INF;
        return F[(size_t)e.code * 4 + (j - 1)];
    };
    // post-order over the binary tree from the root (node 0)
    std::vector<int> order;
    order.reserve(m2);
    {
        std::vector<int> stk{0};
        while (!stk.empty()) {
            int x = stk.back();
            stk.pop_back();
            order.push_back(x);
            for (int c = 0; c < 2; ++c) {
                int code = c == 0 ? n2[x].kids.x : n2[x].kids.y;
                if (code >= 0) stk.push_back(code);
            }
        }
    }
    for (int oi = (int)order.size() - 1; oi >= 0; --oi) {
        const int x = order[oi];
        Entry4 a, b;
        node2_child(n2[x], 0, a);
        node2_child(n2[x], 1, b);
        Entry4 u = a;
        if (b.code != kLeafEmpty)
            for (int k = 0; k < 3; ++k) {
                u.lo[k] = a.code == kLeafEmpty ? b.lo[k] : std::min(a.lo[k], b.lo[k]);
                u.hi[k] = a.code == kLeafEmpty ? b.hi[k] : std::max(a.hi[k], b.hi[k]);
            }
        const float A = area(u);
        float G[5] = {INF, INF, INF, INF, INF};
        for (int j = 1; j <= 4; ++j) {
            if (a.code == kLeafEmpty || b.code == kLeafEmpty) {  // single child (one-primitive trees)
                G[j] = childF(a.code == kLeafEmpty ? b : a, j);
                split[(size_t)x * 4 + j - 1] = (signed char)(a.code == kLeafEmpty ? 0 : j);
                continue;
            }
            for (int j1 = 1; j1 < j; ++j1) {
                float c = childF(a, j1) + childF(b, j - j1);
                if (c < G[j]) {
                    G[j] = c;
                    split[(size_t)x * 4 + j - 1] = (signed char)j1;
                }
            }
        }
        float best = INF;
        int bj = 2;
        for (int j = 1; j <= 4; ++j) {
            float c = A * ct * (float)j + G[j];
            if (c < best) {
                best = c;
                bj = j;
            }
        }
        if (!(best < INF)) bj = (a.code == kLeafEmpty || b.code == kLeafEmpty) ? 1 : 2;  // unbounded boxes
        bestj[x] = (signed char)bj;
        F[(size_t)x * 4 + 0] = A * cv + best;
        for (int j = 2; j <= 4; ++j) F[(size_t)x * 4 + j - 1] = G[j];
    }
    // top-down emission, breadth first: node4 index 0 is the root
    std::vector<Node4> out;
    out.reserve(m2);
    std::vector<int> queue{0};
    std::vector<Entry4> slots;
    // expand entry e (a child box + code) into j slots
    std::function<void(const Entry4 &, int)> expand = [&](const Entry4 &e, int j) {
        if (j == 1 || e.code < 0) {
            slots.push_back(e);
            return;
        }
        Entry4 a, b;
        node2_child(n2[e.code], 0, a);
        node2_child(n2[e.code], 1, b);
        int j1 = split[(size_t)e.code * 4 + j - 1];
        if (a.code == kLeafEmpty) return expand(b, j);
        if (b.code == kLeafEmpty) return expand(a, j);
        expand(a, j1);
        expand(b, j - j1);
    };
    out.emplace_back();
    for (size_t qi = 0; qi < queue.size(); ++qi) {
        const int x = queue[qi];
        slots.clear();
        Entry4 a, b;
        node2_child(n2[x], 0, a);
        node2_child(n2[x], 1, b);
        const int j = bestj[x];
        if (a.code == kLeafEmpty || b.code == kLeafEmpty) {
            expand(a.code == kLeafEmpty ? b : a, j);
        } else {
            int j1 = split[(size_t)x * 4 + j - 1];
            expand(a, j1);
            expand(b, j - j1);
        }
        int kids[4];
        const int cnt = (int)slots.size();
        for (int k = 0; k < 4; ++k) {
            if (k < cnt && slots[k].code >= 0) {
                kids[k] = (int)out.size();
                out.emplace_back();
                queue.push_back(slots[k].code);
            } else {
                kids[k] = k < cnt ? slots[k].code : kLeafEmpty;
            }
        }
        make_node4(out[qi], slots.data(), cnt, kids);
    }
    if (s->d_nodes4) cudaFree(s->d_nodes4);
    s->d_nodes4 = nullptr;
    rc = cuda_status(cudaMalloc(&s->d_nodes4, sizeof(Node4) * out.size()), "node4 alloc");
    if (!rc)
        rc = cuda_status(cudaMemcpy(s->d_nodes4, out.data(), sizeof(Node4) * out.size(), cudaMemcpyHostToDevice),
                         "node4 upload");
    if (!rc) s->num_nodes4 = (int32_t)out.size();
    return rc;
}

// The 4-wide tree per direction octant (SceneView::nodes8): record j of copy
// `oct` is node j with the lo / hi plane arrays of every axis that is
// negative in `oct` swapped, so the first array of an axis holds the planes a
// ray of that octant enters through.  Empty slots (lo = +3e38, hi = -3e38)
// stay empty in every copy.
__global__ void k_octant_nodes(const Node4 *__restrict__ n4, int m, Node4 *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)m * 8) return;
    const int oct = (int)(i / m), j = (int)(i % m);
    Node4 a = n4[j];
    Node4 o = a;
    if (oct & 1) { o.lox = a.hix; o.hix = a.lox; }
    if (oct & 2) { o.loy = a.hiy; o.hiy = a.loy; }
    if (oct & 4) { o.loz = a.hiz; o.hiz = a.loz; }
    out[i] = o;
}

static srt_status collapse4_tree(SrtScene *s);

srt_status octant_copies(const Node4 *n4, int32_t m, Node4 **out8, cudaStream_t st) {
    *out8 = nullptr;
    if (m == 0) return SRT_OK;
    if ((uint64_t)m * 8 >= (1ull << 32)) {  // packet kernels index the octant copies with 32 bits
        set_error("BVH too large for the octant node copies");
        return SRT_ERR_INVALID_ARG;
    }
    srt_status rc = cuda_status(cudaMalloc(out8, sizeof(Node4) * 8 * (size_t)m), "octant node alloc");
    if (rc) return rc;
    const int64_t total = (int64_t)m * 8;
    k_octant_nodes<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n4, m, *out8);
    rc = cuda_status(cudaGetLastError(), "k_octant_nodes");
    if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "octant nodes");
    return rc;
}

srt_status collapse4(SrtScene *s) {
    srt_status rc = collapse4_tree(s);
    if (rc) return rc;
    if (s->d_nodes8) cudaFree(s->d_nodes8);
    s->d_nodes8 = nullptr;
    return octant_copies(s->d_nodes4, s->num_nodes4, &s->d_nodes8, s->stream);
}

static srt_status collapse4_tree(SrtScene *s) {
#ifdef SRT_EXPERIMENTS
    // the cost-optimal collapse (measured 4% slower than greedy), experiments build only
    if (s->num_nodes > 0) {
        static const char *mode = getenv("SRT_COLLAPSE");
        if (mode && !strcmp(mode, "dp")) {
            float cv = 1.0f, ct = 0.25f, cj = 1.0f;
            if (const char *c = getenv("SRT_COLLAPSE_COSTS")) sscanf(c, "%f,%f,%f", &cv, &ct, &cj);
            cudaStreamSynchronize(s->stream);
            return collapse4_dp(s, cv, ct, cj);
        }
    }
#endif
    if (s->d_nodes4) cudaFree(s->d_nodes4);
    s->d_nodes4 = nullptr;
    s->num_nodes4 = 0;
    return collapse_tree(s->d_nodes, s->num_nodes, &s->d_nodes4, &s->num_nodes4, s->stream);
}

srt_status collapse_tree(const Node2 *n2, int32_t m2, Node4 **out4, int32_t *m4, cudaStream_t st) {
    *out4 = nullptr;
    *m4 = 0;
    if (m2 == 0) return SRT_OK;
    srt_status rc = SRT_OK;
    int2 *wa = nullptr, *wb = nullptr;
    int *counters = nullptr;  // [0] n4 count, [1] work_out count
    int h[2] = {1, 0};
    int n_in = 1;
    int2 root = make_int2(0, 0);
    // a 4-wide tree over m2 binary inner nodes has at most m2 nodes
    rc = cuda_status(cudaMalloc(out4, sizeof(Node4) * m2), "node4 alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&wa, sizeof(int2) * m2), "worklist");
    if (!rc) rc = cuda_status(cudaMalloc(&wb, sizeof(int2) * m2), "worklist");
    if (!rc) rc = cuda_status(cudaMalloc(&counters, sizeof(int) * 2), "counters");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(wa, &root, sizeof(int2), cudaMemcpyHostToDevice, st), "root");
    if (!rc) rc = cuda_status(cudaMemcpyAsync(counters, h, sizeof(h), cudaMemcpyHostToDevice, st), "counters");
    while (!rc && n_in > 0) {
        rc = cuda_status(cudaMemsetAsync(counters + 1, 0, sizeof(int), st), "counter reset");
        if (rc) break;
        k_collapse4<<<(n_in + 127) / 128, 128, 0, st>>>(n2, wa, n_in, wb, counters + 1, counters, *out4);
        rc = cuda_status(cudaGetLastError(), "k_collapse4");
        if (!rc) rc = cuda_status(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, st), "counters");
        if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "collapse");
        n_in = h[1];
        int2 *t = wa;
        wa = wb;
        wb = t;
    }
    if (!rc) *m4 = h[0];
    cudaFree(wa);
    cudaFree(wb);
    cudaFree(counters);
    return rc;
}

}  // namespace srt
