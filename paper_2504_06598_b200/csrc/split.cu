// split.cu -- the packet walk's spatially split tree.
//
// The PLOC tree over whole primitive boxes has overlapping top-level children:
// every Gaussian box that straddles a top split widens both halves, so a band
// around each top split plane belongs to both subtrees.  Camera rays that run
// inside such a band (the image's central column and row for the front
// camera, whose view axis lies in the scene's central planes) walk both halves
// for their whole length; they are the frame's slowest packets (DESIGN.md §5,
// "where a frame's time goes") and bound a multi-GPU tile shard (§6).
//
// This builder removes the overlap at the top of the tree:
//   1. a uniform grid of C x C x C cells over the primitives' centre bounds
//      (interior planes only; the outer cells are open);
//   2. each primitive gets one leaf REFERENCE per cell its box overlaps, the
//      box clipped to the cell and widened by eps past each clipped plane
//      (the references' boxes overlap by 2 eps, so the fp32 slab test of a
//      point on a plane cannot miss both);
//   3. references sorted by (cell, 16-bit/axis Morton code of the clipped box
//      centre), PLOC clustering restricted to each cell until every cell is
//      one cluster, then the cells' roots clustered freely (ploc.cu);
//   4. the greedy 4-wide collapse and the octant copies, plus the geometry
//      records in reference order (a duplicated primitive's record repeats).
//
// Correctness: a candidate the walk reports lies inside the primitive's
// cutoff ellipsoid (kernels.py:187; mean depth: the peak, center depth: the
// centre projection, both tested against the ellipsoid), hence inside the
// primitive's box, hence inside at least one clipped reference box -- so the
// far-bound culling never drops it.  A duplicated reference evaluates the same
// primitive with the same (ray, slot, primitive) draw and the same depth: the
// 64-bit (t, id) atomicMin of each slot is idempotent, so the closest accepted
// hit per slot is exactly the unsplit tree's (the per-lane walks' slot update
// is idempotent too: strict t, ties to the smaller id).  Only the closest-hit
// walks (k_trace_packet, k_trace, k_trace_coop and the trig64 bridge walks)
// use this tree.  The compositing walks (transmittance, exact, biased) keep
// the unsplit tree: they walk every candidate along the ray, so duplicated
// references only add work -- measured with an ownership rule that counts
// each candidate at one reference (the cell of its point): 1080p exact frame
// 52 -> 65 ms, transmittance of 1M random rays 25.8 -> 22.1 Mrays/s.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "srt_internal.h"

namespace srt {

constexpr int64_t kSplitMinPrims = 1 << 14;  // smaller scenes: the packet walk uses the unsplit tree

// cells per axis (0: no split tree).  Measured on density-preserving clouds
// (device-timed frames, tools/exp_split_sizes.sh, profiles/r02g_split/):
//   100k, 512^2:        none 0.395 ms, C=2 0.375, C=3 0.375, C=4 0.454
//   1M, 1080p (3 seeds): none 1.654, C=2 1.572, C=4 1.503, C=6 1.480, C=7 1.454, C=8 1.565
//   3M, 4K:             none 6.50, C=4 5.53, C=6 5.87, C=8 5.17, C=10 6.46
//   6M, 1080p:          none 2.10, C=6 1.85, C=8 1.75, C=10 2.03, C=12 2.12
// Finer grids duplicate more references (C=8 at 1M: 1.79 references per
// primitive) and their planes interact with the Morton order inside a cell,
// so the optimum is not monotone; the table keeps the measured best.
static int split_cells_for(int64_t n) {
#ifdef SRT_EXPERIMENTS
    if (const char *e = getenv("SRT_SPLIT_CELLS")) return atoi(e);
#endif
    if (n < kSplitMinPrims) return 0;
    if (n < (1 << 18)) return 2;
    if (n < 2000000) return 7;
    return 8;
}

struct Grid {
    float lo[3];    // plane k of axis a: lo[a] + step[a] * k, interior planes k = 1 .. c[a] - 1
    float step[3];
    float eps[3];   // overlap past a clipped plane
    int c[3];       // cells along the axis (1 when the axis has no extent)
    float mlo[3];   // Morton frame
    float minv[3];
};

__device__ __forceinline__ float plane(const Grid &g, int a, int k) { return __fmaf_rn(g.step[a], (float)k, g.lo[a]); }

// cells k0 .. k1 that [l, h] overlaps: k0 = #{interior planes <= l}, k1 = #{interior planes < h}
__device__ __forceinline__ void cell_range(const Grid &g, int a, float l, float h, int &k0, int &k1) {
    k0 = 0;
    k1 = 0;
    for (int k = 1; k < g.c[a]; ++k) {
        const float p = plane(g, a, k);
        k0 += p <= l;
        k1 += p < h;
    }
    if (k1 < k0) k1 = k0;
}

__global__ void k_ref_count(int64_t n, const float *__restrict__ plo, const float *__restrict__ phi, Grid g,
                            uint32_t *cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) {  // the scan's tail element
        cnt[n] = 0;
        return;
    }
    uint32_t c = 1;
    for (int a = 0; a < 3; ++a) {
        int k0, k1;
        cell_range(g, a, plo[i * 3 + a], phi[i * 3 + a], k0, k1);
        c *= (uint32_t)(k1 - k0 + 1);
    }
    cnt[i] = c;
}

__device__ __forceinline__ uint64_t spread16(uint64_t x) {  // 16 bits -> every third bit
    x &= 0xffffull;
    x = (x | x << 16) & 0x0000ff0000ffull;
    x = (x | x << 8) & 0x00f00f00f00full;
    x = (x | x << 4) & 0x0c30c30c30c3ull;
    x = (x | x << 2) & 0x249249249249ull;
    return x;
}

__global__ void k_ref_emit(int64_t n, const float *__restrict__ plo, const float *__restrict__ phi, Grid g,
                           const uint32_t *__restrict__ off, float *rlo, float *rhi, uint64_t *keys, uint32_t *vals,
                           uint32_t *rprim) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float l[3], h[3];
    int k0[3], k1[3];
    for (int a = 0; a < 3; ++a) {
        l[a] = plo[i * 3 + a];
        h[a] = phi[i * 3 + a];
        cell_range(g, a, l[a], h[a], k0[a], k1[a]);
    }
    uint32_t o = off[i];
    for (int iz = k0[2]; iz <= k1[2]; ++iz)
        for (int iy = k0[1]; iy <= k1[1]; ++iy)
            for (int ix = k0[0]; ix <= k1[0]; ++ix) {
                const int kk[3] = {ix, iy, iz};
                uint64_t code = 0;
                for (int a = 0; a < 3; ++a) {
                    const float bl = kk[a] == k0[a] ? l[a] : plane(g, a, kk[a]) - g.eps[a];
                    const float bh = kk[a] == k1[a] ? h[a] : plane(g, a, kk[a] + 1) + g.eps[a];
                    rlo[(size_t)o * 3 + a] = bl;
                    rhi[(size_t)o * 3 + a] = bh;
                    float u = (0.5f * bl + 0.5f * bh - g.mlo[a]) * g.minv[a];
                    u = fminf(fmaxf(u, 0.f), 1.f);  // (NaN -> 0)
                    const uint64_t q = (uint64_t)fminf(u * 65536.0f, 65535.0f);
                    code |= spread16(q) << (2 - a);
                }
                const uint64_t cell = (uint64_t)((iz * g.c[1] + iy) * g.c[0] + ix);
                keys[o] = (cell << 48) | code;
                vals[o] = o;
                rprim[o] = (uint32_t)i;
                ++o;
            }
}

__global__ void k_ref_slots(int64_t nr, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                            const uint32_t *__restrict__ rprim, int *cell, uint32_t *slot_prim) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nr) return;
    cell[j] = (int)(keys[j] >> 48);
    slot_prim[j] = rprim[vals[j]];
}

static float host_from_ordered(int i) {
    const int b = i >= 0 ? i : i ^ 0x7FFFFFFF;
    float f;
    memcpy(&f, &b, sizeof(f));
    return f;
}

void free_split(SrtScene *s) {
    cudaFree(s->d_geom_split);
    cudaFree(s->d_nodes8_split);
    cudaFree(s->d_nodes4_split);
    s->d_nodes4_split = nullptr;
    s->d_geom_split = nullptr;
    s->d_nodes8_split = nullptr;
    s->num_nodes4_split = 0;
    s->n_refs = 0;
    s->split_cells = 0;
}

srt_status split_build(SrtScene *s, const float *plo, const float *phi, const int *cbounds, cudaStream_t st) {
    free_split(s);
    const int64_t n = s->n;
    const int C = split_cells_for(n);
    if (C < 2 || n < 2) return SRT_OK;
    int cb[6];
    srt_status rc = cuda_status(cudaMemcpyAsync(cb, cbounds, sizeof(cb), cudaMemcpyDeviceToHost, st), "split bounds");
    if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "split bounds");
    if (rc) return rc;
    Grid g;
    for (int a = 0; a < 3; ++a) {
        const float lo = host_from_ordered(cb[a]), hi = host_from_ordered(cb[3 + a]);
        const float ext = hi - lo;
        const bool flat = !(ext > 0.f) || !std::isfinite(ext);
        g.c[a] = flat ? 1 : C;
        g.lo[a] = lo;
        g.step[a] = flat ? 0.f : ext / (float)C;
        g.eps[a] = flat ? 0.f : ext * 1e-5f;
        g.mlo[a] = lo;
        g.minv[a] = flat ? 0.f : 1.0f / ext;
    }
    if (g.c[0] == 1 && g.c[1] == 1 && g.c[2] == 1) return SRT_OK;  // all centres coincide: nothing to split
    uint32_t *cnt = nullptr, *off = nullptr, *vals = nullptr, *vals2 = nullptr, *rprim = nullptr, *slot_prim = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    float *rlo = nullptr, *rhi = nullptr;
    int *cell = nullptr, *parent_int = nullptr, *parent_leaf = nullptr;
    Node2 *nodes = nullptr;
    Node4 *n4 = nullptr;
    void *temp = nullptr;
    size_t temp_bytes = 0, tb2 = 0;
    uint32_t nr32 = 0;
    int64_t nr = 0;
    int32_t m4 = 0;
    const unsigned B = 256;
#define SRT_TRY(x)          \
    do {                    \
        rc = (x);           \
        if (rc) goto done;  \
    } while (0)
    SRT_TRY(cuda_status(cudaMalloc(&cnt, sizeof(uint32_t) * (n + 1)), "split counts"));
    SRT_TRY(cuda_status(cudaMalloc(&off, sizeof(uint32_t) * (n + 1)), "split offsets"));
    k_ref_count<<<(unsigned)((n + 1 + B - 1) / B), B, 0, st>>>(n, plo, phi, g, cnt);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_ref_count"));
    SRT_TRY(cuda_status(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, cnt, off, (int)(n + 1), st), "scan size"));
    SRT_TRY(cuda_status(cudaMalloc(&temp, temp_bytes ? temp_bytes : 1), "scan temp"));
    SRT_TRY(cuda_status(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, cnt, off, (int)(n + 1), st), "split scan"));
    SRT_TRY(cuda_status(cudaMemcpyAsync(&nr32, off + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st), "ref count"));
    SRT_TRY(cuda_status(cudaStreamSynchronize(st), "ref count"));
    cudaFree(temp);
    temp = nullptr;
    nr = nr32;
    if (nr < n || nr > 4 * n + (1 << 20) || nr > (int64_t)INT32_MAX / 2) {
        // (fully degenerate boxes land in every cell: keep the unsplit tree)
        rc = SRT_OK;
        goto done;
    }
    SRT_TRY(cuda_status(cudaMalloc(&rlo, sizeof(float) * 3 * nr), "ref boxes"));
    SRT_TRY(cuda_status(cudaMalloc(&rhi, sizeof(float) * 3 * nr), "ref boxes"));
    SRT_TRY(cuda_status(cudaMalloc(&keys, sizeof(uint64_t) * nr), "ref keys"));
    SRT_TRY(cuda_status(cudaMalloc(&keys2, sizeof(uint64_t) * nr), "ref keys"));
    SRT_TRY(cuda_status(cudaMalloc(&vals, sizeof(uint32_t) * nr), "ref vals"));
    SRT_TRY(cuda_status(cudaMalloc(&vals2, sizeof(uint32_t) * nr), "ref vals"));
    SRT_TRY(cuda_status(cudaMalloc(&rprim, sizeof(uint32_t) * nr), "ref prims"));
    SRT_TRY(cuda_status(cudaMalloc(&slot_prim, sizeof(uint32_t) * nr), "ref slots"));
    SRT_TRY(cuda_status(cudaMalloc(&cell, sizeof(int) * nr), "ref cells"));
    k_ref_emit<<<(unsigned)((n + B - 1) / B), B, 0, st>>>(n, plo, phi, g, off, rlo, rhi, keys, vals, rprim);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_ref_emit"));
    SRT_TRY(cuda_status(cub::DeviceRadixSort::SortPairs(nullptr, tb2, keys, keys2, vals, vals2, (int)nr, 0, 58, st),
                        "ref sort sizing"));
    SRT_TRY(cuda_status(cudaMalloc(&temp, tb2 ? tb2 : 1), "ref sort temp"));
    SRT_TRY(cuda_status(cub::DeviceRadixSort::SortPairs(temp, tb2, keys, keys2, vals, vals2, (int)nr, 0, 58, st),
                        "ref sort"));
    k_ref_slots<<<(unsigned)((nr + B - 1) / B), B, 0, st>>>(nr, keys2, vals2, rprim, cell, slot_prim);
    SRT_TRY(cuda_status(cudaGetLastError(), "k_ref_slots"));
    SRT_TRY(cuda_status(cudaMalloc(&nodes, sizeof(Node2) * (nr - 1)), "split nodes"));
    SRT_TRY(cuda_status(cudaMalloc(&parent_int, sizeof(int) * (nr - 1)), "split parents"));
    SRT_TRY(cuda_status(cudaMalloc(&parent_leaf, sizeof(int) * nr), "split parents"));
    SRT_TRY(ploc_build(s, nr, vals2, rlo, rhi, parent_int, parent_leaf, st, nodes, cell));
    SRT_TRY(collapse_tree(nodes, (int32_t)(nr - 1), &n4, &m4, st));
    SRT_TRY(octant_copies(n4, m4, &s->d_nodes8_split, st));
    s->d_nodes4_split = n4;
    n4 = nullptr;
    SRT_TRY(cuda_status(cudaMalloc(&s->d_geom_split, sizeof(Geom) * nr), "split geom"));
    SRT_TRY(launch_geom(nr, slot_prim, s, s->d_geom_split, st));
    SRT_TRY(cuda_status(cudaStreamSynchronize(st), "split build"));
    s->num_nodes4_split = m4;
    s->n_refs = nr;
    s->split_cells = C;
done:
#undef SRT_TRY
    if (rc) free_split(s);
    cudaFree(cnt);
    cudaFree(off);
    cudaFree(vals);
    cudaFree(vals2);
    cudaFree(rprim);
    cudaFree(slot_prim);
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(rlo);
    cudaFree(rhi);
    cudaFree(cell);
    cudaFree(parent_int);
    cudaFree(parent_leaf);
    cudaFree(nodes);
    cudaFree(n4);
    cudaFree(temp);
    return rc;
}

}  // namespace srt
