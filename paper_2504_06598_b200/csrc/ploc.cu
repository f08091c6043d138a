// ploc.cu -- PLOC BVH build (Meister & Bittner, "Parallel Locally-Ordered
// Clustering for Bounding Volume Hierarchy Construction", TVCG 2018): starting
// from the primitives in Morton order, every cluster finds its nearest
// neighbour (smallest union-box surface) within +-R positions; mutual nearest
// neighbours merge into a new node; the survivors are compacted in order and
// the process repeats until one cluster is left.  The tree is built bottom up
// in agglomerative (SAH-like) order, entirely on the GPU, and is markedly
// better than the Karras radix tree for traversal.
// Node2 records are written as the merges happen (both child boxes are known),
// so no refit pass is needed; the last merge becomes node 0, the root.
#include <cstdlib>

#include <cub/device/device_scan.cuh>

#include "srt_internal.h"

namespace srt {

constexpr int kPlocRadius = 16;  // neighbourhood half-width (SRT_PLOC_RADIUS overrides in the experiments build)

__device__ __forceinline__ float half_area(float4 lo, float4 hi) {
    float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
    return dx * dy + dy * dz + dz * dx;
}

__global__ void k_ploc_init(int64_t n, const uint32_t *__restrict__ slot_prim, const float *__restrict__ plo,
                            const float *__restrict__ phi, int *code, float4 *lo, float4 *hi) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int64_t p = slot_prim[j];
    code[j] = ~(int)j;
    lo[j] = make_float4(plo[p * 3], plo[p * 3 + 1], plo[p * 3 + 2], 0.f);
    hi[j] = make_float4(phi[p * 3], phi[p * 3 + 1], phi[p * 3 + 2], 0.f);
}

// cell (optional): clusters only pair within their cell of the split grid
// (split.cu); a cluster alone in its cell names itself and stays
__global__ void k_ploc_nn(int nc, int radius, const float4 *__restrict__ lo, const float4 *__restrict__ hi, int *nn,
                          const int *__restrict__ cell) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc) return;
    float4 l = lo[i], h = hi[i];
    float best = INFINITY;
    const int ci = cell ? cell[i] : 0;
    int bj = cell ? i : ((i ^ 1) < nc ? (i ^ 1) : i - 1);
    int j0 = max(0, i - radius), j1 = min(nc - 1, i + radius);
    for (int j = j0; j <= j1; ++j) {
        if (j == i) continue;
        if (cell && cell[j] != ci) continue;
        float4 l2 = lo[j], h2 = hi[j];
        float4 ul = make_float4(fminf(l.x, l2.x), fminf(l.y, l2.y), fminf(l.z, l2.z), 0.f);
        float4 uh = make_float4(fmaxf(h.x, h2.x), fmaxf(h.y, h2.y), fmaxf(h.z, h2.z), 0.f);
        float a = half_area(ul, uh);
        if (!(a <= 3.0e38f)) a = INFINITY;  // degenerate (unbounded) boxes: inf*0 must not give NaN orderings
        // ties go to the partner i ^ 1 (then the lower index): runs of equal
        // boxes pair up all at once and build a balanced subtree
        if (a < best || (a == best && j == (i ^ 1))) {
            best = a;
            bj = j;
        }
    }
    nn[i] = bj;
}

__global__ void k_ploc_merge(int nc, int64_t n, const int *__restrict__ nn, const int *__restrict__ code,
                             const float4 *__restrict__ lo, const float4 *__restrict__ hi, int *code2, float4 *lo2,
                             float4 *hi2, int *keep, int *counter, Node2 *nodes, int *parent_int, int *parent_leaf,
                             const int *__restrict__ cell, int *cell2) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc) return;
    int j = nn[i];
    float4 l = lo[i], h = hi[i];
    int c = code[i];
    if (cell) cell2[i] = cell[i];  // a merged cluster stays in its cell
    if (j != i && nn[j] == i) {
        if (i > j) {  // absorbed by its partner
            keep[i] = 0;
            return;
        }
        int node = (int)(n - 2) - atomicAdd(counter, 1);
        float4 l2 = lo[j], h2 = hi[j];
        int c2 = code[j];
        Node2 nd;
        nd.xy0 = make_float4(l.x, h.x, l.y, h.y);
        nd.xy1 = make_float4(l2.x, h2.x, l2.y, h2.y);
        nd.z01 = make_float4(l.z, h.z, l2.z, h2.z);
        nd.kids = make_int4(c, c2, 0, 0);
        nodes[node] = nd;
        if (c >= 0) parent_int[c] = node; else parent_leaf[~c] = node;
        if (c2 >= 0) parent_int[c2] = node; else parent_leaf[~c2] = node;
        code2[i] = node;
        lo2[i] = make_float4(fminf(l.x, l2.x), fminf(l.y, l2.y), fminf(l.z, l2.z), 0.f);
        hi2[i] = make_float4(fmaxf(h.x, h2.x), fmaxf(h.y, h2.y), fmaxf(h.z, h2.z), 0.f);
    } else {
        code2[i] = c;
        lo2[i] = l;
        hi2[i] = h;
    }
    keep[i] = 1;
}

__global__ void k_ploc_compact(int nc, const int *__restrict__ keep, const int *__restrict__ pos,
                               const int *__restrict__ code2, const float4 *__restrict__ lo2,
                               const float4 *__restrict__ hi2, int *code, float4 *lo, float4 *hi,
                               const int *__restrict__ cell2, int *cell) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc || !keep[i]) return;
    int o = pos[i];
    if (cell) cell[o] = cell2[i];
    code[o] = code2[i];
    lo[o] = lo2[i];
    hi[o] = hi2[i];
}

// Builds `nodes` (n - 1 Node2, root 0) from the Morton-sorted primitives (or
// leaf references).  With `cell` (per sorted position, sorted by cell first)
// clusters merge only within their cell until every cell is one cluster; the
// cells' roots are then clustered freely (the split tree's top, split.cu).
srt_status ploc_build(SrtScene *s, int64_t n, const uint32_t *slot_prim, const float *plo, const float *phi,
                      int *parent_int, int *parent_leaf, cudaStream_t st, Node2 *nodes, const int *cell) {
    (void)s;
    srt_status rc = SRT_OK;
    int *code = nullptr, *code2 = nullptr, *nn = nullptr, *keep = nullptr, *pos = nullptr, *counter = nullptr;
    float4 *lo = nullptr, *hi = nullptr, *lo2 = nullptr, *hi2 = nullptr;
    int *ccell = nullptr, *ccell2 = nullptr;
    bool restricted = cell != nullptr;
    void *temp = nullptr;
    size_t temp_bytes = 0;
    int nc = (int)n;
    const int B = 256;
#ifdef SRT_EXPERIMENTS
    const char *env = getenv("SRT_PLOC_RADIUS");  // radius sweeps (tools/tree_probe.py), experiments build only
    const int radius = env ? max(1, atoi(env)) : kPlocRadius;
#else
    const int radius = kPlocRadius;
#endif
    rc = cuda_status(cudaMalloc(&code, sizeof(int) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&code2, sizeof(int) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&nn, sizeof(int) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&keep, sizeof(int) * (n + 1)), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&pos, sizeof(int) * (n + 1)), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&counter, sizeof(int)), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&lo, sizeof(float4) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&hi, sizeof(float4) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&lo2, sizeof(float4) * n), "ploc alloc");
    if (!rc) rc = cuda_status(cudaMalloc(&hi2, sizeof(float4) * n), "ploc alloc");
    if (!rc && restricted) rc = cuda_status(cudaMalloc(&ccell, sizeof(int) * n), "ploc alloc");
    if (!rc && restricted) rc = cuda_status(cudaMalloc(&ccell2, sizeof(int) * n), "ploc alloc");
    if (!rc && restricted)
        rc = cuda_status(cudaMemcpyAsync(ccell, cell, sizeof(int) * n, cudaMemcpyDeviceToDevice, st), "ploc cells");
    if (!rc) rc = cuda_status(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, keep, pos, (int)(n + 1), st), "scan size");
    if (!rc) rc = cuda_status(cudaMalloc(&temp, temp_bytes ? temp_bytes : 1), "scan temp");
    if (!rc) rc = cuda_status(cudaMemsetAsync(counter, 0, sizeof(int), st), "ploc counter");
    if (!rc) {
        k_ploc_init<<<(unsigned)((n + B - 1) / B), B, 0, st>>>(n, slot_prim, plo, phi, code, lo, hi);
        rc = cuda_status(cudaGetLastError(), "k_ploc_init");
    }
    while (!rc && nc > 1) {
        unsigned g = (unsigned)((nc + B - 1) / B);
        int *cc = restricted ? ccell : nullptr, *cc2 = restricted ? ccell2 : nullptr;
        k_ploc_nn<<<g, B, 0, st>>>(nc, radius, lo, hi, nn, cc);
        k_ploc_merge<<<g, B, 0, st>>>(nc, n, nn, code, lo, hi, code2, lo2, hi2, keep, counter, nodes,
                                     parent_int, parent_leaf, cc, cc2);
        rc = cuda_status(cudaMemsetAsync(keep + nc, 0, sizeof(int), st), "ploc keep tail");
        if (!rc) rc = cuda_status(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, keep, pos, nc + 1, st), "ploc scan");
        if (!rc) {
            k_ploc_compact<<<g, B, 0, st>>>(nc, keep, pos, code2, lo2, hi2, code, lo, hi, cc2, cc);
            rc = cuda_status(cudaGetLastError(), "ploc kernels");
        }
        int next = 0;
        if (!rc) rc = cuda_status(cudaMemcpyAsync(&next, pos + nc, sizeof(int), cudaMemcpyDeviceToHost, st), "ploc count");
        if (!rc) rc = cuda_status(cudaStreamSynchronize(st), "ploc iteration");
        if (!rc && next >= nc) {
            if (restricted) {
                restricted = false;  // every cell is one cluster: cluster the cells' roots
            } else {
                set_error("PLOC made no progress");
                rc = SRT_ERR_CUDA;
            }
        }
        nc = next;
    }
    cudaFree(code);
    cudaFree(code2);
    cudaFree(nn);
    cudaFree(keep);
    cudaFree(pos);
    cudaFree(counter);
    cudaFree(lo);
    cudaFree(hi);
    cudaFree(lo2);
    cudaFree(hi2);
    cudaFree(ccell);
    cudaFree(ccell2);
    cudaFree(temp);
    return rc;
}

}  // namespace srt
