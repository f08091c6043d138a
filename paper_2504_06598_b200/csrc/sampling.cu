// sampling.cu -- the reference's two batch sampling utilities on the GPU,
// so the kernels shim exports every public entry point of
// splatray/kernels.py (its callers, e.g. validate.py:146-160, then run
// unchanged against libsrt):
//   hash_position_batch  kernels.py:119-122  -> srt_hash_positions
//   pixel_jitter_batch   kernels.py:125-135  -> srt_pixel_jitter
// The trig hash is the fp64 restatement of srt_trig64.cuh (device sin: the
// value agrees with glibc's to ~1e-5 absolute after the 43758.5453 scaling);
// the jitter is integer exact.
#include <algorithm>

#include "srt_internal.h"
#include "srt_trig64.cuh"

namespace srt {

__global__ void k_hash_positions(const double *__restrict__ pts, int64_t n, int64_t slot, double *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = t64::hash_position(pts[i * 3], pts[i * 3 + 1], pts[i * 3 + 2], (int)slot);
}

__global__ void k_pixel_jitter(uint32_t px, uint32_t py, const int64_t *__restrict__ frames, int64_t n, uint32_t seed,
                               double *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double jx, jy;
    pixel_jitter(px, py, (uint32_t)frames[i], seed, jx, jy);
    out[i * 2] = jx;
    out[i * 2 + 1] = jy;
}

// Host buffers in, host buffers out, on `device` (synchronous).
template <class Launch>
static srt_status run_small(int32_t device, size_t in_bytes, const void *in, size_t out_bytes, void *out, Launch launch) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        set_error("CUDA device not available");
        return SRT_ERR_CUDA;
    }
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    srt_status rc = cuda_status(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream create");
    if (rc) return rc;
    char *d = nullptr;
    const size_t off = (in_bytes + 255) & ~(size_t)255;
    rc = cuda_status(cudaMallocAsync((void **)&d, off + out_bytes, st), "alloc");
    if (!rc && in_bytes) rc = cuda_status(cudaMemcpyAsync(d, in, in_bytes, cudaMemcpyHostToDevice, st), "upload");
    if (!rc) rc = launch(d, d + off, st);
    if (!rc) rc = cuda_status(cudaMemcpyAsync(out, d + off, out_bytes, cudaMemcpyDeviceToHost, st), "download");
    if (d) cudaFreeAsync(d, st);
    srt_status rs = cuda_status(cudaStreamSynchronize(st), "sync");
    cudaStreamDestroy(st);
    return rc ? rc : rs;
}

}  // namespace srt

using namespace srt;

extern "C" {

srt_status srt_hash_positions(const double *points, int64_t n, int64_t slot, double *out, int32_t device) {
    if (n < 0 || (n > 0 && (!points || !out))) {
        set_error("invalid hash arguments");
        return SRT_ERR_INVALID_ARG;
    }
    if (n == 0) return SRT_OK;
    return run_small(device, sizeof(double) * 3 * n, points, sizeof(double) * n, out,
                     [&](char *din, char *dout, cudaStream_t st) {
                         k_hash_positions<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const double *)din, n, slot,
                                                                                         (double *)dout);
                         return cuda_status(cudaGetLastError(), "k_hash_positions");
                     });
}

srt_status srt_pixel_jitter(int64_t px, int64_t py, const int64_t *frames, int64_t n, uint32_t seed, double *out,
                            int32_t device) {
    if (n < 0 || (n > 0 && (!frames || !out))) {
        set_error("invalid jitter arguments");
        return SRT_ERR_INVALID_ARG;
    }
    if (n == 0) return SRT_OK;
    return run_small(device, sizeof(int64_t) * n, frames, sizeof(double) * 2 * n, out,
                     [&](char *din, char *dout, cudaStream_t st) {
                         k_pixel_jitter<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
                             (uint32_t)px, (uint32_t)py, (const int64_t *)din, n, seed, (double *)dout);
                         return cuda_status(cudaGetLastError(), "k_pixel_jitter");
                     });
}

}  // extern "C"
