// PCIe write rate of SM stores into mapped page-locked host memory for the
// f64 AccumBuffer of a 1920x1080 frame (rgb (H,W,3) + opacity (H,W) f64):
// packet rows of 8 pixels (8x4 packets: 192 B rgb + 64 B opacity per row),
// of 16 pixels (16x2 packets: 384 B + 128 B, whole 128 B lines), and a
// linear copy.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pcie tools/probes/pcie_store_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 1920, H = 1080;

// one warp per packet of PW x PH pixels; lanes store double2 words of each row
template <int PW, int PH>
__global__ void k_packets(double *rgb, double *op) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int pw = W / PW, ph = H / PH;
    for (int p = warp; p < pw * ph; p += (gridDim.x * blockDim.x) >> 5) {
        const int px = (p % pw) * PW, py = (p / pw) * PH;
        constexpr int RGB2 = PW * 3 / 2, OP2 = PW / 2;  // double2 words per row
        for (int g = lane; g < PH * RGB2; g += 32) {
            const int r = g / RGB2, q = g - r * RGB2;
            reinterpret_cast<double2 *>(rgb + ((size_t)(py + r) * W + px) * 3)[q] = make_double2(r, q);
        }
        for (int g = lane; g < PH * OP2; g += 32) {
            const int r = g / OP2, q = g - r * OP2;
            reinterpret_cast<double2 *>(op + (size_t)(py + r) * W + px)[q] = make_double2(r, q);
        }
    }
}

__global__ void k_linear(double2 *dst, size_t n2) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = make_double2(1.0, 2.0);
}

int main() {
    const size_t bytes = (size_t)W * H * 4 * sizeof(double);
    double *h = nullptr, *d = nullptr;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostGetDevicePointer(&d, h, 0);
    double *rgb = d, *op = d + (size_t)W * H * 3;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 8, block = 128;
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 3; ++v) {
            float best = 1e9f;
            for (int it = 0; it < 10; ++it) {
                cudaEventRecord(a);
                if (v == 0) k_packets<8, 4><<<grid, block>>>(rgb, op);
                if (v == 1) k_packets<16, 2><<<grid, block>>>(rgb, op);
                if (v == 2) k_linear<<<grid, block>>>(reinterpret_cast<double2 *>(d), bytes / 16);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const char *name[] = {"8x4 packets (192 B + 64 B rows)", "16x2 packets (384 B + 128 B rows)", "linear"};
            printf("%-36s %.3f ms  %.1f GB/s\n", name[v], best, bytes / best / 1e6);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
