// pack.cu -- GPU packing of raw splats: the inverse
// covariance A = Sigma^-1 = R diag(1/s^2) R^T of every primitive, in fp64,
// straight from its unit quaternion (w, x, y, z) and scales.  This replaces
// SplatAsset.packed (assets.py:145-171: a per-primitive Python loop for R,
// then numpy inversion of R S^2 R^T), which takes ~11 s at 1M primitives in
// the reference.  The closed form differs from numpy's inverse only in the
// last bits; the trig64 bridge mode needs the reference's exact bits and
// uses host packing instead.
#include "srt_internal.h"

namespace srt {

__global__ void k_pack_splats(int64_t n, const double *__restrict__ q, const double *__restrict__ scales,
                              double *cov6) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double w = q[i * 4], x = q[i * 4 + 1], y = q[i * 4 + 2], z = q[i * 4 + 3];
    // rotation matrix of a unit quaternion (gaussians.py:166-176)
    double R[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                      {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                      {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
    double inv2[3];
    for (int k = 0; k < 3; ++k) {
        double s = scales[i * 3 + k];
        inv2[k] = 1.0 / (s * s);
    }
    double a[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) a[r][c] = R[r][0] * R[c][0] * inv2[0] + R[r][1] * R[c][1] * inv2[1] + R[r][2] * R[c][2] * inv2[2];
    double *o = cov6 + i * 6;
    o[0] = a[0][0];
    o[1] = a[0][1];
    o[2] = a[0][2];
    o[3] = a[1][1];
    o[4] = a[1][2];
    o[5] = a[2][2];
}

srt_status launch_pack_splats(int64_t n, const double *d_q, const double *d_scales, double *d_cov6, cudaStream_t st) {
    if (n == 0) return SRT_OK;
    k_pack_splats<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d_q, d_scales, d_cov6);
    return cuda_status(cudaGetLastError(), "k_pack_splats launch");
}

}  // namespace srt
