// shade.cu -- fused SH-eval + accumulate (kernels.py:657-673), the resolve to
// the reference's fp64 (H,W,3)/(H,W) outputs, and the multi-GPU tile unpack.
#include "srt_internal.h"

namespace srt {

__device__ __forceinline__ void tile_pixel_s(const RenderArgs &a, int64_t lt, int tid, int &px, int &py) {
    int64_t gt = lt * a.shard_count + a.shard_index;
    int tx = (int)(gt % a.tiles_x), ty = (int)(gt / a.tiles_x);
    int w = tid >> 5, lane = tid & 31;
    px = tx * 16 + (w & 1) * 8 + (lane & 7);
    py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
}

// One thread per pixel: SH colour of every slot's hit on the pass's ray
// direction (kernels.py:660, view dir = ray dir), background for misses,
// accumulated into a float4 running sum (r, g, b, hits).  On the last pass
// the mean (x 1/(passes*nslots), kernels.py:669-673) is written to d_out:
// row-major (H*W) float4 when unsharded, tile-compact when sharded.
__global__ void __launch_bounds__(256) k_shade_pass(SceneView s, CamD cam, RenderArgs a, int pass,
                                                    const int32_t *__restrict__ hits, float4 *accum, int first,
                                                    int last, float4 *out) {
    int64_t lt = blockIdx.x;
    int px, py;
    tile_pixel_s(a, lt, threadIdx.x, px, py);
    if (px >= a.width || py >= a.height) return;
    int64_t cidx = lt * 256 + threadIdx.x;
    const int32_t *h = hits + cidx * a.nslots;
    float r = 0.f, g = 0.f, b = 0.f, o = 0.f;
    bool need_dir = false;
    for (int k = 0; k < a.nslots; ++k) need_dir |= __ldg(h + k) >= 0;
    float fx = 0.f, fy = 0.f, fz = 0.f;
    if (need_dir) {
        double dx, dy, dz;
        camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)pass, a.seed, a.width, a.height, dx, dy, dz);
        fx = (float)dx;
        fy = (float)dy;
        fz = (float)dz;
    }
    for (int k = 0; k < a.nslots; ++k) {
        int pid = __ldg(h + k);
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
    float4 acc = first ? make_float4(0.f, 0.f, 0.f, 0.f) : accum[cidx];
    acc.x += r;
    acc.y += g;
    acc.z += b;
    acc.w += o;
    if (last) {
        float inv = 1.0f / ((float)a.passes * (float)a.nslots);
        float4 res = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        int64_t oidx = a.shard_count > 1 ? cidx : (int64_t)py * a.width + px;
        out[oidx] = res;
    } else {
        accum[cidx] = acc;
    }
}

srt_status launch_shade_pass(const SrtScene *s, const CamD &cam, const RenderArgs &a, int pass,
                             const int32_t *d_hits, float4 *d_accum, bool first, bool last, float4 *d_out,
                             cudaStream_t st) {
    if (a.local_tiles <= 0) return SRT_OK;
    k_shade_pass<<<(unsigned)a.local_tiles, 256, 0, st>>>(s->view(), cam, a, pass, d_hits, d_accum, first ? 1 : 0,
                                                         last ? 1 : 0, d_out);
    return cuda_status(cudaGetLastError(), "k_shade_pass launch");
}

// float4 rgba means -> the reference's AccumBuffer arrays, fp64
__global__ void k_resolve_f64(int64_t npix, const float4 *__restrict__ in, double *rgb, double *op) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    float4 v = in[i];
    rgb[i * 3 + 0] = v.x;
    rgb[i * 3 + 1] = v.y;
    rgb[i * 3 + 2] = v.z;
    op[i] = v.w;
}

srt_status launch_resolve_f64(const RenderArgs &a, const float4 *d_out, double *d_rgb, double *d_op, cudaStream_t st) {
    int64_t npix = (int64_t)a.width * a.height;
    if (npix == 0) return SRT_OK;
    k_resolve_f64<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(npix, d_out, d_rgb, d_op);
    return cuda_status(cudaGetLastError(), "k_resolve_f64 launch");
}

// Fixed-point frame sums (unit * 4 u64, 2^-32 units; opacity in 2^32 units)
// -> per-pixel means: float4 d_out (row-major unsharded, tile-compact when
// sharded) or, when d_rgb is set, the f64 frame (H,W,3)+(H,W) straight into
// its final (possibly mapped host) buffers.  A warp resolves one 8x4 pixel
// block; the f64 values are staged in shared memory and written as the
// block's 4 rows of contiguous 16-byte words (192 B rgb + 64 B opacity per
// row), as the fused walk stores its packets: over PCIe into mapped memory,
// scattered 8-byte stores at a 24-byte stride made the 1080p 16-spp
// render() resolve ~7 ms, full rows ~1.3 ms.
__global__ void __launch_bounds__(256) k_resolve_fixed(RenderArgs a, int64_t unit,
                                                       const unsigned long long *__restrict__ acc, double inv,
                                                       float4 *out, double *rgb, double *op) {
    __shared__ __align__(16) double srgb[8][96];
    __shared__ __align__(16) double sop[8][32];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int px = 0, py = 0;
    bool valid = i < unit;
    if (valid) {
        tile_pixel_s(a, i >> 8, (int)(i & 255), px, py);
        valid = px < a.width && py < a.height;
    }
    double r = 0.0, g = 0.0, b = 0.0, o = 0.0;
    if (valid) {
        const unsigned long long *q = acc + i * 4;
        const double k = inv * 2.3283064365386963e-10;  // 2^-32
        r = (double)q[0] * k;
        g = (double)q[1] * k;
        b = (double)q[2] * k;
        o = (double)(q[3] >> 32) * inv;
    }
    if (!rgb) {
        if (valid) {
            int64_t oidx = a.shard_count > 1 ? i : (int64_t)py * a.width + px;
            out[oidx] = make_float4((float)r, (float)g, (float)b, (float)o);
        }
        return;
    }
    const unsigned FULL = 0xffffffffu;
    const int64_t W = a.width;
    const int64_t pix = (int64_t)py * W + px;
    const int64_t pix0 = __shfl_sync(FULL, pix, 0);
    const bool block = __all_sync(FULL, valid && pix == pix0 + (int64_t)(lane >> 3) * W + (lane & 7));
    const bool aligned = ((((uintptr_t)rgb | (uintptr_t)op) & 15u) == 0) && !((pix0 | W) & 1);
    if (block && aligned) {
        srgb[wid][lane * 3] = r;
        srgb[wid][lane * 3 + 1] = g;
        srgb[wid][lane * 3 + 2] = b;
        sop[wid][lane] = o;
        __syncwarp();
        for (int gq = lane; gq < 48; gq += 32) {  // 4 rows x 12 double2 of rgb
            const int rr = gq / 12, q = gq - rr * 12;
            *reinterpret_cast<double2 *>(rgb + (pix0 + rr * W) * 3 + 2 * q) =
                *reinterpret_cast<const double2 *>(&srgb[wid][rr * 24 + 2 * q]);
        }
        if (lane < 16) {  // 4 rows x 4 double2 of opacity
            const int rr = lane >> 2, q = lane & 3;
            *reinterpret_cast<double2 *>(op + pix0 + rr * W + 2 * q) =
                *reinterpret_cast<const double2 *>(&sop[wid][rr * 8 + 2 * q]);
        }
    } else if (valid) {
        rgb[pix * 3 + 0] = r;
        rgb[pix * 3 + 1] = g;
        rgb[pix * 3 + 2] = b;
        op[pix] = o;
    }
}

srt_status launch_resolve_fixed(const RenderArgs &a, const unsigned long long *d_acc, int npass, float4 *d_out,
                                double *d_rgb, double *d_op, cudaStream_t st) {
    int64_t unit = a.local_tiles * 256;
    if (unit == 0) return SRT_OK;
    double inv = 1.0 / ((double)npass * (double)a.nslots);
    k_resolve_fixed<<<(unsigned)((unit + 255) / 256), 256, 0, st>>>(a, unit, d_acc, inv, d_out, d_rgb, d_op);
    return cuda_status(cudaGetLastError(), "k_resolve_fixed launch");
}

// gathered: [shard][max_tiles*256] float4, tile-compact per shard.
__global__ void k_unpack_tiles(const float4 *__restrict__ gathered, int width, int height, int shard_count,
                               int64_t max_tiles, int tiles_x, int64_t total_tiles, float4 *frame) {
    int64_t gt = blockIdx.x;
    if (gt >= total_tiles) return;
    int shard = (int)(gt % shard_count);
    int64_t lt = gt / shard_count;
    int tx = (int)(gt % tiles_x), ty = (int)(gt / tiles_x);
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int px = tx * 16 + (w & 1) * 8 + (lane & 7);
    int py = ty * 16 + (w >> 1) * 4 + (lane >> 3);
    if (px >= width || py >= height) return;
    frame[(int64_t)py * width + px] = gathered[((int64_t)shard * max_tiles + lt) * 256 + threadIdx.x];
}

srt_status launch_unpack(const float4 *d_gathered, int width, int height, int shard_count, int64_t max_tiles,
                         float4 *d_frame, cudaStream_t st) {
    int tiles_x = (width + 15) / 16, tiles_y = (height + 15) / 16;
    int64_t total = (int64_t)tiles_x * tiles_y;
    if (total == 0) return SRT_OK;
    k_unpack_tiles<<<(unsigned)total, 256, 0, st>>>(d_gathered, width, height, shard_count, max_tiles, tiles_x, total,
                                                     d_frame);
    return cuda_status(cudaGetLastError(), "k_unpack_tiles launch");
}

}  // namespace srt
