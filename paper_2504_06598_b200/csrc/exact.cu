// exact.cu -- exact sorted compositing: the RNG-free
// converged reference of the estimator, `render(..., reference_mode=True)`.
//
// The reference brute-forces every primitive per ray (kernels.py:441-475).
// Here each ray walks the BVH WITHOUT clipping, collecting every valid
// candidate (the same set: a valid candidate lies inside its ellipsoid, hence
// inside its conservative box), sorts them by (t, prim id) -- the stable
// order of np.argsort(kind="mergesort") over ids appended in increasing order
// -- and composites front to back in fp64: L = sum T_i a_i c_i + T bg.
#include <cfloat>

#include "srt_internal.h"

namespace srt {

constexpr int kExactCap = 512;  // candidates per ray (overflow -> SRT_ERR_STACK_OVERFLOW)

template <int MODE>
__device__ void exact_ray(const SceneView &s, const RayState &r, float s2, const float *bg, double out[4],
                          int *overflow) {
    float ct[kExactCap];
    float ca[kExactCap];
    int cid[kExactCap];
    int m = 0;
    if (s.num_nodes4 > 0) {
        int stk[kStackSize];
        int sp = 0, node = 0;
        while (node >= 0) {
            const float4 *np = reinterpret_cast<const float4 *>(s.nodes4 + node);
            float4 lox = __ldg(np), hix = __ldg(np + 1), loy = __ldg(np + 2), hiy = __ldg(np + 3),
                   loz = __ldg(np + 4), hiz = __ldg(np + 5);
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
                float tf = fminf(fminf(fmaxf(xa, xb), fmaxf(ya, yb)), fminf(fmaxf(za, zb), r.t_max0));
                if (!(tn <= tf)) continue;
                if (kid[k] >= 0) {
                    if (sp >= kStackSize) {
                        atomicExch(overflow, 1);
                        break;
                    }
                    stk[sp++] = kid[k];
                    continue;
                }
                const float4 *g = reinterpret_cast<const float4 *>(s.geom + ~kid[k]);
                float4 gm = __ldg(g), ga = __ldg(g + 1), gb = __ldg(g + 2);
                Cand c = candidate<MODE>(r, gm, ga, gb, s2);
                if (!c.valid) continue;
                if (m >= kExactCap) {
                    atomicExch(overflow, 1);
                    continue;
                }
                ct[m] = c.t;
                ca[m] = c.alpha;
                cid[m] = __float_as_int(gb.z);
                ++m;
            }
            if (sp > 0) node = stk[--sp];
        }
    }
    // insertion sort by (t, prim id)
    for (int i = 1; i < m; ++i) {
        float t = ct[i], a = ca[i];
        int id = cid[i];
        int j = i - 1;
        while (j >= 0 && (ct[j] > t || (ct[j] == t && cid[j] > id))) {
            ct[j + 1] = ct[j];
            ca[j + 1] = ca[j];
            cid[j + 1] = cid[j];
            --j;
        }
        ct[j + 1] = t;
        ca[j + 1] = a;
        cid[j + 1] = id;
    }
    double rr = 0.0, gg = 0.0, bb = 0.0, trans = 1.0;
    for (int i = 0; i < m; ++i) {
        float3 col = sh_color(s.sh, s.sh_k, s.sh_deg, cid[i], r.fdx, r.fdy, r.fdz);
        double w = trans * (double)ca[i];
        rr += w * col.x;
        gg += w * col.y;
        bb += w * col.z;
        trans *= 1.0 - (double)ca[i];
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

// render_exact (kernels.py:677-723): per pixel, the mean over `passes`
// jittered rays of the exact composite.  Row-major fp64 outputs.
template <int MODE>
__global__ void __launch_bounds__(128) k_exact_frame(SceneView s, CamD cam, RenderArgs a, double *rgb, double *op,
                                                     int *overflow) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)a.width * a.height) return;
    int px = (int)(i % a.width), py = (int)(i / a.width);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int f = 0; f < a.passes; ++f) {
        double dx, dy, dz;
        camera_ray(cam, (uint32_t)px, (uint32_t)py, (uint32_t)(a.pass0 + f), a.seed, a.width, a.height, dx, dy, dz);
        RayState r;
        init_ray(r, cam.e[0], cam.e[1], cam.e[2], dx, dy, dz, 0.0, DBL_MAX);
        double o[4];
        exact_ray<MODE>(s, r, a.s2, a.bg, o, overflow);
        for (int c = 0; c < 4; ++c) acc[c] += o[c];
    }
    double inv = 1.0 / (double)a.passes;
    rgb[i * 3] = acc[0] * inv;
    rgb[i * 3 + 1] = acc[1] * inv;
    rgb[i * 3 + 2] = acc[2] * inv;
    op[i] = acc[3] * inv;
}

srt_status launch_exact_rays(const SrtScene *s, const double *d_rays, int64_t R, double t_min, double t_max, int mode,
                             double s2, const double *bg, double *d_rgb, double *d_op, cudaStream_t st) {
    unsigned blocks = (unsigned)((R + 127) / 128);
    if (blocks == 0) return SRT_OK;
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
    int64_t n = (int64_t)a.width * a.height;
    unsigned blocks = (unsigned)((n + 127) / 128);
    if (blocks == 0) return SRT_OK;
    if (a.mode == 0)
        k_exact_frame<0><<<blocks, 128, 0, st>>>(s->view(), cam, a, d_rgb, d_op, s->d_flag);
    else
        k_exact_frame<1><<<blocks, 128, 0, st>>>(s->view(), cam, a, d_rgb, d_op, s->d_flag);
    return cuda_status(cudaGetLastError(), "k_exact_frame launch");
}

}  // namespace srt
