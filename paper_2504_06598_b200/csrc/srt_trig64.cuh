// srt_trig64.cuh -- fp64 restatement of the reference's candidate and trig
// hash (kernels.py:47-60, 139-189) with explicitly rounded operations in the
// reference's expression order, shared by the trig64 walk (trig64.cu) and the
// biased k-nearest composite (exact.cu).
#pragma once
#include <cmath>

#include "srt_device.cuh"

namespace srt {

namespace t64 {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
// a*x + b*y + c*z with Python's left-to-right rounding
__device__ __forceinline__ double dot3(double a, double x, double b, double y, double c, double z) {
    return add(add(mul(a, x), mul(b, y)), mul(c, z));
}

// kernels.py:47-51
__device__ __forceinline__ double fract(double x) {
    double r = sub(x, floor(x));
    return r >= 1.0 ? 0.0 : r;
}

// kernels.py:55-60 (sampling.py:41-46 constants)
__device__ __forceinline__ double hash_position(double x, double y, double z, int slot) {
    if (slot != 0) z = add(z, mul((double)slot, 0.6180339887498949));
    double r1 = fract(mul(47453.5453, sin(mul(91.3458, z))));
    double s = add(mul(12.9898, add(x, r1)), mul(78.233, add(y, r1)));
    return fract(mul(43758.5453, sin(s)));
}

struct Ray64 {
    double ox, oy, oz, dx, dy, dz, t_min, t_max;
};

// kernels.py:139-189, expression for expression
template <int MODE>
__device__ __forceinline__ bool candidate(const Ray64 &r, const double *m, const double *c, double s2, double &t,
                                          double &resid, double &hx, double &hy, double &hz) {
    double mx = m[0], my = m[1], mz = m[2];
    double a00 = c[0], a01 = c[1], a02 = c[2], a11 = c[3], a12 = c[4], a22 = c[5];
    double vx = sub(r.ox, mx), vy = sub(r.oy, my), vz = sub(r.oz, mz);
    double avx = dot3(a00, vx, a01, vy, a02, vz);
    double avy = dot3(a01, vx, a11, vy, a12, vz);
    double avz = dot3(a02, vx, a12, vy, a22, vz);
    double adx = dot3(a00, r.dx, a01, r.dy, a02, r.dz);
    double ady = dot3(a01, r.dx, a11, r.dy, a12, r.dz);
    double adz = dot3(a02, r.dx, a12, r.dy, a22, r.dz);
    double dad = dot3(r.dx, adx, r.dy, ady, r.dz, adz);
    if (!isfinite(dad) || dad <= 0.0) return false;
    double dav = dot3(r.dx, avx, r.dy, avy, r.dz, avz);
    double vav = dot3(vx, avx, vy, avy, vz, avz);
    resid = sub(vav, dv(mul(dav, dav), dad));
    if (resid < 0.0) resid = 0.0;
    double mah;
    if (MODE == 0) {
        t = dv(-dav, dad);
        mah = resid;
    } else {
        t = dot3(sub(mx, r.ox), r.dx, sub(my, r.oy), r.dy, sub(mz, r.oz), r.dz);
        double qx = add(vx, mul(t, r.dx)), qy = add(vy, mul(t, r.dy)), qz = add(vz, mul(t, r.dz));
        mah = add(add(mul(qx, dot3(a00, qx, a01, qy, a02, qz)), mul(qy, dot3(a01, qx, a11, qy, a12, qz))),
                  mul(qz, dot3(a02, qx, a12, qy, a22, qz)));
    }
    if (!isfinite(t) || mah > s2) return false;
    hx = add(r.ox, mul(t, r.dx));
    hy = add(r.oy, mul(t, r.dy));
    hz = add(r.oz, mul(t, r.dz));
    return true;
}

}  // namespace t64

}  // namespace srt
