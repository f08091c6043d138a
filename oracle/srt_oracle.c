/*
 * srt_oracle.c -- CPU restatement of the reference's stochastic Gaussian
 * tracer.  TEST INFRASTRUCTURE ONLY: this is the parity checker for the
 * sm_100a product path (paper_2504_06598_b200/csrc) and the CPU baseline of
 * bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load it; the product never does.
 *
 * Every function follows the reference expression for expression, in IEEE
 * double, with no FMA contraction (built with -ffp-contract=off), so that in
 * RNG mode SRT_RNG_TRIG it reproduces the reference bit for bit (pinned by
 * tests/golden, generated from the reference by oracle/gen_golden.py).
 * The only deliberate departure is the acceptance draw
 * (/root/reference/pkg/src/splatray/kernels.py:354), which is switchable:
 *
 *   SRT_RNG_TRIG    reference trig hash of the fp64 hit position
 *                   (kernels.py:47-60, sampling.py:50-78)
 *   SRT_RNG_COUNTER counter hash u(seed, ray, sample, prim) -- the stream the
 *                   GPU reproduces bit for bit
 *   SRT_RNG_TABLE   explicit per-(prim, slot) uniforms (scripted tests,
 *                   tests/test_tracer.py:28-121 of the reference)
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SRT_RNG_TRIG 0
#define SRT_RNG_COUNTER 1
#define SRT_RNG_TABLE 2

#define STACK_SIZE 128 /* kernels.py:26 */

/* sampling.py:28, sampling.py:41-46 */
static const double SLOT_OFFSET = 0.6180339887498949;
static const double HA1 = 91.3458;
static const double HB1 = 47453.5453;
static const double HA2X = 12.9898;
static const double HA2Y = 78.233;
static const double HB2X = 43758.5453;

/* gaussians.py:26-43 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* ------------------------------------------------------------------------ */
/* randomness                                                               */
/* ------------------------------------------------------------------------ */

/* kernels.py:47-51 */
static double fract_(double x) {
    double r = x - floor(x);
    if (r >= 1.0) r = 0.0;
    return r;
}

/* kernels.py:55-60 */
double srt_oracle_hash_position(double x, double y, double z, int64_t slot) {
    if (slot != 0) z = z + (double)slot * SLOT_OFFSET;
    double r1 = fract_(HB1 * sin(HA1 * z));
    double s = HA2X * (x + r1) + HA2Y * (y + r1);
    return fract_(HB2X * sin(s));
}

/* Counter RNG: lowbias32 mixer. */
static inline uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

uint32_t srt_oracle_walk_key(uint32_t seed, uint32_t ray_id, uint32_t sample) {
    return mix32(mix32(mix32(seed ^ 0x9E3779B9u) ^ ray_id) ^ sample);
}

double srt_oracle_counter_u(uint32_t key, uint32_t prim) {
    uint32_t h = mix32(mix32(key ^ prim) ^ 0x68E31DA4u);
    return (double)(h >> 8) * (1.0 / 16777216.0);
}

/* kernels.py:64-71 */
static uint64_t wang32(uint64_t x) {
    const uint64_t M = 0xFFFFFFFFull;
    x = x & M;
    x = (x ^ 61ull) ^ (x >> 16);
    x = (x * 9ull) & M;
    x = x ^ (x >> 4);
    x = (x * 0x27D4EB2Dull) & M;
    x = x ^ (x >> 15);
    return x;
}

/* kernels.py:74-84: direction numbers of Sobol dimension 1 (x^2+x+1). */
static uint64_t SOBOL_V2[32];
static int sobol_ready = 0;
static void sobol_init(void) {
    if (sobol_ready) return;
    uint64_t m = 1;
    for (int k = 0; k < 32; ++k) {
        SOBOL_V2[k] = m << (31 - k);
        m = m ^ (m << 1);
        m &= (1ull << (k + 2)) - 1ull;
    }
    sobol_ready = 1;
}

/* kernels.py:88-103 */
static void sobol2_bits(uint64_t index, uint64_t *bx, uint64_t *by) {
    const uint64_t M = 0xFFFFFFFFull;
    uint64_t i = index & M;
    i = ((i & 0x55555555ull) << 1) | ((i >> 1) & 0x55555555ull);
    i = ((i & 0x33333333ull) << 2) | ((i >> 2) & 0x33333333ull);
    i = ((i & 0x0F0F0F0Full) << 4) | ((i >> 4) & 0x0F0F0F0Full);
    i = ((i & 0x00FF00FFull) << 8) | ((i >> 8) & 0x00FF00FFull);
    *bx = ((i << 16) | (i >> 16)) & M;
    uint64_t y = 0, j = index & M;
    int k = 0;
    while (j != 0) {
        if (j & 1ull) y ^= SOBOL_V2[k];
        j >>= 1;
        k += 1;
    }
    *by = y & M;
}

/* kernels.py:107-116 */
void srt_oracle_pixel_jitter(int64_t px, int64_t py, int64_t frame, int64_t seed, double *jx,
                             double *jy) {
    const uint64_t M = 0xFFFFFFFFull;
    sobol_init();
    uint64_t base = wang32((((uint64_t)px * 0x9E3779B1ull) & M) ^ (((uint64_t)py * 0x85EBCA77ull) & M) ^
                           (((uint64_t)seed * 0xC2B2AE3Dull) & M));
    uint64_t sx = wang32(base ^ 0x68E31DA4ull);
    uint64_t sy = wang32(base ^ 0xB5297A4Dull);
    uint64_t bx, by;
    sobol2_bits((uint64_t)frame, &bx, &by);
    *jx = (double)(bx ^ sx) * (1.0 / 4294967296.0);
    *jy = (double)(by ^ sy) * (1.0 / 4294967296.0);
}

/* ------------------------------------------------------------------------ */
/* per-primitive response                                                   */
/* ------------------------------------------------------------------------ */

typedef struct {
    const double *means;    /* (n,3) */
    const double *cov6;     /* (n,6) */
    const double *opac;     /* (n,)  */
    const double *sh;       /* (n,3,K) */
    int64_t n;
    int64_t deg;
} Scene;

typedef struct {
    const double *node_lo, *node_hi; /* (M,3) */
    const int64_t *node_left, *node_right, *node_count;
    const int64_t *prim_order;
    const double *prim_lo, *prim_hi; /* (n,3) */
    int64_t num_nodes;
} Bvh;

typedef struct {
    int mode;       /* 0 mean, 1 center */
    double s2;
    int clip;
    int rng;        /* SRT_RNG_* */
    uint32_t seed;
    const double *table; /* SRT_RNG_TABLE: (n, table_slots) */
    int64_t table_slots;
} TraceCfg;

/* optional per-walk work counters (I / P / C / draws / hits) */
typedef struct {
    int64_t inner, prim_tests, candidates, draws, hits, max_depth;
} Counters;

/* kernels.py:139-189 */
static int candidate(const Scene *sc, int64_t pid, double ox, double oy, double oz, double dx,
                     double dy, double dz, int mode, double s2, double *t_out, double *resid_out,
                     double *hx, double *hy, double *hz) {
    double mx = sc->means[pid * 3 + 0];
    double my = sc->means[pid * 3 + 1];
    double mz = sc->means[pid * 3 + 2];
    const double *c = sc->cov6 + pid * 6;
    double a00 = c[0], a01 = c[1], a02 = c[2], a11 = c[3], a12 = c[4], a22 = c[5];
    double vx = ox - mx;
    double vy = oy - my;
    double vz = oz - mz;
    double avx = a00 * vx + a01 * vy + a02 * vz;
    double avy = a01 * vx + a11 * vy + a12 * vz;
    double avz = a02 * vx + a12 * vy + a22 * vz;
    double adx = a00 * dx + a01 * dy + a02 * dz;
    double ady = a01 * dx + a11 * dy + a12 * dz;
    double adz = a02 * dx + a12 * dy + a22 * dz;
    double dad = dx * adx + dy * ady + dz * adz;
    if (!isfinite(dad) || dad <= 0.0) return 0;
    double dav = dx * avx + dy * avy + dz * avz;
    double vav = vx * avx + vy * avy + vz * avz;
    double residual = vav - dav * dav / dad;
    if (residual < 0.0) residual = 0.0;
    double t, mah;
    if (mode == 0) {
        t = -dav / dad;
        mah = residual;
    } else {
        t = (mx - ox) * dx + (my - oy) * dy + (mz - oz) * dz;
        double qx = vx + t * dx;
        double qy = vy + t * dy;
        double qz = vz + t * dz;
        mah = qx * (a00 * qx + a01 * qy + a02 * qz) + qy * (a01 * qx + a11 * qy + a12 * qz) +
              qz * (a02 * qx + a12 * qy + a22 * qz);
    }
    *resid_out = residual;
    if (!isfinite(t) || mah > s2) return 0;
    *t_out = t;
    *hx = ox + t * dx;
    *hy = oy + t * dy;
    *hz = oz + t * dz;
    return 1;
}

/* kernels.py:193-257 */
void srt_oracle_sh_color(const double *sh, int64_t deg, int64_t pid, double x, double y, double z,
                         double *out) {
    int64_t K = (deg + 1) * (deg + 1);
    const double *s0 = sh + (pid * 3 + 0) * K;
    const double *s1 = sh + (pid * 3 + 1) * K;
    const double *s2 = sh + (pid * 3 + 2) * K;
    const double *ch[3] = {s0, s1, s2};
    double r = SH_C0 * s0[0];
    double g = SH_C0 * s1[0];
    double b = SH_C0 * s2[0];
    if (deg >= 1) {
        r = r - SH_C1 * y * s0[1] + SH_C1 * z * s0[2] - SH_C1 * x * s0[3];
        g = g - SH_C1 * y * s1[1] + SH_C1 * z * s1[2] - SH_C1 * x * s1[3];
        b = b - SH_C1 * y * s2[1] + SH_C1 * z * s2[2] - SH_C1 * x * s2[3];
    }
    if (deg >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        double b0 = x * y;
        double b1 = y * z;
        double b2 = 2.0 * zz - xx - yy;
        double b3 = x * z;
        double b4 = xx - yy;
        double acc[3] = {r, g, b};
        for (int c = 0; c < 3; ++c) {
            const double *s = ch[c];
            double val = SH_C2[0] * b0 * s[4] + SH_C2[1] * b1 * s[5] + SH_C2[2] * b2 * s[6] +
                         SH_C2[3] * b3 * s[7] + SH_C2[4] * b4 * s[8];
            acc[c] += val;
        }
        if (deg >= 3) {
            double c0 = y * (3.0 * xx - yy);
            double c1 = b0 * z;
            double c2 = y * (4.0 * zz - xx - yy);
            double c3 = z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            double c4 = x * (4.0 * zz - xx - yy);
            double c5 = z * b4;
            double c6 = x * (xx - 3.0 * yy);
            for (int c = 0; c < 3; ++c) {
                const double *s = ch[c];
                double val = SH_C3[0] * c0 * s[9] + SH_C3[1] * c1 * s[10] + SH_C3[2] * c2 * s[11] +
                             SH_C3[3] * c3 * s[12] + SH_C3[4] * c4 * s[13] + SH_C3[5] * c5 * s[14] +
                             SH_C3[6] * c6 * s[15];
                acc[c] += val;
            }
        }
        r = acc[0];
        g = acc[1];
        b = acc[2];
    }
    r += 0.5;
    g += 0.5;
    b += 0.5;
    if (r < 0.0) r = 0.0;
    if (g < 0.0) g = 0.0;
    if (b < 0.0) b = 0.0;
    out[0] = r;
    out[1] = g;
    out[2] = b;
}

/* ------------------------------------------------------------------------ */
/* traversal                                                                */
/* ------------------------------------------------------------------------ */

/* kernels.py:266-308 (also bvh.py:201-226) */
static double slab_entry(const double *lo, const double *hi, int64_t id, double ox, double oy,
                         double oz, double dx, double dy, double dz, double t_min, double t_max) {
    const double *l = lo + id * 3, *h = hi + id * 3;
    double t0 = t_min, t1 = t_max;
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0) {
            double ta = (l[a] - o[a]) / d[a];
            double tb = (h[a] - o[a]) / d[a];
            if (ta > tb) {
                double tmp = ta;
                ta = tb;
                tb = tmp;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
            if (t0 > t1) return INFINITY;
        } else if (o[a] < l[a] || o[a] > h[a]) {
            return INFINITY;
        }
    }
    return t0;
}

static inline double draw(const TraceCfg *cfg, int64_t pid, int64_t k, double hx, double hy,
                          double hz, const uint32_t *keys) {
    switch (cfg->rng) {
    case SRT_RNG_COUNTER:
        return srt_oracle_counter_u(keys[k], (uint32_t)pid);
    case SRT_RNG_TABLE:
        return cfg->table[pid * cfg->table_slots + k];
    default:
        return srt_oracle_hash_position(hx, hy, hz, k);
    }
}

/* kernels.py:312-388.  keys[k] = walk key of slot k (counter mode only). */
static void trace_slots(const Bvh *bv, const Scene *sc, double ox, double oy, double oz, double dx,
                        double dy, double dz, double t_min, double t_max0, const TraceCfg *cfg,
                        const uint32_t *keys, int64_t nslots, double *slot_t, int64_t *slot_id,
                        Counters *cnt) {
    for (int64_t k = 0; k < nslots; ++k) {
        slot_t[k] = INFINITY;
        slot_id[k] = -1;
    }
    if (bv->num_nodes == 0) return;
    double far = t_max0;
    double entry = slab_entry(bv->node_lo, bv->node_hi, 0, ox, oy, oz, dx, dy, dz, t_min, far);
    if (entry == INFINITY) return;
    int64_t stack_id[STACK_SIZE];
    double stack_t[STACK_SIZE];
    stack_id[0] = 0;
    stack_t[0] = entry;
    int64_t sp = 1;
    while (sp > 0) {
        if (cnt && sp > cnt->max_depth) cnt->max_depth = sp;
        sp -= 1;
        int64_t nid = stack_id[sp];
        if (stack_t[sp] > far) continue;
        int64_t count = bv->node_count[nid];
        if (count > 0) {
            int64_t start = bv->node_left[nid];
            for (int64_t idx = start; idx < start + count; ++idx) {
                int64_t pid = bv->prim_order[idx];
                if (cnt) cnt->prim_tests++;
                if (slab_entry(bv->prim_lo, bv->prim_hi, pid, ox, oy, oz, dx, dy, dz, t_min, far) ==
                    INFINITY)
                    continue;
                if (cnt) cnt->candidates++;
                double t = 0, resid = 0, hx = 0, hy = 0, hz = 0;
                int valid = candidate(sc, pid, ox, oy, oz, dx, dy, dz, cfg->mode, cfg->s2, &t, &resid,
                                      &hx, &hy, &hz);
                if (!valid || t <= t_min || t >= t_max0) continue;
                double alpha = sc->opac[pid] * exp(-0.5 * resid);
                int improved = 0;
                for (int64_t k = 0; k < nslots; ++k) {
                    if (t < slot_t[k]) {
                        if (cnt) cnt->draws++;
                        if (draw(cfg, pid, k, hx, hy, hz, keys) < alpha) {
                            slot_t[k] = t;
                            slot_id[k] = pid;
                            improved = 1;
                        }
                    }
                }
                if (improved && cfg->clip) {
                    double worst = slot_t[0];
                    for (int64_t k = 1; k < nslots; ++k)
                        if (slot_t[k] > worst) worst = slot_t[k];
                    if (worst < far) far = worst;
                }
            }
        } else {
            if (cnt) cnt->inner++;
            int64_t lid = bv->node_left[nid];
            int64_t rid = bv->node_right[nid];
            double el = slab_entry(bv->node_lo, bv->node_hi, lid, ox, oy, oz, dx, dy, dz, t_min, far);
            double er = slab_entry(bv->node_lo, bv->node_hi, rid, ox, oy, oz, dx, dy, dz, t_min, far);
            if (el <= er) {
                if (er != INFINITY) {
                    stack_id[sp] = rid;
                    stack_t[sp] = er;
                    sp++;
                }
                if (el != INFINITY) {
                    stack_id[sp] = lid;
                    stack_t[sp] = el;
                    sp++;
                }
            } else {
                if (el != INFINITY) {
                    stack_id[sp] = lid;
                    stack_t[sp] = el;
                    sp++;
                }
                if (er != INFINITY) {
                    stack_id[sp] = rid;
                    stack_t[sp] = er;
                    sp++;
                }
            }
        }
    }
    if (cnt)
        for (int64_t k = 0; k < nslots; ++k)
            if (slot_id[k] >= 0) cnt->hits++;
}

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

int srt_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* kernels.py:527-540 (trace_batch), with ray_id = ray_id0 + i and
 * sample = sample0 + k in counter mode. */
void srt_oracle_trace_batch(const double *node_lo, const double *node_hi, const int64_t *node_left,
                            const int64_t *node_right, const int64_t *node_count, int64_t num_nodes,
                            const int64_t *prim_order, const double *prim_lo, const double *prim_hi,
                            const double *means, const double *cov6, const double *opac, int64_t n,
                            const double *origins, const double *dirs, int64_t R, double t_min,
                            double t_max, int mode, double s2, int clip, int rng, uint32_t seed,
                            uint32_t ray_id0, uint32_t sample0, const double *table,
                            int64_t table_slots, int64_t nslots, double *out_t, int64_t *out_id,
                            int64_t *counters, int threads) {
    Bvh bv = {node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi, num_nodes};
    Scene sc = {means, cov6, opac, NULL, n, 0};
    TraceCfg cfg = {mode, s2, clip, rng, seed, table, table_slots};
    set_threads(threads);
    int64_t tot[6] = {0, 0, 0, 0, 0, 0};
#pragma omp parallel
    {
        Counters c = {0, 0, 0, 0, 0, 0};
        uint32_t *keys = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(nslots > 0 ? nslots : 1));
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < R; ++i) {
            if (rng == SRT_RNG_COUNTER)
                for (int64_t k = 0; k < nslots; ++k)
                    keys[k] = srt_oracle_walk_key(seed, ray_id0 + (uint32_t)i, sample0 + (uint32_t)k);
            trace_slots(&bv, &sc, origins[i * 3], origins[i * 3 + 1], origins[i * 3 + 2], dirs[i * 3],
                        dirs[i * 3 + 1], dirs[i * 3 + 2], t_min, t_max, &cfg, keys, nslots,
                        out_t + i * nslots, out_id + i * nslots, counters ? &c : NULL);
        }
        free(keys);
        if (counters) {
#pragma omp critical
            {
                tot[0] += c.inner;
                tot[1] += c.prim_tests;
                tot[2] += c.candidates;
                tot[3] += c.draws;
                tot[4] += c.hits;
                if (c.max_depth > tot[5]) tot[5] = c.max_depth;
            }
        }
    }
    if (counters) memcpy(counters, tot, sizeof(tot));
}

/* kernels.py:613-618 */
static inline void camera_dir(const double *cam, double u, double v, double *dx, double *dy,
                              double *dz) {
    /* cam = ex ey ez rx ry rz ux uy uz fx fy fz half_w half_h (render.py:144-150) */
    double rx = cam[3], ry = cam[4], rz = cam[5], ux = cam[6], uy = cam[7], uz = cam[8];
    double fx = cam[9], fy = cam[10], fz = cam[11], half_w = cam[12], half_h = cam[13];
    double ddx = fx + u * half_w * rx + v * half_h * ux;
    double ddy = fy + u * half_w * ry + v * half_h * uy;
    double ddz = fz + u * half_w * rz + v * half_h * uz;
    double inv = 1.0 / sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    *dx = ddx * inv;
    *dy = ddy * inv;
    *dz = ddz * inv;
}

/* kernels.py:622-673 (render_stochastic).  Pixels may be restricted to a
 * row/column stride (bounded CPU-baseline samples); pass 1/1 for the full
 * frame.  pass0 offsets the pass index (sample sharding).  If out_ids is
 * non-NULL it receives the slot ids of pass pass0 as (H, W, nslots). */
void srt_oracle_render(const double *node_lo, const double *node_hi, const int64_t *node_left,
                       const int64_t *node_right, const int64_t *node_count, int64_t num_nodes,
                       const int64_t *prim_order, const double *prim_lo, const double *prim_hi,
                       const double *means, const double *cov6, const double *opac, const double *sh,
                       int64_t n, int64_t deg, const double *cam, int64_t width, int64_t height,
                       int64_t passes, int64_t pass0, int64_t nslots, int mode, double s2, int clip,
                       int64_t seed, int rng, const double *bg, int64_t stride_x, int64_t stride_y,
                       double *out_rgb, double *out_op, int64_t *out_ids, int64_t *counters,
                       int threads) {
    Bvh bv = {node_lo, node_hi, node_left, node_right, node_count, prim_order, prim_lo, prim_hi, num_nodes};
    Scene sc = {means, cov6, opac, sh, n, deg};
    TraceCfg cfg = {mode, s2, clip, rng, (uint32_t)seed, NULL, 0};
    const double TMAX = DBL_MAX;
    int64_t tiles_x = (width + 15) / 16, tiles_y = (height + 15) / 16;
    sobol_init();
    set_threads(threads);
    int64_t tot[6] = {0, 0, 0, 0, 0, 0};
#pragma omp parallel
    {
        Counters c = {0, 0, 0, 0, 0, 0};
        double *slot_t = (double *)malloc(sizeof(double) * (size_t)nslots);
        int64_t *slot_id = (int64_t *)malloc(sizeof(int64_t) * (size_t)nslots);
        uint32_t *keys = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)nslots);
#pragma omp for schedule(dynamic, 1)
        for (int64_t tile = 0; tile < tiles_x * tiles_y; ++tile) {
            int64_t ty = tile / tiles_x, tx = tile % tiles_x;
            int64_t y_end = (ty + 1) * 16 < height ? (ty + 1) * 16 : height;
            int64_t x_end = (tx + 1) * 16 < width ? (tx + 1) * 16 : width;
            for (int64_t py = ty * 16; py < y_end; ++py) {
                if (py % stride_y) continue;
                for (int64_t px = tx * 16; px < x_end; ++px) {
                    if (px % stride_x) continue;
                    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_o = 0.0;
                    for (int64_t f = pass0; f < pass0 + passes; ++f) {
                        double jx, jy, dx, dy, dz;
                        srt_oracle_pixel_jitter(px, py, f, seed, &jx, &jy);
                        double u = 2.0 * ((double)px + jx) / (double)width - 1.0;
                        double v = 1.0 - 2.0 * ((double)py + jy) / (double)height;
                        camera_dir(cam, u, v, &dx, &dy, &dz);
                        if (rng == SRT_RNG_COUNTER)
                            for (int64_t k = 0; k < nslots; ++k)
                                keys[k] = srt_oracle_walk_key((uint32_t)seed, (uint32_t)(py * width + px),
                                                              (uint32_t)(f * nslots + k));
                        trace_slots(&bv, &sc, cam[0], cam[1], cam[2], dx, dy, dz, 0.0, TMAX, &cfg, keys,
                                    nslots, slot_t, slot_id, counters ? &c : NULL);
                        if (out_ids && f == pass0)
                            for (int64_t k = 0; k < nslots; ++k)
                                out_ids[(py * width + px) * nslots + k] = slot_id[k];
                        for (int64_t k = 0; k < nslots; ++k) {
                            int64_t pid = slot_id[k];
                            if (pid >= 0) {
                                double col[3];
                                srt_oracle_sh_color(sh, deg, pid, dx, dy, dz, col);
                                acc_r += col[0];
                                acc_g += col[1];
                                acc_b += col[2];
                                acc_o += 1.0;
                            } else {
                                acc_r += bg[0];
                                acc_g += bg[1];
                                acc_b += bg[2];
                            }
                        }
                    }
                    double inv = 1.0 / (double)(passes * nslots);
                    out_rgb[(py * width + px) * 3 + 0] = acc_r * inv;
                    out_rgb[(py * width + px) * 3 + 1] = acc_g * inv;
                    out_rgb[(py * width + px) * 3 + 2] = acc_b * inv;
                    out_op[py * width + px] = acc_o * inv;
                }
            }
        }
        free(slot_t);
        free(slot_id);
        free(keys);
        if (counters) {
#pragma omp critical
            {
                tot[0] += c.inner;
                tot[1] += c.prim_tests;
                tot[2] += c.candidates;
                tot[3] += c.draws;
                tot[4] += c.hits;
                if (c.max_depth > tot[5]) tot[5] = c.max_depth;
            }
        }
    }
    if (counters) memcpy(counters, tot, sizeof(tot));
}

/* kernels.py:392-432 (_transmittance_one) over explicit rays. */
void srt_oracle_transmittance(const double *node_lo, const double *node_hi, const int64_t *node_left,
                              const int64_t *node_right, const int64_t *node_count, int64_t num_nodes,
                              const int64_t *prim_order, const double *prim_lo, const double *prim_hi,
                              const double *means, const double *cov6, const double *opac, int64_t n,
                              const double *origins, const double *dirs, int64_t R, double t_min,
                              double t_max, int mode, double s2, double *out, int threads) {
    Scene sc = {means, cov6, opac, NULL, n, 0};
    set_threads(threads);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < R; ++i) {
        double ox = origins[i * 3], oy = origins[i * 3 + 1], oz = origins[i * 3 + 2];
        double dx = dirs[i * 3], dy = dirs[i * 3 + 1], dz = dirs[i * 3 + 2];
        double result = 1.0;
        if (num_nodes > 0 &&
            slab_entry(node_lo, node_hi, 0, ox, oy, oz, dx, dy, dz, t_min, t_max) != INFINITY) {
            int64_t stack_id[STACK_SIZE];
            int64_t sp = 1;
            stack_id[0] = 0;
            while (sp > 0) {
                sp -= 1;
                int64_t nid = stack_id[sp];
                int64_t count = node_count[nid];
                if (count > 0) {
                    int64_t start = node_left[nid];
                    for (int64_t idx = start; idx < start + count; ++idx) {
                        int64_t pid = prim_order[idx];
                        if (slab_entry(prim_lo, prim_hi, pid, ox, oy, oz, dx, dy, dz, t_min, t_max) ==
                            INFINITY)
                            continue;
                        double t = 0, resid = 0, hx, hy, hz;
                        if (candidate(&sc, pid, ox, oy, oz, dx, dy, dz, mode, s2, &t, &resid, &hx, &hy,
                                      &hz) &&
                            t > t_min && t < t_max)
                            result *= 1.0 - opac[pid] * exp(-0.5 * resid);
                    }
                } else {
                    int64_t lid = node_left[nid], rid = node_right[nid];
                    if (slab_entry(node_lo, node_hi, lid, ox, oy, oz, dx, dy, dz, t_min, t_max) != INFINITY)
                        stack_id[sp++] = lid;
                    if (slab_entry(node_lo, node_hi, rid, ox, oy, oz, dx, dy, dz, t_min, t_max) != INFINITY)
                        stack_id[sp++] = rid;
                }
            }
        }
        out[i] = result;
    }
}

/* ------------------------------------------------------------------------ */
/* binned-SAH BVH build: bvh.py:87-193, bit for bit                          */
/* ------------------------------------------------------------------------ */

#define SAH_BINS 16      /* bvh.py:19 */
#define MAX_SAH_DEPTH 32 /* bvh.py:22 */

typedef struct {
    const double *lo, *hi;
    double *centers; /* (n,3) */
    int64_t leaf_size;
    double *node_lo, *node_hi;
    int64_t *node_left, *node_right, *node_count;
    int64_t num_nodes;
    int64_t *prim_order;
    int64_t num_prims;
    /* scratch */
    int64_t *tmp_idx;
    double *key, *tmp_key;
    double *pre_lo, *pre_hi, *suf_lo, *suf_hi;
} Builder;

/* stable merge sort of ids[0..m) by key[0..m) (np.argsort kind="stable") */
static void stable_sort(int64_t *ids, double *key, int64_t m, int64_t *tmp_ids, double *tmp_key) {
    for (int64_t width = 1; width < m; width *= 2) {
        for (int64_t i = 0; i < m; i += 2 * width) {
            int64_t a = i, am = i + width < m ? i + width : m, b = am, bm = i + 2 * width < m ? i + 2 * width : m;
            int64_t o = i;
            while (a < am && b < bm) {
                if (key[b] < key[a]) {
                    tmp_key[o] = key[b];
                    tmp_ids[o++] = ids[b++];
                } else {
                    tmp_key[o] = key[a];
                    tmp_ids[o++] = ids[a++];
                }
            }
            while (a < am) {
                tmp_key[o] = key[a];
                tmp_ids[o++] = ids[a++];
            }
            while (b < bm) {
                tmp_key[o] = key[b];
                tmp_ids[o++] = ids[b++];
            }
        }
        memcpy(ids, tmp_ids, sizeof(int64_t) * (size_t)m);
        memcpy(key, tmp_key, sizeof(double) * (size_t)m);
    }
}

static double surface(const double *blo, const double *bhi) {
    double dx = bhi[0] - blo[0], dy = bhi[1] - blo[1], dz = bhi[2] - blo[2];
    return 2.0 * (dx * dy + dy * dz + dz * dx);
}

/* bvh.py:153-179 */
static int64_t sah_cut(Builder *B, const int64_t *order, int64_t m, int axis) {
    double *c = B->key; /* sorted keys == centers[order, axis] */
    double c0 = c[0], c1 = c[m - 1];
    int64_t counts[SAH_BINS];
    memset(counts, 0, sizeof(counts));
    for (int64_t i = 0; i < m; ++i) {
        double rel = (c[i] - c0) / (c1 - c0);
        int64_t bin = (int64_t)(rel * (double)SAH_BINS);
        if (bin > SAH_BINS - 1) bin = SAH_BINS - 1;
        counts[bin]++;
    }
    for (int64_t i = 0; i < m; ++i) {
        int64_t p = order[i];
        for (int a = 0; a < 3; ++a) {
            double l = B->lo[p * 3 + a], h = B->hi[p * 3 + a];
            B->pre_lo[i * 3 + a] = (i == 0 || l < B->pre_lo[(i - 1) * 3 + a]) ? l : B->pre_lo[(i - 1) * 3 + a];
            B->pre_hi[i * 3 + a] = (i == 0 || h > B->pre_hi[(i - 1) * 3 + a]) ? h : B->pre_hi[(i - 1) * 3 + a];
        }
    }
    for (int64_t i = m - 1; i >= 0; --i) {
        int64_t p = order[i];
        for (int a = 0; a < 3; ++a) {
            double l = B->lo[p * 3 + a], h = B->hi[p * 3 + a];
            B->suf_lo[i * 3 + a] = (i == m - 1 || l < B->suf_lo[(i + 1) * 3 + a]) ? l : B->suf_lo[(i + 1) * 3 + a];
            B->suf_hi[i * 3 + a] = (i == m - 1 || h > B->suf_hi[(i + 1) * 3 + a]) ? h : B->suf_hi[(i + 1) * 3 + a];
        }
    }
    double best_cost = INFINITY;
    int64_t best_cut = m / 2, cut = 0;
    for (int b = 0; b < SAH_BINS - 1; ++b) {
        cut += counts[b];
        if (cut == 0 || cut == m) continue;
        double cost = (double)cut * surface(B->pre_lo + (cut - 1) * 3, B->pre_hi + (cut - 1) * 3) +
                      (double)(m - cut) * surface(B->suf_lo + cut * 3, B->suf_hi + cut * 3);
        if (cost < best_cost) {
            best_cost = cost;
            best_cut = cut;
        }
    }
    return best_cut;
}

/* bvh.py:121-151: ids[0..m) is reordered in place (left part, right part). */
static int64_t build_rec(Builder *B, int64_t *ids, int64_t m, int depth) {
    int64_t nid = B->num_nodes++;
    if (m <= B->leaf_size) {
        for (int a = 0; a < 3; ++a) {
            double l = INFINITY, h = -INFINITY;
            for (int64_t i = 0; i < m; ++i) {
                double vl = B->lo[ids[i] * 3 + a], vh = B->hi[ids[i] * 3 + a];
                if (vl < l) l = vl;
                if (vh > h) h = vh;
            }
            B->node_lo[nid * 3 + a] = l;
            B->node_hi[nid * 3 + a] = h;
        }
        B->node_left[nid] = B->num_prims;
        B->node_right[nid] = -1;
        B->node_count[nid] = m;
        for (int64_t i = 0; i < m; ++i) B->prim_order[B->num_prims++] = ids[i];
        return nid;
    }
    /* _split (bvh.py:142-151) */
    double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < m; ++i)
        for (int a = 0; a < 3; ++a) {
            double c = B->centers[ids[i] * 3 + a];
            if (c < cmin[a]) cmin[a] = c;
            if (c > cmax[a]) cmax[a] = c;
        }
    double extent[3] = {cmax[0] - cmin[0], cmax[1] - cmin[1], cmax[2] - cmin[2]};
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (extent[a] > extent[axis]) axis = a;
    for (int64_t i = 0; i < m; ++i) B->key[i] = B->centers[ids[i] * 3 + axis];
    stable_sort(ids, B->key, m, B->tmp_idx, B->tmp_key);
    int64_t cut;
    if (depth >= MAX_SAH_DEPTH || extent[axis] <= 0.0)
        cut = m / 2;
    else
        cut = sah_cut(B, ids, m, axis);
    int64_t lid = build_rec(B, ids, cut, depth + 1);
    int64_t rid = build_rec(B, ids + cut, m - cut, depth + 1);
    for (int a = 0; a < 3; ++a) {
        double ll = B->node_lo[lid * 3 + a], rl = B->node_lo[rid * 3 + a];
        double lh = B->node_hi[lid * 3 + a], rh = B->node_hi[rid * 3 + a];
        B->node_lo[nid * 3 + a] = ll < rl ? ll : rl; /* np.minimum */
        B->node_hi[nid * 3 + a] = lh > rh ? lh : rh; /* np.maximum */
    }
    B->node_left[nid] = lid;
    B->node_right[nid] = rid;
    B->node_count[nid] = 0;
    return nid;
}

/* Outputs must hold 2n nodes; returns the node count (0 for n == 0). */
int64_t srt_oracle_sah_build(const double *lo, const double *hi, int64_t n, int64_t leaf_size,
                             double *node_lo, double *node_hi, int64_t *node_left,
                             int64_t *node_right, int64_t *node_count, int64_t *prim_order) {
    if (n <= 0) return 0;
    Builder B;
    memset(&B, 0, sizeof(B));
    B.lo = lo;
    B.hi = hi;
    B.leaf_size = leaf_size;
    B.node_lo = node_lo;
    B.node_hi = node_hi;
    B.node_left = node_left;
    B.node_right = node_right;
    B.node_count = node_count;
    B.prim_order = prim_order;
    B.centers = (double *)malloc(sizeof(double) * (size_t)n * 3);
    for (int64_t i = 0; i < n * 3; ++i) B.centers[i] = 0.5 * (lo[i] + hi[i]);
    B.tmp_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    B.key = (double *)malloc(sizeof(double) * (size_t)n);
    B.tmp_key = (double *)malloc(sizeof(double) * (size_t)n);
    B.pre_lo = (double *)malloc(sizeof(double) * (size_t)n * 3);
    B.pre_hi = (double *)malloc(sizeof(double) * (size_t)n * 3);
    B.suf_lo = (double *)malloc(sizeof(double) * (size_t)n * 3);
    B.suf_hi = (double *)malloc(sizeof(double) * (size_t)n * 3);
    int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) ids[i] = i;
    build_rec(&B, ids, n, 0);
    free(ids);
    free(B.centers);
    free(B.tmp_idx);
    free(B.key);
    free(B.tmp_key);
    free(B.pre_lo);
    free(B.pre_hi);
    free(B.suf_lo);
    free(B.suf_hi);
    return B.num_nodes;
}

/* ------------------------------------------------------------------------ */
/* exact compositing (brute force, no BVH): kernels.py:441-475, 584-604,    */
/* 677-723                                                                   */
/* ------------------------------------------------------------------------ */

/* stable merge sort of idx[0..m) by key (np.argsort kind="mergesort") */
static void stable_argsort(const double *key, int64_t *idx, int64_t *tmp, int64_t m) {
    for (int64_t i = 0; i < m; ++i) idx[i] = i;
    for (int64_t width = 1; width < m; width *= 2) {
        for (int64_t i = 0; i < m; i += 2 * width) {
            int64_t a = i, am = i + width < m ? i + width : m, b = am, bm = i + 2 * width < m ? i + 2 * width : m;
            int64_t o = i;
            while (a < am && b < bm) tmp[o++] = key[idx[b]] < key[idx[a]] ? idx[b++] : idx[a++];
            while (a < am) tmp[o++] = idx[a++];
            while (b < bm) tmp[o++] = idx[b++];
        }
        memcpy(idx, tmp, sizeof(int64_t) * (size_t)m);
    }
}

/* kernels.py:441-475 */
static void exact_ray(const Scene *sc, double ox, double oy, double oz, double dx, double dy, double dz,
                      double t_min, double t_max, int mode, double s2, const double *bg, double *t_buf,
                      double *a_buf, int64_t *id_buf, int64_t *order, int64_t *tmp, double *out4) {
    int64_t m = 0;
    for (int64_t pid = 0; pid < sc->n; ++pid) {
        double t = 0, resid = 0, hx, hy, hz;
        if (candidate(sc, pid, ox, oy, oz, dx, dy, dz, mode, s2, &t, &resid, &hx, &hy, &hz) && t > t_min &&
            t < t_max) {
            t_buf[m] = t;
            a_buf[m] = sc->opac[pid] * exp(-0.5 * resid);
            id_buf[m] = pid;
            m++;
        }
    }
    stable_argsort(t_buf, order, tmp, m);
    double r = 0.0, g = 0.0, b = 0.0, trans = 1.0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t j = order[i];
        double alpha = a_buf[j], col[3];
        srt_oracle_sh_color(sc->sh, sc->deg, id_buf[j], dx, dy, dz, col);
        double w = trans * alpha;
        r += w * col[0];
        g += w * col[1];
        b += w * col[2];
        trans *= 1.0 - alpha;
    }
    r += trans * bg[0];
    g += trans * bg[1];
    b += trans * bg[2];
    out4[0] = r;
    out4[1] = g;
    out4[2] = b;
    out4[3] = 1.0 - trans;
}

/* kernels.py:584-604 */
void srt_oracle_exact_batch(const double *means, const double *cov6, const double *opac, const double *sh,
                            int64_t n, int64_t deg, const double *origins, const double *dirs, int64_t R,
                            double t_min, double t_max, int mode, double s2, const double *bg, double *out_rgb,
                            double *out_op, int threads) {
    Scene sc = {means, cov6, opac, sh, n, deg};
    set_threads(threads);
#pragma omp parallel
    {
        size_t cap = (size_t)(n > 0 ? n : 1);
        double *t_buf = (double *)malloc(sizeof(double) * cap), *a_buf = (double *)malloc(sizeof(double) * cap);
        int64_t *id_buf = (int64_t *)malloc(sizeof(int64_t) * cap), *order = (int64_t *)malloc(sizeof(int64_t) * cap),
                *tmp = (int64_t *)malloc(sizeof(int64_t) * cap);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < R; ++i) {
            double o4[4];
            exact_ray(&sc, origins[i * 3], origins[i * 3 + 1], origins[i * 3 + 2], dirs[i * 3], dirs[i * 3 + 1],
                      dirs[i * 3 + 2], t_min, t_max, mode, s2, bg, t_buf, a_buf, id_buf, order, tmp, o4);
            out_rgb[i * 3] = o4[0];
            out_rgb[i * 3 + 1] = o4[1];
            out_rgb[i * 3 + 2] = o4[2];
            out_op[i] = o4[3];
        }
        free(t_buf);
        free(a_buf);
        free(id_buf);
        free(order);
        free(tmp);
    }
}

/* kernels.py:479-518 (_biased_ray): one draw per valid candidate (slot 0),
 * the kk nearest accepted composited with their own alphas.  rng selects the
 * draw: SRT_RNG_TRIG (the reference's hash), COUNTER (key from seed,
 * ray_id0 + i, sample0) or TABLE (table[pid * table_slots]). */
static void biased_ray(const Scene *sc, double ox, double oy, double oz, double dx, double dy, double dz,
                       double t_min, double t_max, int mode, double s2, int64_t kk, const double *bg,
                       const TraceCfg *cfg, uint32_t key, double *t_buf, double *a_buf, int64_t *id_buf,
                       int64_t *order, int64_t *tmp, double *out3) {
    int64_t m = 0;
    for (int64_t pid = 0; pid < sc->n; ++pid) {
        double t = 0, resid = 0, hx, hy, hz;
        if (!candidate(sc, pid, ox, oy, oz, dx, dy, dz, mode, s2, &t, &resid, &hx, &hy, &hz) || t <= t_min ||
            t >= t_max)
            continue;
        double alpha = sc->opac[pid] * exp(-0.5 * resid);
        if (draw(cfg, pid, 0, hx, hy, hz, &key) < alpha) {
            t_buf[m] = t;
            a_buf[m] = alpha;
            id_buf[m] = pid;
            m++;
        }
    }
    stable_argsort(t_buf, order, tmp, m);
    double r = 0.0, g = 0.0, b = 0.0, trans = 1.0;
    int64_t take = m < kk ? m : kk;
    for (int64_t i = 0; i < take; ++i) {
        int64_t j = order[i];
        double alpha = a_buf[j], col[3];
        srt_oracle_sh_color(sc->sh, sc->deg, id_buf[j], dx, dy, dz, col);
        double w = trans * alpha;
        r += w * col[0];
        g += w * col[1];
        b += w * col[2];
        trans *= 1.0 - alpha;
    }
    out3[0] = r + trans * bg[0];
    out3[1] = g + trans * bg[1];
    out3[2] = b + trans * bg[2];
}

/* kernels.py:561-580 */
void srt_oracle_biased_batch(const double *means, const double *cov6, const double *opac, const double *sh,
                             int64_t n, int64_t deg, const double *origins, const double *dirs, int64_t R,
                             double t_min, double t_max, int mode, double s2, int64_t kk, const double *bg,
                             int rng, uint32_t seed, uint32_t ray_id0, uint32_t sample0, const double *table,
                             int64_t table_slots, double *out_rgb, int threads) {
    Scene sc = {means, cov6, opac, sh, n, deg};
    TraceCfg cfg = {mode, s2, 0, rng, seed, table, table_slots};
    set_threads(threads);
#pragma omp parallel
    {
        size_t cap = (size_t)(n > 0 ? n : 1);
        double *t_buf = (double *)malloc(sizeof(double) * cap), *a_buf = (double *)malloc(sizeof(double) * cap);
        int64_t *id_buf = (int64_t *)malloc(sizeof(int64_t) * cap), *order = (int64_t *)malloc(sizeof(int64_t) * cap),
                *tmp = (int64_t *)malloc(sizeof(int64_t) * cap);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < R; ++i) {
            uint32_t key = srt_oracle_walk_key(seed, ray_id0 + (uint32_t)i, sample0);
            biased_ray(&sc, origins[i * 3], origins[i * 3 + 1], origins[i * 3 + 2], dirs[i * 3], dirs[i * 3 + 1],
                       dirs[i * 3 + 2], t_min, t_max, mode, s2, kk, bg, &cfg, key, t_buf, a_buf, id_buf, order, tmp,
                       out_rgb + i * 3);
        }
        free(t_buf);
        free(a_buf);
        free(id_buf);
        free(order);
        free(tmp);
    }
}

/* kernels.py:677-723 (render_exact): per-pixel mean over `frames` jittered rays */
void srt_oracle_render_exact(const double *means, const double *cov6, const double *opac, const double *sh,
                             int64_t n, int64_t deg, const double *cam, int64_t width, int64_t height,
                             int64_t frames, int mode, double s2, int64_t seed, const double *bg, double *out_rgb,
                             double *out_op, int threads) {
    Scene sc = {means, cov6, opac, sh, n, deg};
    int64_t tiles_x = (width + 15) / 16, tiles_y = (height + 15) / 16;
    sobol_init();
    set_threads(threads);
#pragma omp parallel
    {
        size_t cap = (size_t)(n > 0 ? n : 1);
        double *t_buf = (double *)malloc(sizeof(double) * cap), *a_buf = (double *)malloc(sizeof(double) * cap);
        int64_t *id_buf = (int64_t *)malloc(sizeof(int64_t) * cap), *order = (int64_t *)malloc(sizeof(int64_t) * cap),
                *tmp = (int64_t *)malloc(sizeof(int64_t) * cap);
#pragma omp for schedule(dynamic, 1)
        for (int64_t tile = 0; tile < tiles_x * tiles_y; ++tile) {
            int64_t ty = tile / tiles_x, tx = tile % tiles_x;
            int64_t y_end = (ty + 1) * 16 < height ? (ty + 1) * 16 : height;
            int64_t x_end = (tx + 1) * 16 < width ? (tx + 1) * 16 : width;
            for (int64_t py = ty * 16; py < y_end; ++py)
                for (int64_t px = tx * 16; px < x_end; ++px) {
                    double acc[4] = {0.0, 0.0, 0.0, 0.0};
                    for (int64_t f = 0; f < frames; ++f) {
                        double jx, jy, dx, dy, dz, o4[4];
                        srt_oracle_pixel_jitter(px, py, f, seed, &jx, &jy);
                        double u = 2.0 * ((double)px + jx) / (double)width - 1.0;
                        double v = 1.0 - 2.0 * ((double)py + jy) / (double)height;
                        camera_dir(cam, u, v, &dx, &dy, &dz);
                        exact_ray(&sc, cam[0], cam[1], cam[2], dx, dy, dz, 0.0, DBL_MAX, mode, s2, bg, t_buf, a_buf,
                                  id_buf, order, tmp, o4);
                        for (int c = 0; c < 4; ++c) acc[c] += o4[c];
                    }
                    double inv = 1.0 / (double)frames;
                    for (int c = 0; c < 3; ++c) out_rgb[(py * width + px) * 3 + c] = acc[c] * inv;
                    out_op[py * width + px] = acc[3] * inv;
                }
        }
        free(t_buf);
        free(a_buf);
        free(id_buf);
        free(order);
        free(tmp);
    }
}
