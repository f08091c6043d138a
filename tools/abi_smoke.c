/* Minimal C client of libsrt (include/srt.h): builds a tiny scene, an LBVH,
 * traces a few rays and renders a small frame.  Useful to debug the ABI
 * without Python. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "../include/srt.h"

int main(void) {
    enum { N = 64 };
    double means[N * 3], cov[N * 6], op[N], sh[N * 3];
    for (int i = 0; i < N; ++i) {
        means[i * 3] = (i % 4) * 0.5 - 0.75;
        means[i * 3 + 1] = ((i / 4) % 4) * 0.5 - 0.75;
        means[i * 3 + 2] = (i / 16) * 0.5;
        cov[i * 6 + 0] = 100; cov[i * 6 + 1] = 0; cov[i * 6 + 2] = 0;
        cov[i * 6 + 3] = 100; cov[i * 6 + 4] = 0; cov[i * 6 + 5] = 100;
        op[i] = 0.5;
        sh[i * 3] = sh[i * 3 + 1] = sh[i * 3 + 2] = 1.0;
    }
    SrtSceneDesc d = {N, means, cov, op, sh, 0};
    SrtScene *s = NULL;
    int rc = srt_scene_create(&d, 0, &s);
    printf("create %d %s\n", rc, srt_last_error()); fflush(stdout);
    rc = srt_bvh_build(s, 2.8284271247461903);
    printf("build %d %s\n", rc, srt_last_error()); fflush(stdout);
    double o[6] = {0, 0, -5, 0.1, 0.1, -5}, dir[6] = {0, 0, 1, 0, 0, 1};
    double t[2]; int64_t id[2];
    SrtTraceParams p = {0.0, 1e300, 0, 1, 8.0, SRT_RNG_COUNTER, 0, 0, 0, NULL, 0};
    rc = srt_trace_rays(s, &p, o, dir, 2, 1, t, id);
    printf("trace %d %s -> %g %lld %g %lld\n", rc, srt_last_error(), t[0], (long long)id[0], t[1], (long long)id[1]);
    fflush(stdout);
    srt_scene_destroy(s);
    return 0;
}
