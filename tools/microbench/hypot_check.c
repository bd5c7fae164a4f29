// hypot_check.c — the device replay-PNG amplitude (capi.cu ref_hypot) must equal
// glibc hypot bit for bit: this restatement of the same sequence is compared
// with the host libm on 3e7 float pairs.  gcc -O2 -ffp-contract=off hypot_check.c -lm
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
// Borges, "An Improved Algorithm for hypot(a,b)" (arXiv:1904.09481), the
// corrected (non-FMA) variant, for ax >= ay > 0.
static double kern(double ax, double ay) {
    double t1, t2, h = sqrt(ax * ax + ay * ay);
    if (h <= 2.0 * ay) {
        double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}
static double hyp(double x, double y) {
    x = fabs(x); y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ay <= ax * 0x1p-54) return ax + ay;
    return kern(ax, ay);
}
int main() {
    srand(7);
    long bad = 0, N = 30000000;
    for (long i = 0; i < N; ++i) {
        double u = rand() / (double)RAND_MAX, v = rand() / (double)RAND_MAX;
        int ex = rand() % 60 - 30, ey = (rand() % 8 == 0) ? ex - (rand() % 40) : ex + (rand() % 5 - 2);
        float x = (float)ldexp(u * 2 - 1, ex), y = (float)ldexp(v * 2 - 1, ey);
        if (i % 1000 == 0) y = 0.0f;
        double g = hypot(x, y), m = hyp(x, y);
        if (g != m) { if (bad < 5) printf("x=%a y=%a glibc=%a mine=%a\n", x, y, g, m); ++bad; }
    }
    printf("N=%ld mismatches %ld\n", N, bad);
}
