// Host-side accuracy check of ss::sincos_fast against long-double sinl/cosl
// (and glibc's double sin/cos): ulp error histogram over several ranges.
//   nvcc -O2 -std=c++17 tools/micro/sincos_acc.cu -o /tmp/sincos_acc && /tmp/sincos_acc
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <random>

#include "../../paper_2601_22074_b200/csrc/ss_device.cuh"

static long long ulps(double a, double b) {
    if (a == b) return 0;
    long long ia, ib;
    memcpy(&ia, &a, 8);
    memcpy(&ib, &b, 8);
    if (ia < 0) ia = (long long)0x8000000000000000ull - ia;
    if (ib < 0) ib = (long long)0x8000000000000000ull - ib;
    return ia > ib ? ia - ib : ib - ia;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 2000000;
    long long worst = 0;
    std::mt19937_64 g(1);
    const double ranges[] = {1e-6, 0.8, 3.2, 10.0, 100.0, 1e4, 1e6 / 1.0001};
    for (double R : ranges) {
        std::uniform_real_distribution<double> U(-R, R);
        long long hist[4] = {0}, glibc_hist[4] = {0}, diff_glibc = 0;
        for (int i = 0; i < n; ++i) {
            const double x = U(g);
            double s, c;
            ss::sincos_fast(x, &s, &c);
            const double rs = (double)sinl((long double)x), rc = (double)cosl((long double)x);
            long long es = ulps(s, rs), ec = ulps(c, rc);
            worst = es > worst ? es : worst;
            worst = ec > worst ? ec : worst;
            hist[es > 2 ? 3 : es]++;
            hist[ec > 2 ? 3 : ec]++;
            long long gs = ulps(sin(x), rs), gc = ulps(cos(x), rc);
            glibc_hist[gs > 2 ? 3 : gs]++;
            glibc_hist[gc > 2 ? 3 : gc]++;
            diff_glibc += (s != sin(x)) + (c != cos(x));
        }
        printf("|x|<%-8g fast: 0ulp %.5f 1ulp %.5f 2ulp %.6f >2 %lld | glibc: 0ulp %.5f 1ulp %.5f >1 %lld | fast!=glibc %.5f\n",
               R, hist[0] / (2.0 * n), hist[1] / (2.0 * n), hist[2] / (2.0 * n), hist[3], glibc_hist[0] / (2.0 * n),
               glibc_hist[1] / (2.0 * n), glibc_hist[2] + glibc_hist[3], diff_glibc / (2.0 * n));
    }
    double s, c;
    const double specials[] = {0.0, -0.0, 1.5707963267948966, 3.141592653589793, -3.141592653589793, 1e-300};
    for (double x : specials) {
        ss::sincos_fast(x, &s, &c);
        printf("x=%.17g sin=%.17g (%.17g) cos=%.17g (%.17g)\n", x, s, sin(x), c, cos(x));
    }
    printf("worst %lld ulp\n", worst);
    return worst <= 1 ? 0 : 1;
}
