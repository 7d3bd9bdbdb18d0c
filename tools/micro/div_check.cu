// Host check that ss::div_rn(a, b, RN(1/b)) == a / b (correctly rounded).
//   nvcc -O2 -std=c++17 tools/micro/div_check.cu -o /tmp/div_check && /tmp/div_check [n]
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2601_22074_b200/csrc/ss_device.cuh"

static unsigned long long st = 88172645463325252ull;
static unsigned long long xr() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
}
static double rnd(double lo, double hi) { return lo + (hi - lo) * ((xr() >> 11) * 0x1p-53); }

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 40000000;
    long long bad = 0, total = 0;
    const double spacings[] = {0.05, 0.1, 0.025, 0.2, 0.02, 0.3, 0.07};
    for (double b : spacings) {
        const double y = 1.0 / b;
        for (long i = 0; i < n; ++i) {
            const double a = (i & 1) ? rnd(-50, 50) : ldexp(rnd(1, 2), (int)(xr() % 80) - 40) * ((xr() & 1) ? 1 : -1);
            bad += ss::div_rn(a, b, y) != a / b;
            ++total;
        }
    }
    for (long i = 0; i < 2 * n; ++i) {
        const double b = ldexp(rnd(1, 2), (int)(xr() % 20) - 10), a = ldexp(rnd(1, 2), (int)(xr() % 40) - 20);
        bad += ss::div_rn(a, b, 1.0 / b) != a / b;
        ++total;
    }
    const double big = 1.7e308;
    const bool ovf_ok = ss::div_rn(big, 0.05, 20.0) == big / 0.05 && ss::div_rn(-big, 0.05, 20.0) == -big / 0.05;
    printf("mismatches %lld of %lld, overflow %s\n", bad, total, ovf_ok ? "ok" : "WRONG");
    return bad == 0 && ovf_ok ? 0 : 1;
}
