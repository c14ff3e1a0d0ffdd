/* Accurate-table search for the Box-Muller log (Gal's method), used by
 * tools/gen_logtab.py: for each subinterval centre c_i find a double invc near
 * 1/c_i whose 2 ln(invc) lies within 2^-66 of a multiple of 2^-43, so the table
 * needs no low-order correction term: hi = that multiple, |hi - 2 ln invc| < 2^-66.
 * Candidates step through consecutive doubles around 1/c_i; a long-double filter
 * (2^-19 in units of 2^-43) is confirmed in binary128.
 *
 *   gcc -O2 tools/gal_search.c -o /tmp/gal_search -lquadmath -lm
 *   /tmp/gal_search < centres.txt      (one "%a" centre per line) -> "i invc hi" (hex floats)
 */
#include <math.h>
#include <quadmath.h>
#include <stdio.h>
#include <stdlib.h>

int main(void) {
    double c;
    int i = 0;
    const long double S = 0x1p43L;
    while (scanf("%la", &c) == 1) {
        const double inv0 = 1.0 / c;
        /* candidates: consecutive doubles around 1/c_i, nearest first */
        union { double d; unsigned long long u; } b = {inv0};
        const unsigned long long u0 = b.u;
        int found = 0;
        for (long n = 0; n < (1L << 40) && !found; n++) {
            const long k = (n & 1) ? -(n + 1) / 2 : n / 2;
            b.u = u0 + (unsigned long long)k;
            const long double L = 2.0L * logl((long double)b.d) * S;
            const long double m = roundl(L);
            if (fabsl(L - m) > 0x1p-19L) continue;
            const __float128 Lq = 2 * logq((__float128)b.d) * (__float128)0x1p43;
            const __float128 mq = roundq(Lq);
            if (fabsq(Lq - mq) < (__float128)0x1p-23) {  /* |2 ln invc - hi| < 2^-66 */
                printf("%d %a %a\n", i, b.d, (double)(mq * (__float128)0x1p-43));
                found = 1;
            }
        }
        if (!found) { fprintf(stderr, "entry %d: not found\n", i); return 1; }
        fflush(stdout);
        i++;
    }
    return 0;
}
