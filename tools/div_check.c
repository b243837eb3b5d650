// Markstein division check (svx_update.cu div_rn): q = a*y, r = fma(-q, b, a), q2 = fma(r, y, q)
// with y = 1/b must equal a/b bit for bit.  gcc -O2 -o /tmp/div_check tools/div_check.c -lm -include stdlib.h
// && /tmp/div_check 200000000   (prints "checked N bad 0")
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static inline uint64_t xr(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static inline double ud(void){ return (xr() >> 11) * (1.0/9007199254740992.0); }
int main(int argc, char** argv){
  long n = atol(argv[1]); long bad = 0;
  for (long i = 0; i < n; ++i) {
    double b;
    int mode = i % 4;
    if (mode == 0) b = (double)(1 + xr() % 20000);                 /* nobs */
    else if (mode == 1) b = fmax(ud()*1000.0, 1.0) + (double)(1 + xr()%5000); /* lam_post */
    else if (mode == 2) b = ldexp(1.0 + ud(), (int)(xr()%60) - 30);
    else b = (double)(1 + xr() % 300) + ud();
    double a = (ud() - 0.5) * ldexp(1.0, (int)(xr() % 80) - 40);
    if (i % 7 == 0) a = (double)(float)a;
    double y = 1.0 / b;
    double q = a * y;
    double r = fma(-q, b, a);
    double q2 = fma(r, y, q);
    double t = a / b;
    if (memcmp(&q2, &t, 8) != 0) { if (bad < 5) printf("a=%.17g b=%.17g got %.17g want %.17g\n", a, b, q2, t); ++bad; }
  }
  printf("checked %ld bad %ld\n", n, bad);
  return 0;
}
