/* Exhaustive check of edge8's magnitude rounding (csrc/cuda/edge8.cu
 * e8_round_sqrt16): for every n = gx^2 + gy^2 in [0, 2 * 1020^2] and
 * approximate roots perturbed by up to +-7.5e-7 relative (sqrt.approx.f32
 * is within 2^-22), the sequence
 *   km = fma_rd(s, 1/16, 2^23); v = fma(km, 16, -(2^27 - 8)); u = fma(v, v, -n64)
 *   k  = low 16 bits of fma_ru(u, -2^-21, km)   (km + 1 exactly when u < 0)
 * equals llround(sqrt((double) n)), the reference's Magnitude
 * (ref:src/registry.cpp:555-575).  Run by tests/test_cpu_oracle.py. */
#include <math.h>
#include <fenv.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static float fma_rd(float a, float b, float c){ fesetround(FE_DOWNWARD); volatile float r = fmaf(a,b,c); fesetround(FE_TONEAREST); return r; }
static float fma_ru(float a, float b, float c){ fesetround(FE_UPWARD); volatile float r = fmaf(a,b,c); fesetround(FE_TONEAREST); return r; }
static uint32_t bits(float f){ uint32_t u; memcpy(&u,&f,4); return u; }
int main(){
  long bad=0;
  for (long n=0; n<=2*1020*1020; ++n){
    float n64 = (float)(256*n+64);
    if ((long)n64 != 256*n+64) { printf("n64 inexact %ld\n", n); return 1; }
    long kstar = llround(sqrt((double)n));
    for (int p=-3;p<=3;++p){
      float s = sqrtf(n64); s = s*(1.0f+ p*2.5e-7f);  // perturbed approx root
      float km = fma_rd(s, 0.0625f, 8388608.f);
      float v = fmaf(km, 16.f, -134217720.f);
      float u = fmaf(v, v, -n64);
      uint32_t kb = bits(fma_ru(u, -4.76837158203125e-07f, km));
      if (kb != bits(km) + (bits(u)>>31)) { if (bad<10) printf("ru step differs n=%ld\n", n); ++bad; }
      long k = kb & 0xFFFF;
      if (k != kstar) { if (bad<10) printf("n=%ld p=%d k=%ld want %ld\n", n,p,k,kstar); ++bad; }
    }
  }
  printf("bad=%ld\n", bad); return 0;
}
