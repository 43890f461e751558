#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s=88172645463325252ull;
static uint64_t xr(){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
static double rnd(){ // random double with random exponent in [-60,60], random sign
  uint64_t m=xr()>>12; int e=(int)(xr()%121)-60; double v=ldexp(1.0+ (double)m/4503599627370496.0, e); return (xr()&1)?-v:v;}
// Markstein division check (lu2.cu div_rn): q = a*y, y = RN(1/b), q2 = fma(fma(-q,b,a),y,q)
// must equal a/b bit for bit.  gcc -O2 -march=native tools/markstein_check.c -lm && ./a.out
int main(){
  long bad=0,n=200000000;
  for(long i=0;i<n;i++){
    double a=rnd(), b=rnd();
    if(i%4==0) a = b*rnd(); // near-exact quotients
    double y=1.0/b, q=a*y, r=fma(-q,b,a), q2=fma(r,y,q);
    double t=a/b;
    if(memcmp(&q2,&t,8)){ if(bad<5) printf("a=%a b=%a q2=%a t=%a\n",a,b,q2,t); bad++; }
  }
  printf("mismatches %ld of %ld\n",bad,n);
}
