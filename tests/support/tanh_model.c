/* Host restatement of csrc/glibc_tanh.cuh (same operations, same FMA sites),
 * checked against the host libm by tests/test_oracle.py::test_glibc_tanh_model.
 * Test support only. */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static inline uint32_t HI(double x){uint64_t u;memcpy(&u,&x,8);return u>>32;}
static inline double SETHI(double x,uint32_t h){uint64_t u;memcpy(&u,&x,8);u=(u&0xffffffffull)|((uint64_t)h<<32);memcpy(&x,&u,8);return x;}
static const double one=1.0,tiny=1.0e-300,
ln2_hi=6.93147180369123816490e-01,ln2_lo=1.90821492927058770002e-10,invln2=1.44269504088896338700e+00,
Q1=-3.33333333333331316428e-02,Q2=1.58730158725481460165e-03,Q3=-7.93650757867487942473e-05,Q4=4.00821782732936239552e-06,Q5=-2.01099218183624371326e-07;
double my_expm1(double x){
  double y,hi,lo,c=0,t,e,hxs,hfx,r1; int k,xsb; uint32_t hx=HI(x);
  xsb=hx&0x80000000; hx&=0x7fffffff;
  if(hx>=0x4043687A){ if(xsb){return tiny-one;} }
  if(hx>0x3fd62e42){
    if(hx<0x3FF0A2B2){ if(!xsb){hi=x-ln2_hi;lo=ln2_lo;k=1;} else {hi=x+ln2_hi;lo=-ln2_lo;k=-1;} }
    else { k=(int)fma(invln2,x,(xsb==0?0.5:-0.5)); t=k; hi=fma(-t,ln2_hi,x); lo=t*ln2_lo; }
    x=hi-lo; c=(hi-x)-lo;
  } else if(hx<0x3c900000){ return x; } else k=0;
  hfx=0.5*x; hxs=x*hfx;
  double R1=fma(hxs,Q1,one), h2=hxs*hxs, R2=fma(hxs,Q3,Q2), h4=h2*h2, R3=fma(hxs,Q5,Q4);
  r1=fma(h4,R3,fma(h2,R2,R1));
  t=fma(-r1,hfx,3.0); e=hxs*((r1-t)/fma(-x,t,6.0));
  if(k==0) return x-fma(x,e,-hxs);
  e=fma(x,e-c,-c); e-=hxs;
  if(k==-1) return fma(0.5,x-e,-0.5);
  if(k==1){ if(x<-0.25) return -2.0*(e-(x+0.5)); else return fma(2.0,x-e,one); }
  if(k<=-2||k>56){ y=one-(e-x); y=SETHI(y,HI(y)+(k<<20)); return y-one; }
  t=one;
  if(k<20){ t=SETHI(t,0x3ff00000-(0x200000>>k)); y=t-(e-x); y=SETHI(y,HI(y)+(k<<20)); }
  else { t=SETHI(0.0,((0x3ff-k)<<20)); y=x-(e+t); y+=one; y=SETHI(y,HI(y)+(k<<20)); }
  return y;
}
double my_tanh(double x){
  uint32_t jx=HI(x), ix=jx&0x7fffffff; double t,z;
  if(ix<0x40360000){
    if(ix<0x3c800000) return x*(one+x);
    if(ix>=0x3ff00000){ t=my_expm1(2.0*fabs(x)); z=one-2.0/(t+2.0); }
    else { t=my_expm1(-2.0*fabs(x)); z=-t/(t+2.0); }
  } else z=one-tiny;
  return (int32_t)jx>=0? z:-z;
}
int main(int argc,char**argv){
  srand(7); long bad=0,bade=0,n=argc>1?atol(argv[1]):1000000;
  for(long i=0;i<n;i++){
    double u=(double)rand()/RAND_MAX, v=(double)rand()/RAND_MAX;
    double x=(u*2-1)*pow(2.0, v*12-10)*12;
    if(my_tanh(x)!=tanh(x)) { if(bad<3) printf("tanh x=%.17g mine=%.17g glibc=%.17g\n",x,my_tanh(x),tanh(x)); bad++; }
    double y=(u*2-1)*60*v;
    if(my_expm1(y)!=expm1(y)) bade++;
  }
  printf("samples %ld mismatches %ld\n",n,bad+bade);
}
