// Probe: the triangular-solve arithmetic of OpenBLAS cblas_ztrsm (the complex
// reference lu_solve, lu.hpp:52-69, used by itucker<cplx>) against candidate
// restatements; prints the number of differing doubles per candidate (0 =
// bitwise). What csrc/lu_solve.cuh uses: 4-row blocks (ZGEMM_UNROLL_M), the
// GEMM part as four real chains (rr, ii, ri, ir -> (rr - ii, ri + ir)), the
// in-block update c -= p*a as t0 = fma(p.re, a.re, -(p.im*a.im)),
// t1 = fma(p.re, a.im, p.im*a.re) (VAR 0) and the packed reciprocal diagonal
// with a fused 1 + r*r (CV 1): bitwise for extents that are multiples of 4.
// The TV variants are the M-tail dot groupings tried for the remainder
// blocks (none bitwise). Build and run:
//   OB=/opt/prime-rl/.venv/lib/python3.12/site-packages/opencv_python_headless.libs
//   gcc -O2 -ffp-contract=off tools/openblas_ztrsm_probe.c -o /tmp/zp \
//       -L$OB -l:libopenblasp-r0-59ffcd50.3.15.so -Wl,-rpath-link,$OB -lm
//   LD_LIBRARY_PATH=$OB OPENBLAS_CORETYPE=SKYLAKEX /tmp/zp 40 50
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#include <complex.h>
void cblas_ztrsm(int,int,int,int,int,int,int,const void*,const void*,int,void*,int);
static double rnd(){return (double)rand()/RAND_MAX*2-1;}
#define UM 4
static int VAR=0;
// c -= (p0 + i p1) * (a0 + i a1)
__attribute__((target("avx2,fma"))) static void upd(double*c0,double*c1,double p0,double p1,double a0,double a1){
  if(VAR==0){ double t0=fma(p0,a0,-(p1*a1)); double t1=fma(p0,a1,p1*a0); *c0=*c0-t0; *c1=*c1-t1; }
  else if(VAR==1){ *c0=fma(-p0,a0,*c0); *c0=fma(p1,a1,*c0); *c1=fma(-p0,a1,*c1); *c1=fma(-p1,a0,*c1);}
  else if(VAR==2){ double t0=p0*a0-p1*a1; double t1=p0*a1+p1*a0; *c0-=t0; *c1-=t1; }
  else if(VAR==3){ double t0=fma(-p1,a1,p0*a0); double t1=fma(p1,a0,p0*a1); *c0=*c0-t0; *c1=*c1-t1; }
  else if(VAR==4){ *c0=fma(p1,a1,*c0); *c0=fma(-p0,a0,*c0); *c1=fma(-p1,a0,*c1); *c1=fma(-p0,a1,*c1);}
}
// x <- x * inv  (inv = (i0,i1))
__attribute__((target("avx2,fma"))) static void mulinv(double*x0,double*x1,double i0,double i1){
  double b0=*x0,b1=*x1;
  if(VAR==0||VAR==3){ *x0=fma(i0,b0,-(i1*b1)); *x1=fma(i0,b1,i1*b0);} 
  else if(VAR==2){ *x0=i0*b0-i1*b1; *x1=i0*b1+i1*b0; }
  else { *x0=fma(i0,b0,-(i1*b1)); *x1=fma(i0,b1,i1*b0);} 
}
static int CV=0;
__attribute__((target("avx2,fma"))) static void compinv(double*b,double ar,double ai){
  double ratio,den;
  if(CV==0){
  if(fabs(ar)>=fabs(ai)){ratio=ai/ar; den=1./(ar*(1+ratio*ratio)); b[0]=den; b[1]=-ratio*den;}
  else {ratio=ar/ai; den=1./(ai*(1+ratio*ratio)); b[0]=ratio*den; b[1]=-den;}
  } else if(CV==1){
  if(fabs(ar)>=fabs(ai)){ratio=ai/ar; den=1./(ar*fma(ratio,ratio,1)); b[0]=den; b[1]=-ratio*den;}
  else {ratio=ar/ai; den=1./(ai*fma(ratio,ratio,1)); b[0]=ratio*den; b[1]=-den;}
  } else if(CV==2){ double d=ar*ar+ai*ai; b[0]=ar/d; b[1]=-ai/d; }
  else if(CV==3){ double d=fma(ar,ar,ai*ai); b[0]=ar/d; b[1]=-ai/d; }
  else if(CV==4){ double d=1.0/fma(ar,ar,ai*ai); b[0]=ar*d; b[1]=-ai*d; }
  else if(CV==5){ double d=1.0/(ar*ar+ai*ai); b[0]=ar*d; b[1]=-ai*d; }
}
// 4-chain dot: acc = sum_k A(r,k) x(k)
__attribute__((target("avx2,fma"))) static void dot4(const double*A,int n,int r,const double*x,int k0,int k1,double*re,double*im){
  double rr=0,ii=0,ri=0,ir=0;
  for(int k=k0;k<k1;k++){double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
    rr=fma(a0,x0,rr); ii=fma(a1,x1,ii); ri=fma(a0,x1,ri); ir=fma(a1,x0,ir);} 
  *re=rr-ii; *im=ri+ir; }
static int BS=UM; static int TV=0;
__attribute__((target("avx2,fma"))) static void dot_t(const double*A,int n,int r,const double*x,int k0,int k1,double*re,double*im){
  if(TV==0){ dot4(A,n,r,x,k0,k1,re,im); return; }
  if(TV==1){ double a=0,b=0; for(int k=k0;k<k1;k++){double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
     a=fma(a0,x0,a); a=fma(-a1,x1,a); b=fma(a0,x1,b); b=fma(a1,x0,b);} *re=a;*im=b; return; }
  if(TV==2){ double a=0,b=0; for(int k=k0;k<k1;k++){double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
     a=fma(-a1,x1,a); a=fma(a0,x0,a); b=fma(a1,x0,b); b=fma(a0,x1,b);} *re=a;*im=b; return; }
  if(TV==3){ double rr=0,ii=0,ri=0,ir=0; for(int k=k0;k<k1;k++){double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
    rr=fma(x0,a0,rr); ii=fma(x1,a1,ii); ri=fma(x1,a0,ri); ir=fma(x0,a1,ir);} *re=rr-ii; *im=ri+ir; return; }
  if(TV>=5){ int P=(TV-5)/2+2; int comb=(TV-5)%2; double rr[4]={0},ii[4]={0},ri[4]={0},ir[4]={0};
    for(int k=k0;k<k1;k++){int p=(k-k0)%P; double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
    rr[p]=fma(a0,x0,rr[p]); ii[p]=fma(a1,x1,ii[p]); ri[p]=fma(a0,x1,ri[p]); ir[p]=fma(a1,x0,ir[p]);}
    if(comb==0){ double Rr=0,Ii=0,Ri=0,Ir=0; for(int p=0;p<P;p++){Rr+=rr[p];Ii+=ii[p];Ri+=ri[p];Ir+=ir[p];} *re=Rr-Ii; *im=Ri+Ir; }
    else { double a=0,b=0; for(int p=0;p<P;p++){a+=rr[p]-ii[p]; b+=ri[p]+ir[p];} *re=a;*im=b; }
    return; }
  if(TV==4){ double rr=0,ii=0,ri=0,ir=0; for(int k=k0;k<k1;k++){double a0=A[2*(r+(size_t)k*n)],a1=A[2*(r+(size_t)k*n)+1],x0=x[2*k],x1=x[2*k+1];
    rr=fma(a0,x0,rr); ii=fma(a1,x1,ii); ri=fma(a0,x1,ri); ir=fma(a1,x0,ir);} *re=rr-ii; *im=ir+ri; return; }
}
__attribute__((target("avx2,fma"))) void fwd(int n,int nrhs,const double*L,double*X){
  for(int j=0;j<nrhs;j++){double*x=X+(size_t)2*j*n;
    int r0=0; int sizes[256],ns=0; int full=n/BS; for(int b=0;b<full;b++)sizes[ns++]=BS; for(int i=BS/2;i>0;i>>=1) if(n&i) sizes[ns++]=i;
    for(int b=0;b<ns;b++){int bs=sizes[b];
      if(r0>0) for(int r=r0;r<r0+bs;r++){double re,im; if(bs<BS) dot_t(L,n,r,x,0,r0,&re,&im); else dot4(L,n,r,x,0,r0,&re,&im); x[2*r]=x[2*r]-re; x[2*r+1]=x[2*r+1]-im;}
      for(int i=r0;i<r0+bs;i++){ double p0=x[2*i],p1=x[2*i+1]; mulinv(&p0,&p1,1.0,0.0); x[2*i]=p0;x[2*i+1]=p1; for(int k=i+1;k<r0+bs;k++) upd(&x[2*k],&x[2*k+1],p0,p1,L[2*(k+(size_t)i*n)],L[2*(k+(size_t)i*n)+1]); }
      r0+=bs; } } }
__attribute__((target("avx2,fma"))) void bwd(int n,int nrhs,const double*U,double*X){
  for(int j=0;j<nrhs;j++){double*x=X+(size_t)2*j*n;
    int starts[256],lens[256],nb=0;
    for(int i=1;i<BS;i*=2) if(n&i){ int s=(n&~(i-1))-i; starts[nb]=s; lens[nb]=i; nb++; }
    int full=n/BS; int s=(n&~(BS-1))-BS; for(int b=0;b<full;b++){starts[nb]=s;lens[nb]=BS;nb++; s-=BS;}
    for(int b=0;b<nb;b++){int r0=starts[b],bs=lens[b]; int kk=r0+bs;
      if(kk<n) for(int r=r0;r<r0+bs;r++){double re,im; if(bs<BS) dot_t(U,n,r,x,kk,n,&re,&im); else dot4(U,n,r,x,kk,n,&re,&im); x[2*r]-=re; x[2*r+1]-=im;}
      for(int i=r0+bs-1;i>=r0;i--){ double inv[2]; compinv(inv,U[2*(i+(size_t)i*n)],U[2*(i+(size_t)i*n)+1]); double p0=x[2*i],p1=x[2*i+1]; mulinv(&p0,&p1,inv[0],inv[1]); x[2*i]=p0;x[2*i+1]=p1; for(int k=r0;k<i;k++) upd(&x[2*k],&x[2*k+1],p0,p1,U[2*(k+(size_t)i*n)],U[2*(k+(size_t)i*n)+1]); }
    } } }
int main(int argc,char**argv){int n=argc>1?atoi(argv[1]):200,m=argc>2?atoi(argv[2]):200; size_t nn=(size_t)n*n;
 double*A=malloc(16*nn),*B=malloc(16*(size_t)n*m),*X1=malloc(16*(size_t)n*m),*X2=malloc(16*(size_t)n*m);
 for(size_t i=0;i<2*nn;i++)A[i]=rnd(); for(int i=0;i<n;i++)A[2*(i+(size_t)i*n)]+=n*0.1; for(size_t i=0;i<2*(size_t)n*m;i++)B[i]=rnd();
 double one[2]={1,0};
 BS=4;VAR=0;CV=1; for(TV=0;TV<9;TV++){ {
 memcpy(X1,B,16*n*m); memcpy(X2,B,16*n*m);
 cblas_ztrsm(102,141,122,111,132,n,m,one,A,n,X1,n); fwd(n,m,A,X2);
 int d=0; for(size_t i=0;i<2*(size_t)n*m;i++) d+=X1[i]!=X2[i];
 memcpy(X1,B,16*n*m); memcpy(X2,B,16*n*m);
 cblas_ztrsm(102,141,121,111,131,n,m,one,A,n,X1,n); bwd(n,m,A,X2);
 int d2=0; for(size_t i=0;i<2*(size_t)n*m;i++) d2+=X1[i]!=X2[i]; printf("TV=%d BS=%d VAR=%d n=%d fwd diffs=%d bwd diffs=%d\n",TV,BS,VAR,n,d,d2);}}}
