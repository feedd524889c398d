#include <cstdio>
#include <cmath>
#include "../paper_1602_01376_b200/csrc/common.cuh"
__global__ void k(const double* x, double* y, double* z, int n) { int i = blockIdx.x*blockDim.x+threadIdx.x; if (i<n) { y[i]=ks::exp_neg(x[i]); z[i]=exp(x[i]); } }
int main(){ const int n=1<<22; double *x,*y,*z; cudaMallocManaged(&x,n*8); cudaMallocManaged(&y,n*8); cudaMallocManaged(&z,n*8);
 for(int i=0;i<n;++i){ double t=(double)i/n; x[i]= i<n/2 ? -t*2*40 : -t*760.0; }
 x[0]=-0.0; x[1]=-1e-300; x[2]=-745.1; x[3]=-708.5; x[4]=-720;
 k<<<n/256,256>>>(x,y,z,n); cudaDeviceSynchronize();
 double maxulp=0; int bad=0;
 for(int i=0;i<n;++i){ double ref=z[i]; double d=fabs(y[i]-ref); double ulp = ref>0? d/ (nextafter(ref,INFINITY)-ref) : d; if(ulp>maxulp)maxulp=ulp; if(ulp>2) bad++; }
 printf("max ulp vs CUDA exp %.2f  (>2ulp: %d)  exp(-0)=%g exp(-745.1)=%g/%g\n", maxulp, bad, y[0], y[2], z[2]); }
