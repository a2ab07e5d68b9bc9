// Probe: cuFFT throughput for batch-outer vs batch-inner layouts (c2 sizes).
#include <cufft.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do{auto e=(x); if(e){printf("err %d line %d\n",(int)e,__LINE__); return 1;}}while(0)
float timeit(cufftHandle p, cufftComplex* d, int dir, int reps){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  for(int i=0;i<3;i++) cufftExecC2C(p,d,d,dir);
  cudaEventRecord(a);
  for(int i=0;i<reps;i++) cufftExecC2C(p,d,d,dir);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b); return ms/reps;
}
int main(){
  const int Y=2048,X=2048,B=32,T=1536,P=2048;
  size_t n = (size_t)Y*X*B;
  cufftComplex* d; CK(cudaMalloc(&d, n*sizeof(cufftComplex)));
  cudaMemset(d,0,n*sizeof(cufftComplex));
  double gb = n*8.0/1e9;
  { // batch outer 2D
    cufftHandle p; int nn[2]={Y,X}; size_t ws;
    CK(cufftCreate(&p)); CK(cufftMakePlanMany(p,2,nn,nullptr,1,Y*X,nullptr,1,Y*X,CUFFT_C2C,B,&ws));
    float ms=timeit(p,d,CUFFT_FORWARD,10); printf("2D [b][y][x] fwd: %.3f ms  (%.0f GB/s per R+W pass) ws=%zu\n",ms,2*gb/ms*1e3,ws);
    ms=timeit(p,d,CUFFT_INVERSE,10); printf("2D [b][y][x] inv: %.3f ms\n",ms);
    cufftDestroy(p);
  }
  { // batch inner 2D
    cufftHandle p; int nn[2]={Y,X}; size_t ws;
    CK(cufftCreate(&p)); CK(cufftMakePlanMany(p,2,nn,nn,B,1,nn,B,1,CUFFT_C2C,B,&ws));
    float ms=timeit(p,d,CUFFT_FORWARD,10); printf("2D [y][x][b] fwd: %.3f ms  (%.0f GB/s per R+W pass) ws=%zu\n",ms,2*gb/ms*1e3,ws);
    ms=timeit(p,d,CUFFT_INVERSE,10); printf("2D [y][x][b] inv: %.3f ms\n",ms);
    cufftDestroy(p);
  }
  size_t ns=(size_t)T*P*B; double gbs=ns*8.0/1e9;
  { // 1D batch outer [b][t][p]
    cufftHandle p; int nn[1]={P}; size_t ws;
    CK(cufftCreate(&p)); CK(cufftMakePlanMany(p,1,nn,nullptr,1,P,nullptr,1,P,CUFFT_C2C,T*B,&ws));
    float ms=timeit(p,d,CUFFT_FORWARD,10); printf("1D [b][t][p]: %.3f ms (%.0f GB/s R+W)\n",ms,2*gbs/ms*1e3);
    cufftDestroy(p);
  }
  { // 1D batch inner [p][t][b]
    cufftHandle p; int nn[1]={P}; size_t ws;
    CK(cufftCreate(&p)); CK(cufftMakePlanMany(p,1,nn,nn,T*B,1,nn,T*B,1,CUFFT_C2C,T*B,&ws));
    float ms=timeit(p,d,CUFFT_FORWARD,10); printf("1D [p][t][b]: %.3f ms (%.0f GB/s R+W)\n",ms,2*gbs/ms*1e3);
    cufftDestroy(p);
  }
  { // copy bandwidth reference
    cufftComplex* e; cudaMalloc(&e, n*sizeof(cufftComplex));
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaMemcpy(e,d,n*8,cudaMemcpyDeviceToDevice);
    cudaEventRecord(a); for(int i=0;i<10;i++) cudaMemcpy(e,d,n*8,cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); ms/=10; printf("memcpy d2d %.3f ms %.0f GB/s\n",ms,2*gb/ms*1e3);
  }
  { // double precision Z2Z inner layout
    cufftDoubleComplex* z; CK(cudaMalloc(&z, n*sizeof(cufftDoubleComplex))); cudaMemset(z,0,n*16);
    cufftHandle p; int nn[2]={Y,X}; size_t ws;
    CK(cufftCreate(&p)); CK(cufftMakePlanMany(p,2,nn,nn,B,1,nn,B,1,CUFFT_Z2Z,B,&ws));
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    cufftExecZ2Z(p,z,z,CUFFT_FORWARD); cudaEventRecord(a); for(int i=0;i<5;i++) cufftExecZ2Z(p,z,z,CUFFT_FORWARD); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); ms/=5; printf("Z2Z 2D [y][x][b]: %.3f ms\n",ms);
  }
  return 0;
}
