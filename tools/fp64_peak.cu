// Microbenchmark: FP64 DFMA and DMMA peak throughput, plus HBM copy bandwidth, on one B200.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__global__ void dfma_k(double* out, int iters){
  double a0=threadIdx.x*1e-9, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  double b=1.0000001, c=1e-12;
  for(int i=0;i<iters;i++){
    a0=fma(a0,b,c);a1=fma(a1,b,c);a2=fma(a2,b,c);a3=fma(a3,b,c);
    a4=fma(a4,b,c);a5=fma(a5,b,c);a6=fma(a6,b,c);a7=fma(a7,b,c);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
__global__ void dmma_k(double* out, int iters){
  double acc[8][2]; for(int j=0;j<8;j++){acc[j][0]=0;acc[j][1]=0;}
  double x=threadIdx.x*1e-3, y=1.0+threadIdx.x*1e-4;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(x), "d"(y));
  }
  double s=0; for(int j=0;j<8;j++) s+=acc[j][0]+acc[j][1];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, sizeof(double)*sms*8*1024));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int blocks_per_sm : {2,4,8}){
    int iters=20000; int grid=sms*blocks_per_sm, thr=256;
    dfma_k<<<grid,thr>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_k<<<grid,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*8*iters*(double)grid*thr; printf("DFMA bps=%d: %.2f TFLOP/s\n",blocks_per_sm, fl/ms/1e9);
    dmma_k<<<grid,thr>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_k<<<grid,thr>>>(out,iters/4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=2.0*256*8*(iters/4)*(double)grid*(thr/32); printf("DMMA bps=%d: %.2f TFLOP/s\n",blocks_per_sm, fl/ms/1e9);
  }
  {  // sustained DMMA rate: back-to-back launches for ~4 s, rate over the last 2 s (the power-capped clock;
     // the denominator for a kernel timed inside a long step, like MEASURED_PEAKS.json's bf16_tflops_sustained)
    int grid=sms*8, thr=256, iters=20000;
    double per_launch=2.0*256*8*iters*(double)grid*(thr/32);
    cudaEvent_t t0,t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
    float total=0; int launches=0; double last_fl=0; float last_ms=0;
    while(total<4000.f){
      cudaEventRecord(t0); for(int r=0;r<10;r++) dmma_k<<<grid,thr>>>(out,iters); cudaEventRecord(t1); CK(cudaEventSynchronize(t1));
      float ms; cudaEventElapsedTime(&ms,t0,t1); total+=ms; launches+=10;
      if(total>2000.f){ last_fl+=10*per_launch; last_ms+=ms; }
    }
    printf("DMMA sustained (last %.0f ms of %.0f ms, %d launches): %.2f TFLOP/s\n", last_ms, total, launches, last_fl/last_ms/1e9);
  }
  size_t n=(size_t)1<<28; double2 *a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16));
  cudaMemset(a,0,n*16);
  for(int g: {sms*2, sms*4, sms*8}){
    float best=1e9; for(int r=0;r<5;r++){cudaEventRecord(e0); copy_k<<<g,512>>>(a,b,n); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("copy grid=%d: %.1f GB/s\n", g, 2.0*n*16/best/1e6);
  }
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0); printf("SMs %d L2 %d\n", sms, l2);
  return 0;
}
