
#include <cstdio>
#include <cuda_runtime.h>
__constant__ __align__(16) float cw[400];
__device__ __forceinline__ float2 sf_fma2(float2 a, float2 b, float2 c){ unsigned long long r; asm("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(r):"l"(*(unsigned long long*)&a),"l"(*(unsigned long long*)&b),"l"(*(unsigned long long*)&c)); return *(float2*)&r; }
template<int OFF> __device__ __forceinline__ float ldc(int it){ float v; asm("ld.const.f32 %0, [cw+%1];":"=f"(v):"n"(OFF),"r"(it)); return v; }
template<int OFF> __device__ __forceinline__ float2 ldc2(int it){ float2 v; asm("ld.const.v2.f32 {%0,%1}, [cw+%2];":"=f"(v.x),"=f"(v.y):"n"(OFF),"r"(it)); return v; }
__global__ void __launch_bounds__(128) kA(const float* __restrict__ xin, float* out, const float* __restrict__ w, int n){
  __shared__ __align__(16) float sw[400];
  for(int i=threadIdx.x;i<400;i+=128) sw[i]=w[i];
  __syncthreads();
  unsigned sp=(unsigned)__cvta_generic_to_shared(sw);
  int r=blockIdx.x*128+threadIdx.x; if(r>=n) return;
  float x[10]; for (int j=0;j<10;++j) x[j]=xin[r*10+j];
  #pragma unroll 1
  for (int it=0; it<40; ++it) {
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+0];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+16];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+32];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+48];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+64];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+80];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+96];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+112];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+128];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+144];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+160];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+176];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+192];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+208];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+224];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+240];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+256];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+272];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+288];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+304];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+320];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+336];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+352];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+368];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+384];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+400];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+416];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+432];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+448];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+464];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[4]);
   }
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+480];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+496];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+512];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+528];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+544];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+560];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+576];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+592];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+608];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+624];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+640];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+656];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+672];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+688];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+704];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+720];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+736];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+752];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+768];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+784];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+800];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+816];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+832];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+848];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+864];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+880];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+896];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+912];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+928];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+944];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[4]);
   }
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+960];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+976];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+992];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[0],x[0]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1008];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1024];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1040];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[1],x[1]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1056];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1072];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1088];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[2],x[2]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1104];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1120];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1136];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[3],x[3]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1152];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1168];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1184];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[4],x[4]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1200];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1216];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1232];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[5],x[5]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1248];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1264];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1280];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[6],x[6]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1296];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1312];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1328];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[7],x[7]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1344];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1360];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1376];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[8],x[8]), make_float2(w.x,w.y), y[4]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1392];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[0] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[0]);
     y[1] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[1]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1408];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[2] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[2]);
     y[3] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.z,w.w), y[3]);
   }
   { float4 w; asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+1424];" : "=f"(w.x),"=f"(w.y),"=f"(w.z),"=f"(w.w) : "r"(sp));
     y[4] = sf_fma2(make_float2(x[9],x[9]), make_float2(w.x,w.y), y[4]);
   }
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  }
  float t=0; for(int j=0;j<10;++j) t+=x[j]; out[r]=t;
}
__global__ void __launch_bounds__(128) kB(const float* __restrict__ xin, float* out, const float* __restrict__ w, int n){
  int r=blockIdx.x*128+threadIdx.x; if(r>=n) return;
  float x[10]; for (int j=0;j<10;++j) x[j]=xin[r*10+j];
  #pragma unroll 1
  for (int it=0; it<40; ++it) {
  { float y[10]; for(int c=0;c<10;++c) y[c]=0.f;
   y[0] = __fmaf_rn(x[0], ldc<0>(it), y[0]);
   y[1] = __fmaf_rn(x[0], ldc<4>(it), y[1]);
   y[2] = __fmaf_rn(x[0], ldc<8>(it), y[2]);
   y[3] = __fmaf_rn(x[0], ldc<12>(it), y[3]);
   y[4] = __fmaf_rn(x[0], ldc<16>(it), y[4]);
   y[5] = __fmaf_rn(x[0], ldc<20>(it), y[5]);
   y[6] = __fmaf_rn(x[0], ldc<24>(it), y[6]);
   y[7] = __fmaf_rn(x[0], ldc<28>(it), y[7]);
   y[8] = __fmaf_rn(x[0], ldc<32>(it), y[8]);
   y[9] = __fmaf_rn(x[0], ldc<36>(it), y[9]);
   y[0] = __fmaf_rn(x[1], ldc<48>(it), y[0]);
   y[1] = __fmaf_rn(x[1], ldc<52>(it), y[1]);
   y[2] = __fmaf_rn(x[1], ldc<56>(it), y[2]);
   y[3] = __fmaf_rn(x[1], ldc<60>(it), y[3]);
   y[4] = __fmaf_rn(x[1], ldc<64>(it), y[4]);
   y[5] = __fmaf_rn(x[1], ldc<68>(it), y[5]);
   y[6] = __fmaf_rn(x[1], ldc<72>(it), y[6]);
   y[7] = __fmaf_rn(x[1], ldc<76>(it), y[7]);
   y[8] = __fmaf_rn(x[1], ldc<80>(it), y[8]);
   y[9] = __fmaf_rn(x[1], ldc<84>(it), y[9]);
   y[0] = __fmaf_rn(x[2], ldc<96>(it), y[0]);
   y[1] = __fmaf_rn(x[2], ldc<100>(it), y[1]);
   y[2] = __fmaf_rn(x[2], ldc<104>(it), y[2]);
   y[3] = __fmaf_rn(x[2], ldc<108>(it), y[3]);
   y[4] = __fmaf_rn(x[2], ldc<112>(it), y[4]);
   y[5] = __fmaf_rn(x[2], ldc<116>(it), y[5]);
   y[6] = __fmaf_rn(x[2], ldc<120>(it), y[6]);
   y[7] = __fmaf_rn(x[2], ldc<124>(it), y[7]);
   y[8] = __fmaf_rn(x[2], ldc<128>(it), y[8]);
   y[9] = __fmaf_rn(x[2], ldc<132>(it), y[9]);
   y[0] = __fmaf_rn(x[3], ldc<144>(it), y[0]);
   y[1] = __fmaf_rn(x[3], ldc<148>(it), y[1]);
   y[2] = __fmaf_rn(x[3], ldc<152>(it), y[2]);
   y[3] = __fmaf_rn(x[3], ldc<156>(it), y[3]);
   y[4] = __fmaf_rn(x[3], ldc<160>(it), y[4]);
   y[5] = __fmaf_rn(x[3], ldc<164>(it), y[5]);
   y[6] = __fmaf_rn(x[3], ldc<168>(it), y[6]);
   y[7] = __fmaf_rn(x[3], ldc<172>(it), y[7]);
   y[8] = __fmaf_rn(x[3], ldc<176>(it), y[8]);
   y[9] = __fmaf_rn(x[3], ldc<180>(it), y[9]);
   y[0] = __fmaf_rn(x[4], ldc<192>(it), y[0]);
   y[1] = __fmaf_rn(x[4], ldc<196>(it), y[1]);
   y[2] = __fmaf_rn(x[4], ldc<200>(it), y[2]);
   y[3] = __fmaf_rn(x[4], ldc<204>(it), y[3]);
   y[4] = __fmaf_rn(x[4], ldc<208>(it), y[4]);
   y[5] = __fmaf_rn(x[4], ldc<212>(it), y[5]);
   y[6] = __fmaf_rn(x[4], ldc<216>(it), y[6]);
   y[7] = __fmaf_rn(x[4], ldc<220>(it), y[7]);
   y[8] = __fmaf_rn(x[4], ldc<224>(it), y[8]);
   y[9] = __fmaf_rn(x[4], ldc<228>(it), y[9]);
   y[0] = __fmaf_rn(x[5], ldc<240>(it), y[0]);
   y[1] = __fmaf_rn(x[5], ldc<244>(it), y[1]);
   y[2] = __fmaf_rn(x[5], ldc<248>(it), y[2]);
   y[3] = __fmaf_rn(x[5], ldc<252>(it), y[3]);
   y[4] = __fmaf_rn(x[5], ldc<256>(it), y[4]);
   y[5] = __fmaf_rn(x[5], ldc<260>(it), y[5]);
   y[6] = __fmaf_rn(x[5], ldc<264>(it), y[6]);
   y[7] = __fmaf_rn(x[5], ldc<268>(it), y[7]);
   y[8] = __fmaf_rn(x[5], ldc<272>(it), y[8]);
   y[9] = __fmaf_rn(x[5], ldc<276>(it), y[9]);
   y[0] = __fmaf_rn(x[6], ldc<288>(it), y[0]);
   y[1] = __fmaf_rn(x[6], ldc<292>(it), y[1]);
   y[2] = __fmaf_rn(x[6], ldc<296>(it), y[2]);
   y[3] = __fmaf_rn(x[6], ldc<300>(it), y[3]);
   y[4] = __fmaf_rn(x[6], ldc<304>(it), y[4]);
   y[5] = __fmaf_rn(x[6], ldc<308>(it), y[5]);
   y[6] = __fmaf_rn(x[6], ldc<312>(it), y[6]);
   y[7] = __fmaf_rn(x[6], ldc<316>(it), y[7]);
   y[8] = __fmaf_rn(x[6], ldc<320>(it), y[8]);
   y[9] = __fmaf_rn(x[6], ldc<324>(it), y[9]);
   y[0] = __fmaf_rn(x[7], ldc<336>(it), y[0]);
   y[1] = __fmaf_rn(x[7], ldc<340>(it), y[1]);
   y[2] = __fmaf_rn(x[7], ldc<344>(it), y[2]);
   y[3] = __fmaf_rn(x[7], ldc<348>(it), y[3]);
   y[4] = __fmaf_rn(x[7], ldc<352>(it), y[4]);
   y[5] = __fmaf_rn(x[7], ldc<356>(it), y[5]);
   y[6] = __fmaf_rn(x[7], ldc<360>(it), y[6]);
   y[7] = __fmaf_rn(x[7], ldc<364>(it), y[7]);
   y[8] = __fmaf_rn(x[7], ldc<368>(it), y[8]);
   y[9] = __fmaf_rn(x[7], ldc<372>(it), y[9]);
   y[0] = __fmaf_rn(x[8], ldc<384>(it), y[0]);
   y[1] = __fmaf_rn(x[8], ldc<388>(it), y[1]);
   y[2] = __fmaf_rn(x[8], ldc<392>(it), y[2]);
   y[3] = __fmaf_rn(x[8], ldc<396>(it), y[3]);
   y[4] = __fmaf_rn(x[8], ldc<400>(it), y[4]);
   y[5] = __fmaf_rn(x[8], ldc<404>(it), y[5]);
   y[6] = __fmaf_rn(x[8], ldc<408>(it), y[6]);
   y[7] = __fmaf_rn(x[8], ldc<412>(it), y[7]);
   y[8] = __fmaf_rn(x[8], ldc<416>(it), y[8]);
   y[9] = __fmaf_rn(x[8], ldc<420>(it), y[9]);
   y[0] = __fmaf_rn(x[9], ldc<432>(it), y[0]);
   y[1] = __fmaf_rn(x[9], ldc<436>(it), y[1]);
   y[2] = __fmaf_rn(x[9], ldc<440>(it), y[2]);
   y[3] = __fmaf_rn(x[9], ldc<444>(it), y[3]);
   y[4] = __fmaf_rn(x[9], ldc<448>(it), y[4]);
   y[5] = __fmaf_rn(x[9], ldc<452>(it), y[5]);
   y[6] = __fmaf_rn(x[9], ldc<456>(it), y[6]);
   y[7] = __fmaf_rn(x[9], ldc<460>(it), y[7]);
   y[8] = __fmaf_rn(x[9], ldc<464>(it), y[8]);
   y[9] = __fmaf_rn(x[9], ldc<468>(it), y[9]);
  for(int c=0;c<10;++c) x[c]=fmaxf(y[c],0.f); }
  { float y[10]; for(int c=0;c<10;++c) y[c]=0.f;
   y[0] = __fmaf_rn(x[0], ldc<480>(it), y[0]);
   y[1] = __fmaf_rn(x[0], ldc<484>(it), y[1]);
   y[2] = __fmaf_rn(x[0], ldc<488>(it), y[2]);
   y[3] = __fmaf_rn(x[0], ldc<492>(it), y[3]);
   y[4] = __fmaf_rn(x[0], ldc<496>(it), y[4]);
   y[5] = __fmaf_rn(x[0], ldc<500>(it), y[5]);
   y[6] = __fmaf_rn(x[0], ldc<504>(it), y[6]);
   y[7] = __fmaf_rn(x[0], ldc<508>(it), y[7]);
   y[8] = __fmaf_rn(x[0], ldc<512>(it), y[8]);
   y[9] = __fmaf_rn(x[0], ldc<516>(it), y[9]);
   y[0] = __fmaf_rn(x[1], ldc<528>(it), y[0]);
   y[1] = __fmaf_rn(x[1], ldc<532>(it), y[1]);
   y[2] = __fmaf_rn(x[1], ldc<536>(it), y[2]);
   y[3] = __fmaf_rn(x[1], ldc<540>(it), y[3]);
   y[4] = __fmaf_rn(x[1], ldc<544>(it), y[4]);
   y[5] = __fmaf_rn(x[1], ldc<548>(it), y[5]);
   y[6] = __fmaf_rn(x[1], ldc<552>(it), y[6]);
   y[7] = __fmaf_rn(x[1], ldc<556>(it), y[7]);
   y[8] = __fmaf_rn(x[1], ldc<560>(it), y[8]);
   y[9] = __fmaf_rn(x[1], ldc<564>(it), y[9]);
   y[0] = __fmaf_rn(x[2], ldc<576>(it), y[0]);
   y[1] = __fmaf_rn(x[2], ldc<580>(it), y[1]);
   y[2] = __fmaf_rn(x[2], ldc<584>(it), y[2]);
   y[3] = __fmaf_rn(x[2], ldc<588>(it), y[3]);
   y[4] = __fmaf_rn(x[2], ldc<592>(it), y[4]);
   y[5] = __fmaf_rn(x[2], ldc<596>(it), y[5]);
   y[6] = __fmaf_rn(x[2], ldc<600>(it), y[6]);
   y[7] = __fmaf_rn(x[2], ldc<604>(it), y[7]);
   y[8] = __fmaf_rn(x[2], ldc<608>(it), y[8]);
   y[9] = __fmaf_rn(x[2], ldc<612>(it), y[9]);
   y[0] = __fmaf_rn(x[3], ldc<624>(it), y[0]);
   y[1] = __fmaf_rn(x[3], ldc<628>(it), y[1]);
   y[2] = __fmaf_rn(x[3], ldc<632>(it), y[2]);
   y[3] = __fmaf_rn(x[3], ldc<636>(it), y[3]);
   y[4] = __fmaf_rn(x[3], ldc<640>(it), y[4]);
   y[5] = __fmaf_rn(x[3], ldc<644>(it), y[5]);
   y[6] = __fmaf_rn(x[3], ldc<648>(it), y[6]);
   y[7] = __fmaf_rn(x[3], ldc<652>(it), y[7]);
   y[8] = __fmaf_rn(x[3], ldc<656>(it), y[8]);
   y[9] = __fmaf_rn(x[3], ldc<660>(it), y[9]);
   y[0] = __fmaf_rn(x[4], ldc<672>(it), y[0]);
   y[1] = __fmaf_rn(x[4], ldc<676>(it), y[1]);
   y[2] = __fmaf_rn(x[4], ldc<680>(it), y[2]);
   y[3] = __fmaf_rn(x[4], ldc<684>(it), y[3]);
   y[4] = __fmaf_rn(x[4], ldc<688>(it), y[4]);
   y[5] = __fmaf_rn(x[4], ldc<692>(it), y[5]);
   y[6] = __fmaf_rn(x[4], ldc<696>(it), y[6]);
   y[7] = __fmaf_rn(x[4], ldc<700>(it), y[7]);
   y[8] = __fmaf_rn(x[4], ldc<704>(it), y[8]);
   y[9] = __fmaf_rn(x[4], ldc<708>(it), y[9]);
   y[0] = __fmaf_rn(x[5], ldc<720>(it), y[0]);
   y[1] = __fmaf_rn(x[5], ldc<724>(it), y[1]);
   y[2] = __fmaf_rn(x[5], ldc<728>(it), y[2]);
   y[3] = __fmaf_rn(x[5], ldc<732>(it), y[3]);
   y[4] = __fmaf_rn(x[5], ldc<736>(it), y[4]);
   y[5] = __fmaf_rn(x[5], ldc<740>(it), y[5]);
   y[6] = __fmaf_rn(x[5], ldc<744>(it), y[6]);
   y[7] = __fmaf_rn(x[5], ldc<748>(it), y[7]);
   y[8] = __fmaf_rn(x[5], ldc<752>(it), y[8]);
   y[9] = __fmaf_rn(x[5], ldc<756>(it), y[9]);
   y[0] = __fmaf_rn(x[6], ldc<768>(it), y[0]);
   y[1] = __fmaf_rn(x[6], ldc<772>(it), y[1]);
   y[2] = __fmaf_rn(x[6], ldc<776>(it), y[2]);
   y[3] = __fmaf_rn(x[6], ldc<780>(it), y[3]);
   y[4] = __fmaf_rn(x[6], ldc<784>(it), y[4]);
   y[5] = __fmaf_rn(x[6], ldc<788>(it), y[5]);
   y[6] = __fmaf_rn(x[6], ldc<792>(it), y[6]);
   y[7] = __fmaf_rn(x[6], ldc<796>(it), y[7]);
   y[8] = __fmaf_rn(x[6], ldc<800>(it), y[8]);
   y[9] = __fmaf_rn(x[6], ldc<804>(it), y[9]);
   y[0] = __fmaf_rn(x[7], ldc<816>(it), y[0]);
   y[1] = __fmaf_rn(x[7], ldc<820>(it), y[1]);
   y[2] = __fmaf_rn(x[7], ldc<824>(it), y[2]);
   y[3] = __fmaf_rn(x[7], ldc<828>(it), y[3]);
   y[4] = __fmaf_rn(x[7], ldc<832>(it), y[4]);
   y[5] = __fmaf_rn(x[7], ldc<836>(it), y[5]);
   y[6] = __fmaf_rn(x[7], ldc<840>(it), y[6]);
   y[7] = __fmaf_rn(x[7], ldc<844>(it), y[7]);
   y[8] = __fmaf_rn(x[7], ldc<848>(it), y[8]);
   y[9] = __fmaf_rn(x[7], ldc<852>(it), y[9]);
   y[0] = __fmaf_rn(x[8], ldc<864>(it), y[0]);
   y[1] = __fmaf_rn(x[8], ldc<868>(it), y[1]);
   y[2] = __fmaf_rn(x[8], ldc<872>(it), y[2]);
   y[3] = __fmaf_rn(x[8], ldc<876>(it), y[3]);
   y[4] = __fmaf_rn(x[8], ldc<880>(it), y[4]);
   y[5] = __fmaf_rn(x[8], ldc<884>(it), y[5]);
   y[6] = __fmaf_rn(x[8], ldc<888>(it), y[6]);
   y[7] = __fmaf_rn(x[8], ldc<892>(it), y[7]);
   y[8] = __fmaf_rn(x[8], ldc<896>(it), y[8]);
   y[9] = __fmaf_rn(x[8], ldc<900>(it), y[9]);
   y[0] = __fmaf_rn(x[9], ldc<912>(it), y[0]);
   y[1] = __fmaf_rn(x[9], ldc<916>(it), y[1]);
   y[2] = __fmaf_rn(x[9], ldc<920>(it), y[2]);
   y[3] = __fmaf_rn(x[9], ldc<924>(it), y[3]);
   y[4] = __fmaf_rn(x[9], ldc<928>(it), y[4]);
   y[5] = __fmaf_rn(x[9], ldc<932>(it), y[5]);
   y[6] = __fmaf_rn(x[9], ldc<936>(it), y[6]);
   y[7] = __fmaf_rn(x[9], ldc<940>(it), y[7]);
   y[8] = __fmaf_rn(x[9], ldc<944>(it), y[8]);
   y[9] = __fmaf_rn(x[9], ldc<948>(it), y[9]);
  for(int c=0;c<10;++c) x[c]=fmaxf(y[c],0.f); }
  { float y[10]; for(int c=0;c<10;++c) y[c]=0.f;
   y[0] = __fmaf_rn(x[0], ldc<960>(it), y[0]);
   y[1] = __fmaf_rn(x[0], ldc<964>(it), y[1]);
   y[2] = __fmaf_rn(x[0], ldc<968>(it), y[2]);
   y[3] = __fmaf_rn(x[0], ldc<972>(it), y[3]);
   y[4] = __fmaf_rn(x[0], ldc<976>(it), y[4]);
   y[5] = __fmaf_rn(x[0], ldc<980>(it), y[5]);
   y[6] = __fmaf_rn(x[0], ldc<984>(it), y[6]);
   y[7] = __fmaf_rn(x[0], ldc<988>(it), y[7]);
   y[8] = __fmaf_rn(x[0], ldc<992>(it), y[8]);
   y[9] = __fmaf_rn(x[0], ldc<996>(it), y[9]);
   y[0] = __fmaf_rn(x[1], ldc<1008>(it), y[0]);
   y[1] = __fmaf_rn(x[1], ldc<1012>(it), y[1]);
   y[2] = __fmaf_rn(x[1], ldc<1016>(it), y[2]);
   y[3] = __fmaf_rn(x[1], ldc<1020>(it), y[3]);
   y[4] = __fmaf_rn(x[1], ldc<1024>(it), y[4]);
   y[5] = __fmaf_rn(x[1], ldc<1028>(it), y[5]);
   y[6] = __fmaf_rn(x[1], ldc<1032>(it), y[6]);
   y[7] = __fmaf_rn(x[1], ldc<1036>(it), y[7]);
   y[8] = __fmaf_rn(x[1], ldc<1040>(it), y[8]);
   y[9] = __fmaf_rn(x[1], ldc<1044>(it), y[9]);
   y[0] = __fmaf_rn(x[2], ldc<1056>(it), y[0]);
   y[1] = __fmaf_rn(x[2], ldc<1060>(it), y[1]);
   y[2] = __fmaf_rn(x[2], ldc<1064>(it), y[2]);
   y[3] = __fmaf_rn(x[2], ldc<1068>(it), y[3]);
   y[4] = __fmaf_rn(x[2], ldc<1072>(it), y[4]);
   y[5] = __fmaf_rn(x[2], ldc<1076>(it), y[5]);
   y[6] = __fmaf_rn(x[2], ldc<1080>(it), y[6]);
   y[7] = __fmaf_rn(x[2], ldc<1084>(it), y[7]);
   y[8] = __fmaf_rn(x[2], ldc<1088>(it), y[8]);
   y[9] = __fmaf_rn(x[2], ldc<1092>(it), y[9]);
   y[0] = __fmaf_rn(x[3], ldc<1104>(it), y[0]);
   y[1] = __fmaf_rn(x[3], ldc<1108>(it), y[1]);
   y[2] = __fmaf_rn(x[3], ldc<1112>(it), y[2]);
   y[3] = __fmaf_rn(x[3], ldc<1116>(it), y[3]);
   y[4] = __fmaf_rn(x[3], ldc<1120>(it), y[4]);
   y[5] = __fmaf_rn(x[3], ldc<1124>(it), y[5]);
   y[6] = __fmaf_rn(x[3], ldc<1128>(it), y[6]);
   y[7] = __fmaf_rn(x[3], ldc<1132>(it), y[7]);
   y[8] = __fmaf_rn(x[3], ldc<1136>(it), y[8]);
   y[9] = __fmaf_rn(x[3], ldc<1140>(it), y[9]);
   y[0] = __fmaf_rn(x[4], ldc<1152>(it), y[0]);
   y[1] = __fmaf_rn(x[4], ldc<1156>(it), y[1]);
   y[2] = __fmaf_rn(x[4], ldc<1160>(it), y[2]);
   y[3] = __fmaf_rn(x[4], ldc<1164>(it), y[3]);
   y[4] = __fmaf_rn(x[4], ldc<1168>(it), y[4]);
   y[5] = __fmaf_rn(x[4], ldc<1172>(it), y[5]);
   y[6] = __fmaf_rn(x[4], ldc<1176>(it), y[6]);
   y[7] = __fmaf_rn(x[4], ldc<1180>(it), y[7]);
   y[8] = __fmaf_rn(x[4], ldc<1184>(it), y[8]);
   y[9] = __fmaf_rn(x[4], ldc<1188>(it), y[9]);
   y[0] = __fmaf_rn(x[5], ldc<1200>(it), y[0]);
   y[1] = __fmaf_rn(x[5], ldc<1204>(it), y[1]);
   y[2] = __fmaf_rn(x[5], ldc<1208>(it), y[2]);
   y[3] = __fmaf_rn(x[5], ldc<1212>(it), y[3]);
   y[4] = __fmaf_rn(x[5], ldc<1216>(it), y[4]);
   y[5] = __fmaf_rn(x[5], ldc<1220>(it), y[5]);
   y[6] = __fmaf_rn(x[5], ldc<1224>(it), y[6]);
   y[7] = __fmaf_rn(x[5], ldc<1228>(it), y[7]);
   y[8] = __fmaf_rn(x[5], ldc<1232>(it), y[8]);
   y[9] = __fmaf_rn(x[5], ldc<1236>(it), y[9]);
   y[0] = __fmaf_rn(x[6], ldc<1248>(it), y[0]);
   y[1] = __fmaf_rn(x[6], ldc<1252>(it), y[1]);
   y[2] = __fmaf_rn(x[6], ldc<1256>(it), y[2]);
   y[3] = __fmaf_rn(x[6], ldc<1260>(it), y[3]);
   y[4] = __fmaf_rn(x[6], ldc<1264>(it), y[4]);
   y[5] = __fmaf_rn(x[6], ldc<1268>(it), y[5]);
   y[6] = __fmaf_rn(x[6], ldc<1272>(it), y[6]);
   y[7] = __fmaf_rn(x[6], ldc<1276>(it), y[7]);
   y[8] = __fmaf_rn(x[6], ldc<1280>(it), y[8]);
   y[9] = __fmaf_rn(x[6], ldc<1284>(it), y[9]);
   y[0] = __fmaf_rn(x[7], ldc<1296>(it), y[0]);
   y[1] = __fmaf_rn(x[7], ldc<1300>(it), y[1]);
   y[2] = __fmaf_rn(x[7], ldc<1304>(it), y[2]);
   y[3] = __fmaf_rn(x[7], ldc<1308>(it), y[3]);
   y[4] = __fmaf_rn(x[7], ldc<1312>(it), y[4]);
   y[5] = __fmaf_rn(x[7], ldc<1316>(it), y[5]);
   y[6] = __fmaf_rn(x[7], ldc<1320>(it), y[6]);
   y[7] = __fmaf_rn(x[7], ldc<1324>(it), y[7]);
   y[8] = __fmaf_rn(x[7], ldc<1328>(it), y[8]);
   y[9] = __fmaf_rn(x[7], ldc<1332>(it), y[9]);
   y[0] = __fmaf_rn(x[8], ldc<1344>(it), y[0]);
   y[1] = __fmaf_rn(x[8], ldc<1348>(it), y[1]);
   y[2] = __fmaf_rn(x[8], ldc<1352>(it), y[2]);
   y[3] = __fmaf_rn(x[8], ldc<1356>(it), y[3]);
   y[4] = __fmaf_rn(x[8], ldc<1360>(it), y[4]);
   y[5] = __fmaf_rn(x[8], ldc<1364>(it), y[5]);
   y[6] = __fmaf_rn(x[8], ldc<1368>(it), y[6]);
   y[7] = __fmaf_rn(x[8], ldc<1372>(it), y[7]);
   y[8] = __fmaf_rn(x[8], ldc<1376>(it), y[8]);
   y[9] = __fmaf_rn(x[8], ldc<1380>(it), y[9]);
   y[0] = __fmaf_rn(x[9], ldc<1392>(it), y[0]);
   y[1] = __fmaf_rn(x[9], ldc<1396>(it), y[1]);
   y[2] = __fmaf_rn(x[9], ldc<1400>(it), y[2]);
   y[3] = __fmaf_rn(x[9], ldc<1404>(it), y[3]);
   y[4] = __fmaf_rn(x[9], ldc<1408>(it), y[4]);
   y[5] = __fmaf_rn(x[9], ldc<1412>(it), y[5]);
   y[6] = __fmaf_rn(x[9], ldc<1416>(it), y[6]);
   y[7] = __fmaf_rn(x[9], ldc<1420>(it), y[7]);
   y[8] = __fmaf_rn(x[9], ldc<1424>(it), y[8]);
   y[9] = __fmaf_rn(x[9], ldc<1428>(it), y[9]);
  for(int c=0;c<10;++c) x[c]=fmaxf(y[c],0.f); }
  }
  float t=0; for(int j=0;j<10;++j) t+=x[j]; out[r]=t;
}
__global__ void __launch_bounds__(128) kC(const float* __restrict__ xin, float* out, const float* __restrict__ w, int n){
  int r=blockIdx.x*128+threadIdx.x; if(r>=n) return;
  float x[10]; for (int j=0;j<10;++j) x[j]=xin[r*10+j];
  #pragma unroll 1
  for (int it=0; it<40; ++it) {
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   y[0] = sf_fma2(make_float2(x[0],x[0]), ldc2<0>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[0],x[0]), ldc2<8>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[0],x[0]), ldc2<16>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[0],x[0]), ldc2<24>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[0],x[0]), ldc2<32>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[1],x[1]), ldc2<48>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[1],x[1]), ldc2<56>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[1],x[1]), ldc2<64>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[1],x[1]), ldc2<72>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[1],x[1]), ldc2<80>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[2],x[2]), ldc2<96>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[2],x[2]), ldc2<104>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[2],x[2]), ldc2<112>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[2],x[2]), ldc2<120>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[2],x[2]), ldc2<128>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[3],x[3]), ldc2<144>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[3],x[3]), ldc2<152>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[3],x[3]), ldc2<160>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[3],x[3]), ldc2<168>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[3],x[3]), ldc2<176>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[4],x[4]), ldc2<192>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[4],x[4]), ldc2<200>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[4],x[4]), ldc2<208>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[4],x[4]), ldc2<216>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[4],x[4]), ldc2<224>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[5],x[5]), ldc2<240>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[5],x[5]), ldc2<248>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[5],x[5]), ldc2<256>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[5],x[5]), ldc2<264>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[5],x[5]), ldc2<272>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[6],x[6]), ldc2<288>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[6],x[6]), ldc2<296>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[6],x[6]), ldc2<304>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[6],x[6]), ldc2<312>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[6],x[6]), ldc2<320>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[7],x[7]), ldc2<336>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[7],x[7]), ldc2<344>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[7],x[7]), ldc2<352>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[7],x[7]), ldc2<360>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[7],x[7]), ldc2<368>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[8],x[8]), ldc2<384>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[8],x[8]), ldc2<392>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[8],x[8]), ldc2<400>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[8],x[8]), ldc2<408>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[8],x[8]), ldc2<416>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[9],x[9]), ldc2<432>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[9],x[9]), ldc2<440>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[9],x[9]), ldc2<448>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[9],x[9]), ldc2<456>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[9],x[9]), ldc2<464>(it), y[4]);
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   y[0] = sf_fma2(make_float2(x[0],x[0]), ldc2<480>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[0],x[0]), ldc2<488>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[0],x[0]), ldc2<496>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[0],x[0]), ldc2<504>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[0],x[0]), ldc2<512>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[1],x[1]), ldc2<528>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[1],x[1]), ldc2<536>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[1],x[1]), ldc2<544>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[1],x[1]), ldc2<552>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[1],x[1]), ldc2<560>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[2],x[2]), ldc2<576>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[2],x[2]), ldc2<584>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[2],x[2]), ldc2<592>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[2],x[2]), ldc2<600>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[2],x[2]), ldc2<608>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[3],x[3]), ldc2<624>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[3],x[3]), ldc2<632>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[3],x[3]), ldc2<640>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[3],x[3]), ldc2<648>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[3],x[3]), ldc2<656>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[4],x[4]), ldc2<672>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[4],x[4]), ldc2<680>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[4],x[4]), ldc2<688>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[4],x[4]), ldc2<696>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[4],x[4]), ldc2<704>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[5],x[5]), ldc2<720>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[5],x[5]), ldc2<728>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[5],x[5]), ldc2<736>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[5],x[5]), ldc2<744>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[5],x[5]), ldc2<752>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[6],x[6]), ldc2<768>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[6],x[6]), ldc2<776>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[6],x[6]), ldc2<784>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[6],x[6]), ldc2<792>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[6],x[6]), ldc2<800>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[7],x[7]), ldc2<816>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[7],x[7]), ldc2<824>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[7],x[7]), ldc2<832>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[7],x[7]), ldc2<840>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[7],x[7]), ldc2<848>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[8],x[8]), ldc2<864>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[8],x[8]), ldc2<872>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[8],x[8]), ldc2<880>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[8],x[8]), ldc2<888>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[8],x[8]), ldc2<896>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[9],x[9]), ldc2<912>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[9],x[9]), ldc2<920>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[9],x[9]), ldc2<928>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[9],x[9]), ldc2<936>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[9],x[9]), ldc2<944>(it), y[4]);
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  { float2 y[5]; for(int c=0;c<5;++c) y[c]=make_float2(0.f,0.f);
   y[0] = sf_fma2(make_float2(x[0],x[0]), ldc2<960>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[0],x[0]), ldc2<968>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[0],x[0]), ldc2<976>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[0],x[0]), ldc2<984>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[0],x[0]), ldc2<992>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[1],x[1]), ldc2<1008>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[1],x[1]), ldc2<1016>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[1],x[1]), ldc2<1024>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[1],x[1]), ldc2<1032>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[1],x[1]), ldc2<1040>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[2],x[2]), ldc2<1056>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[2],x[2]), ldc2<1064>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[2],x[2]), ldc2<1072>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[2],x[2]), ldc2<1080>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[2],x[2]), ldc2<1088>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[3],x[3]), ldc2<1104>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[3],x[3]), ldc2<1112>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[3],x[3]), ldc2<1120>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[3],x[3]), ldc2<1128>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[3],x[3]), ldc2<1136>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[4],x[4]), ldc2<1152>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[4],x[4]), ldc2<1160>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[4],x[4]), ldc2<1168>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[4],x[4]), ldc2<1176>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[4],x[4]), ldc2<1184>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[5],x[5]), ldc2<1200>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[5],x[5]), ldc2<1208>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[5],x[5]), ldc2<1216>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[5],x[5]), ldc2<1224>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[5],x[5]), ldc2<1232>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[6],x[6]), ldc2<1248>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[6],x[6]), ldc2<1256>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[6],x[6]), ldc2<1264>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[6],x[6]), ldc2<1272>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[6],x[6]), ldc2<1280>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[7],x[7]), ldc2<1296>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[7],x[7]), ldc2<1304>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[7],x[7]), ldc2<1312>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[7],x[7]), ldc2<1320>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[7],x[7]), ldc2<1328>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[8],x[8]), ldc2<1344>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[8],x[8]), ldc2<1352>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[8],x[8]), ldc2<1360>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[8],x[8]), ldc2<1368>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[8],x[8]), ldc2<1376>(it), y[4]);
   y[0] = sf_fma2(make_float2(x[9],x[9]), ldc2<1392>(it), y[0]);
   y[1] = sf_fma2(make_float2(x[9],x[9]), ldc2<1400>(it), y[1]);
   y[2] = sf_fma2(make_float2(x[9],x[9]), ldc2<1408>(it), y[2]);
   y[3] = sf_fma2(make_float2(x[9],x[9]), ldc2<1416>(it), y[3]);
   y[4] = sf_fma2(make_float2(x[9],x[9]), ldc2<1424>(it), y[4]);
  for(int c=0;c<5;++c){ x[2*c]=fmaxf(y[c].x,0.f); x[2*c+1]=fmaxf(y[c].y,0.f);} }
  }
  float t=0; for(int j=0;j<10;++j) t+=x[j]; out[r]=t;
}
int main(){
  int n=100000; float *x,*o,*w; cudaMalloc(&x,n*40); cudaMalloc(&o,n*4); cudaMalloc(&w,1600);
  float h[400]; for(int i=0;i<400;++i) h[i]=((i*37)%17-8)*0.05f; cudaMemcpy(w,h,1600,cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(cw,h,1600); cudaMemset(x,0,n*40);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  float* res[3]; 
  for(int v=0; v<3; ++v){ for(int rep=0; rep<2; ++rep){
    cudaEventRecord(a);
    for(int i=0;i<10;++i){ if(v==0) kA<<<(n+127)/128,128>>>(x,o,w,n); else if(v==1) kB<<<(n+127)/128,128>>>(x,o,w,n); else kC<<<(n+127)/128,128>>>(x,o,w,n);}
    cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b);
    if(rep) printf("variant %c: %.1f us/launch  (%.2f TFLOP/s)\n", "ABC"[v], ms*100, 2.0*3*100*40*n/(ms/10*1e-3)/1e12);
  }}
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
