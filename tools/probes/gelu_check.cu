#include <cstdio>
#include <cmath>
__device__ float g_new(float x){ const float k0 = 0.7978845608028654f, k1 = 0.044715f; const float u = k0 * fmaf(k1 * x * x, x, x); return __fdividef(x, 1.f + __expf(-2.f * u)); }
__device__ float g_old(float x){ const float k0 = 0.7978845608028654f, k1 = 0.044715f; return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x))); }
__global__ void k(float* e){ int i = blockIdx.x*blockDim.x+threadIdx.x; float x = -30.f + 60.f * i / (1<<20); float a=g_new(x), b=g_old(x); float d=fabsf(a-b); float r = d / fmaxf(fabsf(b), 1e-6f); atomicMax((int*)&e[0], __float_as_int(d)); if (fabsf(b)>1e-3f) atomicMax((int*)&e[1], __float_as_int(r)); }
int main(){ float* e; cudaMallocManaged(&e, 8); e[0]=0; e[1]=0; k<<<4096,256>>>(e); cudaDeviceSynchronize(); printf("max abs %g max rel %g\n", e[0], e[1]); }
