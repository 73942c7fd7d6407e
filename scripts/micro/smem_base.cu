#include <cstdio>
__global__ void k(unsigned *o) { extern __shared__ __align__(1024) unsigned char sm[]; if (threadIdx.x == 0) o[0] = (unsigned)__cvta_generic_to_shared(sm); }
int main() { unsigned *d, h; cudaMalloc(&d, 4); cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k<<<1, 32, 200000>>>(d); cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost); printf("dynamic smem base 0x%x\n", h); return 0; }
