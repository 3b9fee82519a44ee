// exhaustive: __float2half_rn(f) vs both lanes of __floats2half2_rn for all 2^32 floats
#include <cuda_fp16.h>
#include <cstdio>
__global__ void k(unsigned long long *bad, unsigned *first)
{
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long b = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; b < (1ull << 32); b += stride) {
        const float f = __uint_as_float((unsigned)b);
        if (f != f) continue;
        const __half s = __float2half_rn(f);
        const __half2 p = __floats2half2_rn(f, f);
        const unsigned short us = __half_as_ushort(s), u0 = __half_as_ushort(__low2half(p)), u1 = __half_as_ushort(__high2half(p));
        if (us != u0 || us != u1) {
            if (atomicAdd(bad, 1ull) == 0) *first = (unsigned)b;
        }
    }
}
int main()
{
    unsigned long long *bad; unsigned *first;
    cudaMallocManaged(&bad, 8); cudaMallocManaged(&first, 4); *bad = 0; *first = 0;
    k<<<148 * 16, 256>>>(bad, first);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    printf("mismatching floats: %llu, first bits %08x\n", *bad, *first);
}
