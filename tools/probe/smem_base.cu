// prints the shared-window address of a kernel's dynamic shared memory (no static smem)
#include <cstdio>
__global__ void k() {
    extern __shared__ float4 s[];
    if (threadIdx.x == 0) printf("dynamic smem base 0x%x\n", (unsigned)__cvta_generic_to_shared(s));
}
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k<<<2, 32, 70000>>>();
    cudaDeviceSynchronize();
    int r = 0;
    cudaDeviceGetAttribute(&r, cudaDevAttrReservedSharedMemoryPerBlock, 0);
    printf("reserved per block %d\n", r);
    return 0;
}
