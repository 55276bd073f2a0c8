// Probe: does setmaxnreg redistribute registers between warpgroups on this device? (12 warps, 168 at launch;
// warps 8-11 drop to 40, warps 0-7 rise to 232.) Prints "ok" when all warps finish.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 1) k(int* out) {
    const int warp = threadIdx.x >> 5;
    if (warp >= 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        atomicAdd(out, 1);
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    atomicAdd(out + 1, 1);
}
int main() {
    int* d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    k<<<2, 384>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    int h[2];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s %d %d\n", cudaGetErrorString(e), h[0], h[1]);
    return 0;
}
