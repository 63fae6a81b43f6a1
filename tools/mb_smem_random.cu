// Shared-memory wavefronts per warp instruction for the walk's access patterns (random partner
// indices over ~1000 staged particles): LDS.32, LDS.64, LDS.128, ATOMS.ADD.
#include <cstdio>
__global__ void k(int *out, int mode, int iters, unsigned seed)
{
    __shared__ __align__(16) int buf[4 * 1088];
    for (int i = threadIdx.x; i < 4 * 1088; i += blockDim.x) buf[i] = i;
    __syncthreads();
    unsigned x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
    int acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const int j = (x >> 8) % 1088;
        if (mode == 0) acc += buf[j];                                                   // LDS.32
        else if (mode == 1) { const int2 v = reinterpret_cast<int2 *>(buf)[j]; acc += v.x + v.y; }   // LDS.64
        else if (mode == 2) { const int4 v = reinterpret_cast<int4 *>(buf)[j]; acc += v.x + v.w; }   // LDS.128
        else atomicAdd(&buf[j], 1);                                                     // ATOMS.ADD
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main()
{
    int *o;
    cudaMalloc(&o, 148 * 256 * sizeof(int));
    for (int m = 0; m <= 3; ++m) { k<<<148, 256>>>(o, m, 1000, 12345u); cudaDeviceSynchronize(); }
    printf("done\n");
    return 0;
}
