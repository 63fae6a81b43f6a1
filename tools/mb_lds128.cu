// LDS.128 wavefronts vs the number of distinct 16-byte addresses per warp and their lane layout.
#include <cstdio>
__global__ void k(float4 *out, int mode, int iters)
{
    __shared__ __align__(16) float4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int idx;
    switch (mode) {
    case 0: idx = 0; break;                         // all lanes one address
    case 1: idx = (lane >> 3) * 37; break;          // 4 addresses, one per quarter (8 consecutive lanes)
    case 2: idx = (lane & 3) * 37; break;           // 4 addresses interleaved (each quarter sees all 4)
    case 3: idx = (lane >> 2) * 37; break;          // 8 addresses, 4 consecutive lanes each
    case 4: idx = lane; break;                      // 32 consecutive float4
    case 5: idx = (lane * 97) & 1023; break;        // 32 scattered
    default: idx = (lane / 6) * 41; break;          // ~5-6 addresses in runs of 6 lanes (lockstep cells)
    }
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
        const float4 v = buf[(idx + it * 8) & 1023];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main()
{
    float4 *o;
    cudaMalloc(&o, 148 * 256 * sizeof(float4));
    for (int m = 0; m <= 6; ++m) {
        k<<<148, 256>>>(o, m, 1000);
        cudaDeviceSynchronize();
    }
    printf("done\n");
    return 0;
}
