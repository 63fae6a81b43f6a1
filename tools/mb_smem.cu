// Shared-memory and integer-reduction rates on sm_100a that decide the force kernel's pair
// phase (round 2): shared integer atomics under different conflict patterns, LDS.128
// (distinct / broadcast / random), REDUX, SHFL.  Every kernel runs 8 warps x 8 blocks per SM
// and reports warp-instructions per clock per SM (clock64 inside the kernel, SM clock domain).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_smem mb_smem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NW = 4096;

// mode 0: lane-distinct banks (addr = lane + 32 k, rotating); 1: random in 4096 words;
// 2: pairs of lanes share an address; 3: 8 lanes per address; 4: all lanes one address
template <int MODE>
__global__ void k_atoms(long long *cyc, int *out, int iters)
{
    __shared__ int s[NW];
    for (int i = threadIdx.x; i < NW; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
    long long t0 = clock64();
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        int a;
        h = h * 1664525u + 1013904223u;
        if (MODE == 0) a = (lane + 32 * (k & 127) + threadIdx.x) & (NW - 1);
        else if (MODE == 1) a = (h >> 12) & (NW - 1);
        else if (MODE == 2) a = ((lane >> 1) + 32 * (k & 127) + (threadIdx.x >> 5) * 16) & (NW - 1);
        else if (MODE == 3) a = ((lane >> 3) + 32 * (k & 127) + (threadIdx.x >> 5) * 4) & (NW - 1);
        else a = (32 * (k & 127) + (threadIdx.x >> 5)) & (NW - 1);
        atomicAdd(&s[a], 1);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { out[blockIdx.x] = s[7]; cyc[blockIdx.x] = t1 - t0; }
}

// control: the same address arithmetic without the atomic
__global__ void k_ctrl(long long *cyc, int *out, int iters)
{
    unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
    int acc = 0;
    long long t0 = clock64();
#pragma unroll 4
    for (int k = 0; k < iters; ++k) { h = h * 1664525u + 1013904223u; acc += (h >> 12) & (NW - 1); }
    long long t1 = clock64();
    if (acc == 0x1234567) out[blockIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LDS.128: mode 0 distinct consecutive float4 per lane; 1 broadcast (one address per warp);
// 2 random float4 in 1024; 3 eight lanes per float4 (4 distinct)
template <int MODE>
__global__ void k_lds128(long long *cyc, float *out, int iters)
{
    __shared__ float4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, 1, 2, 3);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
    float acc = 0.f;
    long long t0 = clock64();
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        int a;
        h = h * 1664525u + 1013904223u;
        if (MODE == 0) a = (lane + 32 * (k & 31)) & 1023;
        else if (MODE == 1) a = (k * 5 + (threadIdx.x >> 5)) & 1023;
        else if (MODE == 2) a = (h >> 12) & 1023;
        else a = ((lane >> 3) + 4 * (k & 255)) & 1023;
        const float4 v = s[a];
        acc += v.x + v.y + v.z + v.w;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// REDUX.SUM (warp integer sum), three per iteration
__global__ void k_redux(long long *cyc, int *out, int iters)
{
    int a = threadIdx.x, b = threadIdx.x * 3, c = threadIdx.x ^ 5, acc = 0;
    long long t0 = clock64();
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        acc += __reduce_add_sync(0xffffffffu, a) + __reduce_add_sync(0xffffffffu, b) +
               __reduce_add_sync(0xffffffffu, c);
        a += k; b ^= k; c += 3;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// SHFL.IDX, three per iteration
__global__ void k_shfl(long long *cyc, float *out, int iters)
{
    float a = threadIdx.x, b = threadIdx.x * 3, c = threadIdx.x * 0.5f;
    long long t0 = clock64();
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        a += __shfl_xor_sync(0xffffffffu, b, 1);
        b += __shfl_xor_sync(0xffffffffu, c, 2);
        c += __shfl_xor_sync(0xffffffffu, a, 4);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int bps = 8, blk = 256, grid = sms * bps, it = 8192;
    long long *cyc, hc[4096];
    int *oi;
    float *of;
    CK(cudaMalloc(&cyc, grid * sizeof(long long)));
    CK(cudaMalloc(&oi, grid * blk * sizeof(int)));
    CK(cudaMalloc(&of, grid * blk * sizeof(float)));
    const double warps_per_sm = bps * blk / 32.0;
    // rate = (warps per SM x ops per warp) / mean block cycles  [warp-instr per clock per SM]
#define RUN(label, launch, opsperit)                                                              \
    launch; CK(cudaDeviceSynchronize()); launch; CK(cudaDeviceSynchronize());                    \
    CK(cudaMemcpy(hc, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));                   \
    { double m = 0; for (int b = 0; b < grid; ++b) m += hc[b]; m /= grid;                          \
      printf("%-44s %8.3f warp-op/clk/SM  (%6.2f clk per warp-op per SMSP)\n", label,             \
             warps_per_sm * it * (opsperit) / m, m / (warps_per_sm / 4 * it * (opsperit))); }
    RUN("ATOMS.ADD lane-distinct banks", (k_atoms<0><<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("ATOMS.ADD random in 4096 words", (k_atoms<1><<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("ATOMS.ADD 2 lanes per address", (k_atoms<2><<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("ATOMS.ADD 8 lanes per address", (k_atoms<3><<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("ATOMS.ADD 32 lanes one address", (k_atoms<4><<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("control (address arithmetic only)", (k_ctrl<<<grid, blk>>>(cyc, oi, it)), 1);
    RUN("LDS.128 lane-distinct consecutive", (k_lds128<0><<<grid, blk>>>(cyc, of, it)), 1);
    RUN("LDS.128 broadcast", (k_lds128<1><<<grid, blk>>>(cyc, of, it)), 1);
    RUN("LDS.128 random in 1024 float4", (k_lds128<2><<<grid, blk>>>(cyc, of, it)), 1);
    RUN("LDS.128 8 lanes per float4", (k_lds128<3><<<grid, blk>>>(cyc, of, it)), 1);
    RUN("REDUX.SUM (3 per it)", (k_redux<<<grid, blk>>>(cyc, oi, it)), 3);
    RUN("SHFL.BFLY (3 per it)", (k_shfl<<<grid, blk>>>(cyc, of, it)), 3);
    return 0;
}
