// Microbenchmarks of the sm_100a instruction/atomic rates that shape the force kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_red_f32x4(float4* a, int n, int per) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned h = t * 2654435761u;
  for (int k = 0; k < per; ++k) { h = h * 1664525u + 1013904223u; atomicAdd(&a[h % n], make_float4(1.f, 2.f, 3.f, 0.f)); }
}
__global__ void k_red_f32x4_seq(float4* a, int n, int per) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < per; ++k) { int idx = (t + k * gridDim.x * blockDim.x) % n; atomicAdd(&a[idx], make_float4(1.f, 2.f, 3.f, 0.f)); }
}
__global__ void k_red_s32_seq(int* a, int n, int per) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < per; ++k) { int idx = (t + k * gridDim.x * blockDim.x) % n; atomicAdd(&a[idx], 3); }
}
__global__ void k_st_f32x4_seq(float4* a, int n, int per) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < per; ++k) { int idx = (t + k * gridDim.x * blockDim.x) % n; a[idx] = make_float4(1.f, 2.f, 3.f, (float)k); }
}
__global__ void k_atoms(int* out, int iters) {
  __shared__ int s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x;
  for (int k = 0; k < iters; ++k) { h = h * 1664525u + 1013904223u; atomicAdd(&s[(h >> 8) & 4095], 1); }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
__global__ void k_atoms_ctrl(int* out, int iters) {  // same address arithmetic, plain add to a register
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x; int acc = 0;
  for (int k = 0; k < iters; ++k) { h = h * 1664525u + 1013904223u; acc += (h >> 8) & 4095; }
  if (acc == 0x12345) out[blockIdx.x] = acc;
}
__global__ void k_mufu(float* out, int iters) {
  float a = threadIdx.x * 1e-3f + 1.0f, b = 1.1f, c = 0.3f, d = 0.7f;
  for (int k = 0; k < iters; ++k) { a = rsqrtf(a) + 1.0f; b = __log2f(b) + 1.5f; c = __cosf(c); asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(d)); d += 0.5f; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_i2f(float* out, int iters) {
  unsigned u = threadIdx.x; float acc = 0.f;
  for (int k = 0; k < iters; ++k) { acc += __uint2float_rn(u); u = u * 1664525u + 1013904223u; acc += __int2float_rn((int)u); u ^= 0x9e3779b9u; acc += __uint2float_rn(u ^ k); acc += __uint2float_rn(u + k);}
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_imadwide(unsigned* out, int iters) {
  unsigned c0 = threadIdx.x, c1 = 1, c2 = blockIdx.x, c3 = 7;
  for (int k = 0; k < iters; ++k) {
    unsigned hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    unsigned hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    c0 = hi1 ^ c1 ^ 0x1234u; c1 = lo1; c2 = hi0 ^ c3 ^ 0x777u; c3 = lo0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 ^ c1 ^ c2 ^ c3;
}
__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x, b = 1.0001f, c = 0.5f, d = 0.25f, e = 2.f, f = 3.f, g = 4.f, h = 5.f;
  for (int k = 0; k < iters; ++k) { a = a * b + c; d = d * b + c; e = e * b + c; f = f * b + c; g = g*b+c; h=h*b+c; c = c * b + d; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f + g + h + c;
}

__global__ void k_ffma2(float* out, int iters) {
  unsigned long long a = threadIdx.x, b = 0x3f8000003f800000ull, c = 0x3f0000003f000000ull, d = 1, e = 2, f = 3, g = 4, h = 5;
  for (int k = 0; k < iters; ++k) {
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(e) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(f) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(g) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(h) : "l"(b), "l"(c));
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(c) : "l"(b), "l"(d));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a ^ d ^ e ^ f ^ g ^ h ^ c);
}
__global__ void k_ffma_mix(float* out, int iters) {  // 4 FFMA + 4 LOP3 per iteration (two pipes)
  float a = threadIdx.x, b = 1.0001f, c = 0.5f, d = 0.25f; unsigned x = threadIdx.x, y = 7, z = 9, w = 11;
  for (int k = 0; k < iters; ++k) { a = a * b + c; d = d * b + c; c = c * b + a; b = b * d + a;
    x = x ^ y ^ k; y = y ^ z ^ x; z = z ^ w ^ y; w = w ^ x ^ z; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + c + b + (float)(x ^ y ^ z ^ w);
}
__global__ void k_lds(float* out, int iters) {
  __shared__ float4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float acc = 0.f; int j = threadIdx.x;
  for (int k = 0; k < iters; ++k) { float4 v = s[(j + k) & 2047]; acc += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int n = 2 * 1024 * 1024;
  float4* a; int* ai; int* o; float* of; unsigned* ou;
  CK(cudaMalloc(&a, n * sizeof(float4))); CK(cudaMalloc(&ai, n * sizeof(int)));
  CK(cudaMalloc(&o, 1 << 20)); CK(cudaMalloc(&of, 64 << 20)); CK(cudaMalloc(&ou, 64 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  const int grid = sms * 8, blk = 256, per = 16;
  const double nthr = (double)grid * blk;
#define TIME(label, launch, ops) \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); launch; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); \
  cudaEventElapsedTime(&ms, e0, e1); printf("%-34s %9.3f ms  %10.3f Gop/s  %8.3f op/clk/SM\n", label, ms, (ops) / ms / 1e6, (ops) / (ms * 1e-3) / (clk * 1e3) / sms);
  TIME("REDG.F32x4 random (op=float4)", (k_red_f32x4<<<grid, blk>>>(a, n, per)), nthr * per);
  TIME("REDG.F32x4 seq", (k_red_f32x4_seq<<<grid, blk>>>(a, n, per)), nthr * per);
  TIME("REDG.S32 seq", (k_red_s32_seq<<<grid, blk>>>(ai, n, per)), nthr * per);
  TIME("STG.128 seq", (k_st_f32x4_seq<<<grid, blk>>>(a, n, per)), nthr * per);
  const int it = 4096;
  TIME("ATOMS.ADD random 16KB (lane-op)", (k_atoms<<<grid, blk>>>(o, it)), nthr * it);
  TIME("  control (same arith, no atom)", (k_atoms_ctrl<<<grid, blk>>>(o, it)), nthr * it);
  TIME("MUFU x4 + 4 FADD (lane-op=MUFU)", (k_mufu<<<grid, blk>>>(of, it)), nthr * it * 4);
  TIME("I2F x4 (lane-op=I2F)", (k_i2f<<<grid, blk>>>(of, it)), nthr * it * 4);
  TIME("philox round: 2 mulwide (lane-op=round)", (k_imadwide<<<grid, blk>>>(ou, it)), nthr * it);
  TIME("FFMA x7 (lane-op=FFMA)", (k_ffma<<<grid, blk>>>(of, it)), nthr * it * 7);
  TIME("FFMA2 x7 (lane-op=FFMA2 instr)", (k_ffma2<<<grid, blk>>>(of, it)), nthr * it * 7);
  TIME("4 FFMA + 4 LOP3 (lane-op=instr)", (k_ffma_mix<<<grid, blk>>>(of, it)), nthr * it * 8);
  TIME("LDS.128 consecutive (lane-op=LDS)", (k_lds<<<grid, blk>>>(of, it)), nthr * it);
  return 0;
}
