// Packed-FP32 throughput probe: can FMUL2/FADD2 (f32x2) carry the exact (separately
// rounded) multiply-add at a higher rate than scalar FMUL+FADD?  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -o packed_probe packed_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

#define NA 8
#define NB 4
// Each variant: NA x NB accumulators (pairs for packed), operands a[NA], b[NB] varied per iteration.
extern "C" __global__ void v_scalar(const float* in, float* out, int iters) {
    float a[NA], b[NB], acc[NA][NB]; const float dl = in[200];
    for (int i = 0; i < NA; ++i) a[i] = in[threadIdx.x + i];
    for (int j = 0; j < NB; ++j) b[j] = in[threadIdx.x + 32 + j];
    for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) acc[i][j] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
#pragma unroll
        for (int i = 0; i < NA; ++i) a[i] = __fadd_rn(a[i], dl);
    }
    float s = 0.f;
    for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
extern "C" __global__ void v_ffma(const float* in, float* out, int iters) {
    float a[NA], b[NB], acc[NA][NB]; const float dl = in[200];
    for (int i = 0; i < NA; ++i) a[i] = in[threadIdx.x + i];
    for (int j = 0; j < NB; ++j) b[j] = in[threadIdx.x + 32 + j];
    for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) acc[i][j] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < NA; ++i) a[i] = __fadd_rn(a[i], dl);
    }
    float s = 0.f;
    for (int i = 0; i < NA; ++i) for (int j = 0; j < NB; ++j) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// packed: a pairs (a[2i], a[2i+1]) times (b[j], b[j]) -> acc pair
#define PACKED_BODY(STEP)                                                                   \
    u64 a[NA / 2], bb[NB], acc[NA / 2][NB], one, nz;                                       \
    const u64* in2 = (const u64*)in;                                                         \
    for (int i = 0; i < NA / 2; ++i) a[i] = in2[threadIdx.x + i];                            \
    for (int j = 0; j < NB; ++j) bb[j] = in2[threadIdx.x + 32 + j];                          \
    one = in2[100]; nz = in2[101]; const u64 d2 = in2[102];                                                           \
    for (int i = 0; i < NA / 2; ++i) for (int j = 0; j < NB; ++j) acc[i][j] = 0ull;          \
    for (int it = 0; it < iters; ++it) {                                                     \
        _Pragma("unroll") for (int i = 0; i < NA / 2; ++i)                                   \
        _Pragma("unroll") for (int j = 0; j < NB; ++j) { STEP; }                             \
        _Pragma("unroll") for (int i = 0; i < NA / 2; ++i) a[i] = add2(a[i], d2);    \
    }                                                                                        \
    u64 s = 0;                                                                               \
    for (int i = 0; i < NA / 2; ++i) for (int j = 0; j < NB; ++j) s ^= acc[i][j];            \
    ((u64*)out)[blockIdx.x * blockDim.x + threadIdx.x] = s;

extern "C" __global__ void v_ffma2(const float* in, float* out, int iters) { PACKED_BODY(acc[i][j] = fma2(a[i], bb[j], acc[i][j])) }
extern "C" __global__ void v_mul2add2(const float* in, float* out, int iters) { PACKED_BODY(acc[i][j] = add2(acc[i][j], mul2(a[i], bb[j]))) }
extern "C" __global__ void v_mul2fma1(const float* in, float* out, int iters) { PACKED_BODY(acc[i][j] = fma2(mul2(a[i], bb[j]), one, acc[i][j])) }
extern "C" __global__ void v_fmaz_add2(const float* in, float* out, int iters) { PACKED_BODY(acc[i][j] = add2(acc[i][j], fma2(a[i], bb[j], nz))) }

typedef void (*kfn)(const float*, float*, int);
int main() {
    float* in; float* out;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 8 * 256 * 8);
    float h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = 1.0f + i * 1e-6f;
    ((unsigned long long*)h)[100] = 0x3f8000003f800000ull;  // (1, 1)
    ((unsigned long long*)h)[101] = 0x8000000080000000ull;  // (-0, -0)
    ((unsigned long long*)h)[102] = 0x3400000034000000ull;  // small step
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    struct { const char* name; kfn f; } vs[] = {{"scalar FMUL+FADD", v_scalar}, {"scalar FFMA", v_ffma}, {"FFMA2", v_ffma2},
        {"mul2+add2", v_mul2add2}, {"mul2+fma2(p,1,acc)", v_mul2fma1}, {"fma2(a,b,-0)+add2", v_fmaz_add2}};
    const int iters = 4096, threads = 256;
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (auto& v : vs) {
        int bps; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v.f, threads, 0);
        int blocks = sms * bps;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        v.f<<<blocks, threads>>>(in, out, 64);
        cudaEventRecord(e0);
        v.f<<<blocks, threads>>>(in, out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double lane_madds = (double)blocks * threads * iters * NA * NB;
        printf("%-22s blocks/SM %d  %.3f ms  %.2f T madd/s (x2 = %.1f TF/s)  err=%s\n", v.name, bps, ms,
               lane_madds / ms / 1e9, 2 * lane_madds / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
