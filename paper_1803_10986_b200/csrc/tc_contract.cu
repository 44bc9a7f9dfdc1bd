// K3t -- tensor-core channel contraction on the B200's 5th-generation tensor
// cores (tcgen05.mma kind::f16, BF16 or FP16 operands, FP32 accumulation in
// TMEM).  The north-star's optional mode: NOT bitwise equal to the reference
// (operands are rounded to 16 bits and the tensor core fixes its own
// accumulation order), so it is reported separately with its own error
// statistics; the exact FP32 path (contract_template.cuh) is the default.
//
//   M_p[k][t] = sum_c U_p[c][k] * V_p[c][t]     (per Winograd point p)
//
// One persistent CTA per SM walks 128x128 output tiles (p, k-block, t-block):
//   warp 4      producer: cp.async.bulk of the fp32 stage blocks of U and V
//               (32 channels x 128) into a 3-deep smem ring (mbarrier complete_tx)
//   warps 0-3   convert each fp32 stage to BF16/FP16 in the canonical UMMA
//               K-major no-swizzle layout (8x8 core matrices, 128 B each),
//               then fence.proxy.async so the tensor core sees them
//   warp 5      one elected thread issues tcgen05.mma (M=128, N=128, K=16) into
//               one of two 128-column TMEM accumulators and tcgen05.commit's
//               the completion to mbarriers (operand buffer free / tile done)
//   warps 6-9   epilogue: tcgen05.ld TMEM -> registers -> M (fp32) while the
//               next tile accumulates into the other TMEM buffer
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wino_internal.h"

namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3, THBUF = 2;
constexpr int kF32Stage = TBK * (TBM + TBN) * 4;  // bytes per fp32 stage
constexpr int kHStage = TBK * (TBM + TBN) * 2;    // bytes per 16-bit operand stage
constexpr int LBO_A = (TBM / 8) * 128;            // bytes between 8-channel (K) core-matrix chunks (A)
constexpr int LBO_B = (TBN / 8) * 128;            // (B); SBO (8-row MN groups) = 128 B

typedef unsigned long long u64;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(u64* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(u64* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(u64* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(u64* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra TC_WAIT_%=;\n}\n" ::"r"(su32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, u64* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}

// UMMA shared-memory descriptor, no swizzle ("interleave"), Blackwell version 1.
__device__ __forceinline__ u64 smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
    u64 d = 0;
    d |= (u64)((addr >> 4) & 0x3FFF);
    d |= (u64)((lbo >> 4) & 0x3FFF) << 16;
    d |= (u64)((sbo >> 4) & 0x3FFF) << 32;
    d |= (u64)1 << 46;  // descriptor version (sm100)
    return d;            // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
}

// instruction descriptor: D f32, A/B bf16 (fmt 1) or f16 (fmt 0), both K-major, M=128, N=128
__device__ __forceinline__ unsigned instr_desc(int fp16) {
    const unsigned fmt = fp16 ? 0u : 1u;
    return (1u << 4) | (fmt << 7) | (fmt << 10) | ((unsigned)(TBN >> 3) << 17) | ((unsigned)(TBM >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(unsigned tmem_d, u64 a, u64 b, unsigned idesc, unsigned accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(u64* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack2(float a, float b, int fp16) {
    if (fp16) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// fp32 stage [TBK][W] (row c, W contiguous) -> 16-bit canonical K-major
// no-swizzle core matrices (8 rows w x 8 channels c = 128 B): byte offset
// (c/8)*LBO + (w/8)*128 + (w%8)*16 + (c%8)*2.  Thread u reads the 8 channels
// of column w (consecutive threads -> consecutive w: conflict-free loads) and
// writes one 16-byte row (consecutive threads -> consecutive rows).
template <int W, int LBO>
__device__ __forceinline__ void convert_stage(const float* __restrict__ src, unsigned char* dst, int tid, int fp16) {
    constexpr int UNITS = W * (TBK / 8);
#pragma unroll
    for (int u = tid; u < UNITS; u += 128) {
        const int w = u % W, kc = u / W;
        const float* col = src + (kc * 8) * W + w;
        uint4 o;
        o.x = pack2(col[0 * W], col[1 * W], fp16);
        o.y = pack2(col[2 * W], col[3 * W], fp16);
        o.z = pack2(col[4 * W], col[5 * W], fp16);
        o.w = pack2(col[6 * W], col[7 * W], fp16);
        *reinterpret_cast<uint4*>(dst + kc * LBO + (w / 8) * 128 + (w % 8) * 16) = o;
    }
}

__global__ void __launch_bounds__(320, 1) tc_contract_kernel(const float* __restrict__ U, const float* __restrict__ V,
                                                             float* __restrict__ M, long long Kp, long long Tp,
                                                             long long Cp, int n_tiles, int fp16) {
    extern __shared__ __align__(1024) unsigned char smem[];
    float* f32 = reinterpret_cast<float*>(smem);                              // [TSTAGES][TBK][TBM + TBN]
    unsigned char* hbuf = smem + TSTAGES * kF32Stage;                         // [THBUF][A | B]
    u64* bars = reinterpret_cast<u64*>(hbuf + THBUF * kHStage);
    u64* f_full = bars;                  // [TSTAGES]
    u64* f_empty = f_full + TSTAGES;     // [TSTAGES]
    u64* h_full = f_empty + TSTAGES;     // [THBUF]
    u64* h_empty = h_full + THBUF;       // [THBUF]
    u64* acc_full = h_empty + THBUF;    // [2] TMEM accumulator buffers
    u64* acc_empty = acc_full + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (int)(Cp / TBK);
    const int n_tb = (int)(Tp / TBN), n_kb = (int)(Kp / TBM);

    if (tid == 0) {
        for (int s = 0; s < TSTAGES; ++s) {
            bar_init(&f_full[s], 1);
            bar_init(&f_empty[s], 4);
        }
        for (int s = 0; s < THBUF; ++s) {
            bar_init(&h_full[s], 4);
            bar_init(&h_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            bar_init(&acc_full[s], 1);
            bar_init(&acc_empty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM: 2 x 128 fp32 columns x 128 lanes (double-buffered accumulator)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(256u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int g = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int tb = tile % n_tb, rest = tile / n_tb, kb = rest % n_kb;
                const long long p = rest / n_kb;
                const float* gU = U + (p * Kp + (long long)kb * TBM) * Cp;
                const float* gV = V + (p * Tp + (long long)tb * TBN) * Cp;
                for (int kt = 0; kt < nk; ++kt, ++g) {
                    const int s = g % TSTAGES;
                    if (g >= TSTAGES) bar_wait(&f_empty[s], (unsigned)(((g / TSTAGES) - 1) & 1));
                    float* dst = f32 + (size_t)s * (kF32Stage / 4);
                    bar_expect(&f_full[s], (unsigned)kF32Stage);
                    bulk_g2s(dst, gU + (long long)kt * TBK * TBM, TBK * TBM * 4, &f_full[s]);
                    bulk_g2s(dst + TBK * TBM, gV + (long long)kt * TBK * TBN, TBK * TBN * 4, &f_full[s]);
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const unsigned idesc = instr_desc(fp16);
            int g = 0, it = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
                const int ab = it & 1;
                if (it >= 2) bar_wait(&acc_empty[ab], (unsigned)(((it >> 1) - 1) & 1));
                tc_fence_after();
                const unsigned tacc = tmem + (unsigned)(ab * TBN);
                for (int kt = 0; kt < nk; ++kt, ++g) {
                    const int h = g % THBUF;
                    bar_wait(&h_full[h], (unsigned)((g / THBUF) & 1));
                    tc_fence_after();
                    const unsigned a0 = su32(hbuf + h * kHStage);
                    const unsigned b0 = a0 + TBK * TBM * 2;
#pragma unroll
                    for (int ks = 0; ks < TBK / 16; ++ks) {
                        const u64 da = smem_desc(a0 + ks * 2 * LBO_A, LBO_A, 128);
                        const u64 db = smem_desc(b0 + ks * 2 * LBO_B, LBO_B, 128);
                        mma_f16(tacc, da, db, idesc, (kt | ks) ? 1u : 0u);
                    }
                    mma_commit(&h_empty[h]);  // operand buffer h free once these MMAs finish
                }
                mma_commit(&acc_full[ab]);  // accumulator buffer ab complete
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------------------ converters
        int g = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            for (int kt = 0; kt < nk; ++kt, ++g) {
                const int s = g % TSTAGES, h = g % THBUF;
                bar_wait(&f_full[s], (unsigned)((g / TSTAGES) & 1));
                if (g >= THBUF) bar_wait(&h_empty[h], (unsigned)(((g / THBUF) - 1) & 1));
                const float* src = f32 + (size_t)s * (kF32Stage / 4);
                unsigned char* dst = hbuf + h * kHStage;
                convert_stage<TBM, LBO_A>(src, dst, tid, fp16);
                convert_stage<TBN, LBO_B>(src + TBK * TBM, dst + TBK * TBM * 2, tid, fp16);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
                __syncwarp();
                if (lane == 0) {
                    bar_arrive(&h_full[h]);
                    bar_arrive(&f_empty[s]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue warps 6..9
        // TMEM lane quarter (warp % 4) = rows k of this warp
        const int q4 = warp & 3;
        int it = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int tb = tile % n_tb, rest = tile / n_tb, kb = rest % n_kb;
            const long long p = rest / n_kb;
            const int ab = it & 1;
            bar_wait(&acc_full[ab], (unsigned)((it >> 1) & 1));
            tc_fence_after();
            const long long krow = (long long)kb * TBM + q4 * 32 + lane;
            float* dst = M + (p * Kp + krow) * Tp + (long long)tb * TBN;
#pragma unroll 1
            for (int j = 0; j < TBN / 32; ++j) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * TBN + j * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    *reinterpret_cast<uint4*>(dst + j * 32 + q * 4) =
                        make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&acc_empty[ab]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
    }
}

}  // namespace

namespace wino {

int tc_contract_launch(const void* U, const void* V, void* M, long long Kp, long long Tp, long long Cp, int P,
                       int fp16, void* stream) {
    if (Kp % TBM || Tp % TBN || Cp % TBK) return fail(WINO_EINVAL, "tc_contract: layout not padded to 128/128/32");
    const long long tiles = (long long)P * (Kp / TBM) * (Tp / TBN);
    if (tiles > (1LL << 30)) return fail(WINO_EUNSUPPORTED, "tc_contract: too many tiles");
    const size_t smem = (size_t)TSTAGES * kF32Stage + (size_t)THBUF * kHStage + 256;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tc_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)(tiles < sms ? tiles : sms);
    tc_contract_kernel<<<grid, 320, smem, (cudaStream_t)stream>>>((const float*)U, (const float*)V, (float*)M, Kp,
                                                                 Tp, Cp, (int)tiles, fp16);
    return after_launch("tc_contract");
}

}  // namespace wino
