// K3t -- tensor-core channel contraction on the B200's 5th-generation tensor
// cores (tcgen05.mma kind::f16, BF16 or FP16 operands, FP32 accumulation in
// TMEM).  The north-star's optional mode: NOT bitwise equal to the reference
// (operands are rounded to 16 bits and the tensor core fixes its own
// accumulation order), so it is reported separately with its own error
// statistics; the exact FP32 path (contract_template.cuh) is the default.
//
//   M_p[k][t] = sum_c U_p[c][k] * V_p[c][t]     (per Winograd point p)
//
// U and V are produced by the generated transforms directly as 16-bit operands
// in the canonical UMMA K-major no-swizzle layout (8x8 core matrices, 128 B
// each), blocked so that one (tile, 32-channel stage) operand is one
// contiguous 8 KB block.  One persistent CTA per SM walks 128x128 output
// tiles (p, k-block, t-block):
//   warp 0      producer: two cp.async.bulk (8 KB each) per stage into a
//               6-deep smem ring (mbarrier complete_tx)
//   warp 1      one elected thread issues tcgen05.mma (M=128, N=128, K=16) into
//               one of two 128-column TMEM accumulators; tcgen05.commit frees
//               the smem stage / publishes the finished accumulator
//   warps 2..   epilogue (4 x EPW warps): tcgen05.ld TMEM -> registers -> M (fp32) while the
//               next tile accumulates into the other TMEM buffer
#include <mutex>
#include <set>
#include <string>
#include <cstdlib>
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
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TC_WAIT_%=;\n}\n" ::"r"(su32(b)),
        "r"(parity)
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

// U and V arrive as 16-bit operands already in the canonical K-major
// no-swizzle UMMA layout (written by the generated transforms, see
// codegen.cpp gen_layer_source_tc): X16[p][rowblock][c/32][(c/8)%4][row/8][row%8][c%8],
// so a (tile, 32-channel stage) operand is one contiguous 8 KB block.
constexpr int kOpStage = TBK * TBM * 2;  // bytes of one operand stage (A or B)
constexpr int OSTAGES = 6;
// epilogue staging: per epilogue warp, 2 buffers of 32 rows x 32 fp32 columns with a
// 144-byte row pitch (16-byte aligned rows for the bulk copies; STS.128 at 4
// wavefronts per warp instead of 32-way bank conflicts at a 128-byte pitch)
constexpr int kStagePitch = 36;                                  // floats per staged row
constexpr int kStageBytes = 32 * kStagePitch * 4;                // one 32x32 block
// 4 EPW warps x (EPW == 4 ? 1 : 2) staging buffers
constexpr int epi_bytes(int epw) { return 4 * epw * (epw == 4 ? 1 : 2) * kStageBytes; }
constexpr int kEpiOffset = OSTAGES * 2 * kOpStage + 256;         // after operands + barriers

// EPW epilogue warps per TMEM lane quarter (64 + 128 EPW threads): the kernel is bound by draining
// the accumulators to M (C <= 512 is at most 16 stages of MMA work per 64 KB of output); with EPW
// warps a quarter's four 32-column chunks drain concurrently (measured: no gain over EPW = 1 once
// the store loop is unpredicated, see epi_warps below).
template <int EPW>
__global__ void __launch_bounds__(64 + 128 * EPW, 1) tc_contract_kernel(const unsigned short* __restrict__ U,
                                                             const unsigned short* __restrict__ V,
                                                             float* __restrict__ M, long long Kp, long long Tp,
                                                             long long Cp, int n_tiles, int fp16, int tc_epi_mode,
                                                             int K) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* ops = smem;                                   // [OSTAGES][A | B]
    u64* bars = reinterpret_cast<u64*>(ops + OSTAGES * 2 * kOpStage);
    u64* full = bars;                 // [OSTAGES] operands landed (complete_tx)
    u64* empty = full + OSTAGES;      // [OSTAGES] MMAs reading the stage done (tcgen05.commit)
    u64* acc_full = empty + OSTAGES;  // [2] accumulator buffer complete
    u64* acc_empty = acc_full + 2;    // [2] accumulator buffer drained (4 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (int)(Cp / TBK);
    const int n_tb = (int)(Tp / TBN), n_kb = (int)(Kp / TBM);

    if (tid == 0) {
        for (int s = 0; s < OSTAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            bar_init(&acc_full[s], 1);
            bar_init(&acc_empty[s], 4 * EPW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 2 x 128 fp32 columns x 128 lanes (double-buffered accumulator)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(256u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int g = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int tb = tile % n_tb, rest = tile / n_tb, kb = rest % n_kb;
                const long long p = rest / n_kb;
                const unsigned short* gU = U + (p * Kp + (long long)kb * TBM) * Cp;
                const unsigned short* gV = V + (p * Tp + (long long)tb * TBN) * Cp;
                for (int kt = 0; kt < nk; ++kt, ++g) {
                    const int s = g % OSTAGES;
                    if (g >= OSTAGES) bar_wait(&empty[s], (unsigned)(((g / OSTAGES) - 1) & 1));
                    unsigned char* dst = ops + s * 2 * kOpStage;
                    bar_expect(&full[s], (unsigned)(2 * kOpStage));
                    bulk_g2s(dst, gU + (long long)kt * TBK * TBM, kOpStage, &full[s]);
                    bulk_g2s(dst + kOpStage, gV + (long long)kt * TBK * TBN, kOpStage, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
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
                    const int s = g % OSTAGES;
                    bar_wait(&full[s], (unsigned)((g / OSTAGES) & 1));
                    tc_fence_after();
                    const unsigned a0 = su32(ops + s * 2 * kOpStage);
                    const unsigned b0 = a0 + kOpStage;
#pragma unroll
                    for (int ks = 0; ks < TBK / 16; ++ks) {
                        const u64 da = smem_desc(a0 + ks * 2 * LBO_A, LBO_A, 128);
                        const u64 db = smem_desc(b0 + ks * 2 * LBO_B, LBO_B, 128);
                        mma_f16(tacc, da, db, idesc, (kt | ks) ? 1u : 0u);
                    }
                    mma_commit(&empty[s]);  // stage s free once these MMAs finish
                }
                mma_commit(&acc_full[ab]);  // accumulator buffer ab complete
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue warps 2 .. 2 + 4 EPW
        // TMEM lane quarter (warp % 4) = rows k of this warp; the EPW warps of a quarter take the
        // 32-column chunks j = jh, jh + EPW, ...
        const int q4 = warp & 3, ew = warp - 2, jh = ew >> 2;
        constexpr int NB = EPW == 4 ? 1 : 2;  // staging buffers per warp
        int it = 0;
        unsigned eb = 0;  // staged blocks issued by this lane (buffer = eb & 1)
        const int epi = tc_epi_mode;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int tb = tile % n_tb, rest = tile / n_tb, kb = rest % n_kb;
            const long long p = rest / n_kb;
            const int ab = it & 1;
            bar_wait(&acc_full[ab], (unsigned)((it >> 1) & 1));
            tc_fence_after();
            // rows of this warp's quarter that are real filters: M's padded rows k >= K are never read
            // (K4 walks k < K), so they are not written either -- at K = 64 (VGG-16 layers 1-2, 6 GB of
            // M each at batch 256) that is half of the 128-row tile's store traffic
            const int live = K - (kb * TBM + q4 * 32);
            if (live <= 0) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&acc_empty[ab]);
                continue;
            }
            const long long krow = (long long)kb * TBM + q4 * 32 + lane;
            float* dst = M + (p * Kp + krow) * Tp + (long long)tb * TBN;
            // Each lane owns one row k: the 32 values of a tcgen05.ld go to its staged row
            // in smem, then one 128-byte cp.async.bulk per row writes a full line of M
            // (TMA engine) -- per-lane 16-byte global stores scattered over 32 rows
            // throttled the LSU (ncu: lg_throttle the top stall).
            float* stage = reinterpret_cast<float*>(smem + kEpiOffset) + (size_t)ew * NB * 32 * kStagePitch;
#pragma unroll 1
            for (int j = jh; j < TBN / 32; j += EPW) {
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
                if (epi == 0) {  // direct: lane-per-row 16-byte stores
                    if (lane < live) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<uint4*>(dst + j * 32 + q * 4) =
                                make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    }
                } else if (epi == 1) {  // staged row + one 128-byte bulk copy per lane
                    float* row = stage + ((eb & (NB - 1)) * 32 + lane) * kStagePitch;
                    if (NB == 2)
                        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<uint4*>(row + q * 4) =
                            make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (lane < live)
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst + j * 32),
                                     "r"((uint32_t)__cvta_generic_to_shared(row))
                                     : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                } else {  // staged, read back 4 rows x 128 B per instruction: full-line stores
                    float* blk = stage + (eb & (NB - 1)) * 32 * kStagePitch;
                    if (NB == 1) __syncwarp();  // the previous chunk's read-back is done
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<uint4*>(blk + lane * kStagePitch + q * 4) =
                            make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    __syncwarp();
                    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
                    float* gbase = M + (p * Kp + (long long)kb * TBM + q4 * 32) * Tp + (long long)tb * TBN + j * 32 + c4;
                    if (live >= 32) {  // warp-uniform: the unpredicated loop keeps its 8 loads ahead of its 8 stores
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int rr = i * 4 + rsub;
                            *reinterpret_cast<uint4*>(gbase + (long long)rr * Tp) =
                                *reinterpret_cast<const uint4*>(blk + rr * kStagePitch + c4);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int rr = i * 4 + rsub;
                            if (rr < live)
                                *reinterpret_cast<uint4*>(gbase + (long long)rr * Tp) =
                                    *reinterpret_cast<const uint4*>(blk + rr * kStagePitch + c4);
                        }
                    }
                }
                ++eb;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&acc_empty[ab]);
        }
        if (epi == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // M written before exit
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
    }
}

}  // namespace

namespace wino {

// epilogue store form (tuning key "tc_epi"): 0 direct per-lane stores, 1 per-row bulk
// copies, 2 (default) staged in smem and stored as full 128-byte lines
// epilogue warps per lane quarter: tuning key "tc_epw" (1, 2 or 4), default 1.  With the full-quarter
// store loop unpredicated, one warp per quarter keeps the store path full: VGG-16 stack K3t 7.17 ms
// against 7.26 / 7.36 ms with 2 / 4 warps, cfg2 17.4 vs 17.3 / 30.5 us, cfg3 39.1 vs 39.3 / 39.4 us.
// (While the loop was predicated per row, the K = 64 layers needed 4 warps: 2.38 -> 1.64 ms.)
static int epi_warps(long long, int) {
    static const int v = [] {
        const std::string e = tuning("tc_epw");
        const int x = e.empty() ? 0 : std::atoi(e.c_str());
        return (x == 1 || x == 2 || x == 4) ? x : 1;
    }();
    return v;
}

static int epi_mode() {
    static const int v = [] {
        const std::string e = tuning("tc_epi");
        const int x = e.empty() ? 2 : std::atoi(e.c_str());
        return (x >= 0 && x <= 2) ? x : 2;
    }();
    return v;
}

// cudaFuncSetAttribute is per device: opt in once for every device a process drives
int tc_contract_prepare_device(int dev) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> g(mu);
    if (done.count(dev)) return WINO_OK;
    cudaError_t e = cudaFuncSetAttribute(tc_contract_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kEpiOffset + epi_bytes(1));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc_contract_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kEpiOffset + epi_bytes(2));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc_contract_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kEpiOffset + epi_bytes(4));
    if (e != cudaSuccess) return fail(WINO_ECUDA, std::string("tc_contract: set smem: ") + cudaGetErrorString(e));
    done.insert(dev);
    return WINO_OK;
}

int tc_contract_launch(const void* U, const void* V, void* M, long long Kp, long long Tp, long long Cp, int P,
                       int fp16, int K, void* stream) {
    if (Kp % TBM || Tp % TBN || Cp % TBK) return fail(WINO_EINVAL, "tc_contract: layout not padded to 128/128/32");
    const long long tiles = (long long)P * (Kp / TBM) * (Tp / TBN);
    if (tiles > (1LL << 30)) return fail(WINO_EUNSUPPORTED, "tc_contract: too many tiles");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (int rc = tc_contract_prepare_device(dev)) return rc;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)(tiles < sms ? tiles : sms);
    const int epw = epi_warps(Kp, K);
    const size_t smem = (size_t)kEpiOffset + epi_bytes(epw);
    auto kern = epw == 1 ? tc_contract_kernel<1> : epw == 2 ? tc_contract_kernel<2> : tc_contract_kernel<4>;
    kern<<<grid, 64 + 128 * epw, smem, (cudaStream_t)stream>>>((const unsigned short*)U, (const unsigned short*)V,
                                                              (float*)M, Kp, Tp, Cp, (int)tiles, fp16, epi_mode(), K);
    return after_launch("tc_contract");
}

}  // namespace wino
