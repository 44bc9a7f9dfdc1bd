// Channel-contraction kernel template (K3), JIT-compiled by NVRTC for sm_100a.
//
//   M_p[k][t] = sum_c U_p[c][k] * V_p[c][t]   for every Winograd point p < P
//
// which is the Hadamard product + channel reduction of the reference
// (engine.py:415 `u * v`, engine.py:252-278 `_reduce_linear/_reduce_pairwise`,
// engine.py:336-338 `channel_reduce`) batched over all (k, tile) pairs.
//
// The host prepends #defines:
//   WINO_DT       float | double
//   WINO_TM/TN    per-thread microtile (rows k / columns t), multiples of the
//                 16-byte vector width
//   WINO_THM/THN  consumer thread grid of the CTA; BM = THM*TM, BN = THN*TN
//   WINO_BK       channels per pipeline stage (multiple of 8)
//   WINO_KU       channels per unrolled inner loop (divides BK; multiple of 8 for pairwise)
//   WINO_STAGES   smem ring depth
//   WINO_SUM      0 exact-linear, 1 exact-pairwise, 2 ffma-linear, 3 ffma-pairwise
//   WINO_LEVELS   pairwise: slots of the chunk-level binary counter
//   WINO_MAXREG   register cap (0 = __launch_bounds__ only)
//   WINO_PACK     1: float only -- packed f32x2 arithmetic (two adjacent t columns per
//                 instruction: FFMA2/FADD2 issue once for 64 lanes of work)
//
// Summation order (exact modes, bitwise equal to the reference):
//   linear   : acc = -0; acc = acc + fl(u*v) for c = 0, 1, ...  (-0 + z = z exactly)
//   pairwise : the reference's halving tree == a binary counter over the
//              products in c order: aligned blocks of 8 are summed as a perfect
//              tree in registers, block sums are pushed into a counter whose
//              slot j holds a block of 2^j chunks; the final fold adds the
//              occupied slots from the smallest block upwards.
// Padded channels (c >= C) carry -0 products and leave every sum unchanged.
//
// Structure: persistent, warp-specialised CTAs.  Each CTA walks tiles
// blockIdx.x, blockIdx.x + gridDim.x, ...; its producer warp streams the
// stages of consecutive tiles through a WINO_STAGES-deep smem ring with
// cp.async.bulk (TMA bulk copies, SASS UBLKCP) -- U and V are stored blocked
// (U[p][k/BM][c][k%BM], V[p][t/BN][c][t%BN]) so a stage is one contiguous
// block per operand -- signalled by "full" mbarriers (complete_tx); the
// consumer warps release stages through "empty" mbarriers and write their
// register tiles of M while the producer already prefetches the next tile.
// No CTA-wide barrier after setup.

#ifndef WINO_KU
#define WINO_KU WINO_BK
#endif
#ifndef WINO_NOPROD
#define WINO_NOPROD 0  // 1: no producer warp; the last consumer warp to release a stage refills it
#endif
#ifndef WINO_PACK
#define WINO_PACK 0
#endif
#ifndef WINO_FUSE_P
// > 0: fused exact K3 + K4 (+ activation).  One CTA contracts all WINO_FUSE_P = alpha^2 points
// of a (filter block, tile block) pair, one after the other, and parks every finished
// accumulator in tensor memory: with the 32x32b access shape a thread reaches only its own
// TMEM lane, so its 512 / (warps per lane quarter) columns are a private scratchpad that holds
// its TM x TN microtile for every point, [pair][point]-major.  After the last point each thread
// reads back the alpha^2 point sums of one (filter, tile) pair with a single tcgen05.ld and runs
// the generated output transform (wino_fused_out, prepended by the host) -- M never exists in
// shared or global memory.  Needs alpha^2 <= 16 with the 4 x 4 microtile and 8 consumer warps
// (16 pairs x 16 points = 256 columns per thread).
#define WINO_FUSE_P 0
#endif
#ifndef WINO_WN
#define WINO_WN 0  // > 0: warp-tiled thread map, WINO_WN lanes along t x 32/WINO_WN lanes along k
#endif
#ifndef WINO_SLOTS_SMEM
#define WINO_SLOTS_SMEM 0  // pairwise: dynamic-counter slots in shared memory instead of registers
#endif
#ifndef WINO_DBUF
#define WINO_DBUF (WINO_SUM == 1 || WINO_SUM == 3)  // explicit fragment double buffer (pairwise)
#endif
#define DT WINO_DT
#define BM (WINO_THM * WINO_TM)
#define BN (WINO_THN * WINO_TN)
#define NTHR (WINO_THM * WINO_THN)
#define NCW (NTHR / 32)
#define VW (16 / (int)sizeof(DT))
#define GM (WINO_TM / VW)
#define GN (WINO_TN / VW)

typedef unsigned long long u64;

#if WINO_DT_IS_DOUBLE
#define XMUL(a, b) __dmul_rn((a), (b))
#define XADD(a, b) __dadd_rn((a), (b))
#define XFMA(a, b, c) __fma_rn((a), (b), (c))
typedef double2 vec_t;
#else
#define XMUL(a, b) __fmul_rn((a), (b))
#define XADD(a, b) __fadd_rn((a), (b))
#define XFMA(a, b, c) __fmaf_rn((a), (b), (c))
typedef float4 vec_t;
#endif

// Arithmetic on the accumulator unit.  Scalar: one DT per value.  Packed
// (WINO_PACK): one u64 = f32x2 pair of adjacent t columns; the k-side operand
// is broadcast into both halves.  The exact product is fma.rn.f32x2(a, b, -0):
// fl(a*b + (-0)) == fl(a*b) for every a, b (including the sign of exact zeros:
// +0 + -0 = +0, -0 + -0 = -0 under round-to-nearest).  The -0 pair arrives as a
// kernel parameter so ptxas cannot fold it into an FMUL2 that it would then fuse
// with the following FADD2 into an FFMA2 (verified on nvcc 12.9:
// mul.rn.f32x2 + add.rn.f32x2 -> FFMA2 even with -fmad=false).  The SASS gate
// (tests/test_abi.py) accepts FFMA2 in exact kernels only with a uniform addend.
#if WINO_PACK
#if WINO_DT_IS_DOUBLE
#error "WINO_PACK needs float"
#endif
typedef u64 acc_t;
#define NJ (WINO_TN / 2)
#define ACC_NEG0 0x8000000080000000ull
#define ACC_POS0 0ull
static __device__ __forceinline__ u64 p_fma(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
static __device__ __forceinline__ u64 p_add(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
static __device__ __forceinline__ u64 p_bcast(float a) {
    u64 r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
    return r;
}
#define AMUL(a, b) p_fma((a), (b), nz2)
#define AADD(a, b) p_add((a), (b))
#define AFMA(a, b, c) p_fma((a), (b), (c))
#else
typedef DT acc_t;
#define NJ WINO_TN
#define ACC_NEG0 ((DT)(-0.0))
#define ACC_POS0 ((DT)0)
#define AMUL(a, b) XMUL((a), (b))
#define AADD(a, b) XADD((a), (b))
#define AFMA(a, b, c) XFMA((a), (b), (c))
#endif

static __device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(u64* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
static __device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WINO_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WINO_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Producer-side wait: the producer is normally STAGES-1 stages ahead and waits
// most of the time; a polling loop there costs issue slots of the consumer
// warp sharing its SMSP.  try_wait with a suspend-time hint parks the thread
// in hardware until the phase completes (or the hint expires).
static __device__ __forceinline__ void mbar_wait_sleep(u64* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WINO_SLEEP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WINO_SLEEP_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

#if WINO_MAXREG > 0
#define WINO_REGS __maxnreg__(WINO_MAXREG)
#else
#define WINO_REGS __launch_bounds__(NTHR + (WINO_NOPROD ? 0 : 32))
#endif

#if WINO_FUSE_P
#define WINO_FUSE_PS 16  // TMEM columns per (filter, tile) pair: alpha^2 rounded up to an x16 load
static_assert(WINO_FUSE_P <= WINO_FUSE_PS && WINO_TM * WINO_TN * WINO_FUSE_PS * (NCW / 4) <= 512 && NCW % 4 == 0 &&
                  !WINO_DT_IS_DOUBLE && !WINO_NOPROD,
              "fused output: alpha^2 x microtile must fit the thread's TMEM columns");
static __device__ __forceinline__ void tmem_st1(unsigned taddr, unsigned v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
static __device__ __forceinline__ void tmem_ld16(unsigned taddr, unsigned* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
#endif

// (one textual kernel definition with textually balanced braces: the host wraps every kernel
// body in an #if by brace matching, wino_host.cu wrap_kernels)
#if WINO_FUSE_P
#define WINO_FUSE_PARAMS , float *__restrict__ Y, int K, int Ho, int Wo, int th, int tw, long long T, int omode
#else
#define WINO_FUSE_PARAMS
#endif
extern "C" __global__ void WINO_REGS wino_contract(const DT* __restrict__ U, const DT* __restrict__ V,
                                                  DT* __restrict__ M, long long Kp, long long Tp, long long Cp,
                                                  int n_tiles, u64 nz2 WINO_FUSE_PARAMS) {
#if WINO_FUSE_P
    __shared__ unsigned tmem_slot;
#endif
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DT* sU = reinterpret_cast<DT*>(smem_raw);      // [STAGES][BK][BM]
    DT* sV = sU + WINO_STAGES * WINO_BK * BM;      // [STAGES][BK][BN]
    u64* full = reinterpret_cast<u64*>(sV + WINO_STAGES * WINO_BK * BN);
    u64* empty = full + WINO_STAGES;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nk = (int)(Cp / WINO_BK);
    const int n_tb = (int)(Tp / BN), n_kb = (int)(Kp / BM);

#if WINO_NOPROD
    unsigned* cnt = reinterpret_cast<unsigned*>(empty);  // per-stage release counters
    auto issue = [&](int gg) {
        const int it = gg / nk, kt = gg - it * nk;
        const int tile = blockIdx.x + it * gridDim.x;
        if (tile >= n_tiles) return;
        const int tb = tile % n_tb;
        const int rest = tile / n_tb;
        const int kb = rest % n_kb;
        const long long p = rest / n_kb;
        const int s = gg % WINO_STAGES;
        const DT* gU = U + (p * Kp + (long long)kb * BM) * Cp + (long long)kt * WINO_BK * BM;
        const DT* gV = V + (p * Tp + (long long)tb * BN) * Cp + (long long)kt * WINO_BK * BN;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s], (unsigned)(WINO_BK * (BM + BN) * sizeof(DT)));
        bulk_g2s(sU + s * WINO_BK * BM, gU, WINO_BK * BM * sizeof(DT), &full[s]);
        bulk_g2s(sV + s * WINO_BK * BN, gV, WINO_BK * BN * sizeof(DT), &full[s]);
    };
#endif
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < WINO_STAGES; ++s) {
            mbar_init(&full[s], 1);
#if WINO_NOPROD
            cnt[2 * s] = 0;
#else
            mbar_init(&empty[s], NCW);
#endif
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#if WINO_NOPROD
        for (int gg = 0; gg < WINO_STAGES; ++gg) issue(gg);
#endif
    }
#if WINO_FUSE_P
    if (warp == 0) {  // all 512 TMEM columns: one CTA per SM
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#endif
    __syncthreads();
#if WINO_FUSE_P
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_slot;
#endif

    if (!WINO_NOPROD && warp == NCW) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            int g = 0;  // global stage counter across this CTA's tiles
#if WINO_FUSE_P
            // fused: a CTA takes whole (kb, tb) groups and walks their points in order
#pragma unroll 1
            for (int gi = blockIdx.x * WINO_FUSE_P; gi < n_tiles; gi += gridDim.x * WINO_FUSE_P)
#pragma unroll 1
            for (int tile = gi; tile < gi + WINO_FUSE_P; ++tile)
#else
#pragma unroll 1
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
#endif
            {
#if WINO_FUSE_P
                const long long p = tile % WINO_FUSE_P;
                const int grp = tile / WINO_FUSE_P;
                const int tb = grp % n_tb;
                const int kb = grp / n_tb;
#else
                const int tb = tile % n_tb;
                const int rest = tile / n_tb;
                const int kb = rest % n_kb;
                const long long p = rest / n_kb;
#endif
                const DT* gU = U + (p * Kp + (long long)kb * BM) * Cp;
                const DT* gV = V + (p * Tp + (long long)tb * BN) * Cp;
#pragma unroll 1
                for (int kt = 0; kt < nk; ++kt, ++g) {
                    const int s = g % WINO_STAGES;
                    if (g >= WINO_STAGES) {
                        mbar_wait_sleep(&empty[s], (unsigned)(((g / WINO_STAGES) - 1) & 1));
                        // the consumers' generic-proxy reads of this slot (released by their
                        // mbarrier arrives, acquired above) must be ordered before the
                        // async-proxy bulk-copy writes that refill it
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    mbar_expect_tx(&full[s], (unsigned)(WINO_BK * (BM + BN) * sizeof(DT)));
                    bulk_g2s(sU + s * WINO_BK * BM, gU + (long long)kt * WINO_BK * BM, WINO_BK * BM * sizeof(DT),
                             &full[s]);
                    bulk_g2s(sV + s * WINO_BK * BN, gV + (long long)kt * WINO_BK * BN, WINO_BK * BN * sizeof(DT),
                             &full[s]);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumer warps
#if WINO_WN
    static_assert(32 % WINO_WN == 0 && WINO_THN % WINO_WN == 0 && WINO_THM % (32 / WINO_WN) == 0,
                  "warp-tiled thread map: WINO_WN x 32/WINO_WN lanes must tile the thread grid");
    const int tn = (warp % (WINO_THN / WINO_WN)) * WINO_WN + lane % WINO_WN;
    const int tm = (warp / (WINO_THN / WINO_WN)) * (32 / WINO_WN) + lane / WINO_WN;
#else
    const int tn = tid % WINO_THN;
    const int tm = tid / WINO_THN;
#endif
    int g = 0;

#if WINO_FUSE_P
    const unsigned tcol0 = tmem + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)((warp >> 2) * (WINO_TM * WINO_TN * WINO_FUSE_PS));
#pragma unroll 1
    for (int gi = blockIdx.x * WINO_FUSE_P; gi < n_tiles; gi += gridDim.x * WINO_FUSE_P)
#endif
    {  // fused: one (filter block, tile block) group; otherwise a plain block
#if WINO_FUSE_P
    const int grp = gi / WINO_FUSE_P;
    const int tb = grp % n_tb;
    const int kb = grp / n_tb;
#pragma unroll 1
    for (int pp = 0; pp < WINO_FUSE_P; ++pp)
#else
#pragma unroll 1
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
#endif
    {
#if WINO_FUSE_P
        const long long p = pp;
#else
        const int tb = tile % n_tb;
        const int rest = tile / n_tb;
        const int kb = rest % n_kb;
        const long long p = rest / n_kb;
#endif

#if WINO_SUM == 0
        acc_t acc[WINO_TM][NJ];
#pragma unroll
        for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j] = ACC_NEG0;
#elif WINO_SUM == 2
        acc_t acc[WINO_TM][NJ];
#pragma unroll
        for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j] = ACC_POS0;
#else
        acc_t pa[WINO_TM][NJ];
#if WINO_SUM == 1
        acc_t pb[WINO_TM][NJ], pd[WINO_TM][NJ];
#endif
        // Z: static counter inside a stage (a stage = WINO_BK/8 chunks of 8 channels);
        // slot: dynamic counter over stages (slot j holds 2^j stages)
#define ZL (WINO_BK == 8 ? 1 : WINO_BK == 16 ? 1 : WINO_BK == 32 ? 2 : 3)
        static_assert(WINO_BK == 8 || WINO_BK == 16 || WINO_BK == 32 || WINO_BK == 64,
                      "pairwise stages: the in-stage counter covers 8, 16, 32 or 64 channels");
        acc_t zs[ZL][WINO_TM][NJ];
#if WINO_SLOTS_SMEM
        // dynamic-counter slots in shared memory (touched once per stage): thread-major
        // so a warp's access is 32 consecutive words; frees LEVELS * TM * NJ registers
        acc_t* const slot_s = reinterpret_cast<acc_t*>(empty + WINO_STAGES);
#define SLOT(L, i, j) slot_s[((L) * (WINO_TM * NJ) + (i) * NJ + (j)) * NTHR + tid]
#else
        acc_t slot[WINO_LEVELS][WINO_TM][NJ];
#define SLOT(L, i, j) slot[L][i][j]
#endif
#endif

#pragma unroll 1
        for (int kt = 0; kt < nk; ++kt, ++g) {
            const int s = g % WINO_STAGES;
            mbar_wait(&full[s], (unsigned)((g / WINO_STAGES) & 1));
            const DT* cu = sU + s * WINO_BK * BM;
            const DT* cv = sV + s * WINO_BK * BN;
#if WINO_SUM == 1 || WINO_SUM == 3
#pragma unroll
#else
#pragma unroll 1
#endif
            for (int kk0 = 0; kk0 < WINO_BK; kk0 += WINO_KU) {
                // register double buffer: fragments of k-step kk+1 are loaded
                // while k-step kk is multiplied
#if WINO_PACK
                u64 fa[2][WINO_TM], fb[2][NJ];
                auto load_frag = [&](int buf, int kk) {
#pragma unroll
                    for (int q = 0; q < GM; ++q) {
                        const float4 w4 = *reinterpret_cast<const float4*>(cu + kk * BM + q * (WINO_THM * VW) + tm * VW);
                        fa[buf][q * VW + 0] = p_bcast(w4.x);
                        fa[buf][q * VW + 1] = p_bcast(w4.y);
                        fa[buf][q * VW + 2] = p_bcast(w4.z);
                        fa[buf][q * VW + 3] = p_bcast(w4.w);
                    }
#pragma unroll
                    for (int q = 0; q < GN; ++q) {
                        const ulonglong2 w2 =
                            *reinterpret_cast<const ulonglong2*>(cv + kk * BN + q * (WINO_THN * VW) + tn * VW);
                        fb[buf][q * 2 + 0] = w2.x;
                        fb[buf][q * 2 + 1] = w2.y;
                    }
                };
#else
                DT fa[2][WINO_TM], fb[2][WINO_TN];
                auto load_frag = [&](int buf, int kk) {
#pragma unroll
                    for (int q = 0; q < GM; ++q) {
                        vec_t w4 = *reinterpret_cast<const vec_t*>(cu + kk * BM + q * (WINO_THM * VW) + tm * VW);
                        const DT* ww = reinterpret_cast<const DT*>(&w4);
#pragma unroll
                        for (int v = 0; v < VW; ++v) fa[buf][q * VW + v] = ww[v];
                    }
#pragma unroll
                    for (int q = 0; q < GN; ++q) {
                        vec_t w4 = *reinterpret_cast<const vec_t*>(cv + kk * BN + q * (WINO_THN * VW) + tn * VW);
                        const DT* ww = reinterpret_cast<const DT*>(&w4);
#pragma unroll
                        for (int v = 0; v < VW; ++v) fb[buf][q * VW + v] = ww[v];
                    }
                };
#endif
#if WINO_DBUF
                load_frag(0, kk0);
#endif
#pragma unroll
                for (int kk1 = 0; kk1 < WINO_KU; ++kk1) {
                    const int kk = kk0 + kk1;
#if WINO_DBUF
                    if (kk1 + 1 < WINO_KU) load_frag((kk1 + 1) & 1, kk + 1);
                    const auto* a = fa[kk1 & 1];
                    const auto* b = fb[kk1 & 1];
#else
                    load_frag(0, kk);
                    const auto* a = fa[0];
                    const auto* b = fb[0];
#endif
#if WINO_SUM == 0
#pragma unroll
                    for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j) acc[i][j] = AADD(acc[i][j], AMUL(a[i], b[j]));
#elif WINO_SUM == 2
#pragma unroll
                    for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j) acc[i][j] = AFMA(a[i], b[j], acc[i][j]);
#else
                    const int pos = kk1 & 7;  // compile-time after unrolling (WINO_KU % 8 == 0)
#pragma unroll
                    for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j) {
#if WINO_SUM == 1
                            const acc_t z = AMUL(a[i], b[j]);
                            if (pos == 0) pa[i][j] = z;
                            else if (pos == 1) pa[i][j] = AADD(pa[i][j], z);
                            else if (pos == 2) pb[i][j] = z;
                            else if (pos == 3) { pb[i][j] = AADD(pb[i][j], z); pa[i][j] = AADD(pa[i][j], pb[i][j]); }
                            else if (pos == 4) pb[i][j] = z;
                            else if (pos == 5) pb[i][j] = AADD(pb[i][j], z);
                            else if (pos == 6) pd[i][j] = z;
                            else { pd[i][j] = AADD(pd[i][j], z); pb[i][j] = AADD(pb[i][j], pd[i][j]); pa[i][j] = AADD(pa[i][j], pb[i][j]); }
#else
                            if (pos == 0) pa[i][j] = AMUL(a[i], b[j]);
                            else pa[i][j] = AFMA(a[i], b[j], pa[i][j]);
#endif
                        }
                    if (pos == 7) {
                        // chunk c of this stage is complete (c compile-time): static
                        // counter inside the stage, dynamic counter over stages
                        const int c = kk >> 3;
                        constexpr int NCH = WINO_BK / 8;
                        const int dc = __ffs(~c) - 1;  // trailing ones of c (constant-folded)
#pragma unroll
                        for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j) {
                                acc_t cy = pa[i][j];
#pragma unroll
                                for (int e = 0; e < ZL; ++e)
                                    if (e < dc) cy = AADD(zs[e][i][j], cy);
                                if (c != NCH - 1) {
#pragma unroll
                                    for (int e = 0; e < ZL; ++e)
                                        if (e == dc) zs[e][i][j] = cy;
                                } else {
                                    pa[i][j] = cy;  // the whole stage's block sum
                                }
                            }
                        if (c == NCH - 1) {
                            const int d = __ffs(~kt) - 1;  // trailing ones of the stage index
#pragma unroll
                            for (int L = 0; L < WINO_LEVELS; ++L) {
                                if (d == L) {
#pragma unroll
                                    for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                                        for (int j = 0; j < NJ; ++j) {
                                            acc_t cy = pa[i][j];
#pragma unroll
                                            for (int e = 0; e < L; ++e) cy = AADD(SLOT(e, i, j), cy);
                                            SLOT(L, i, j) = cy;
                                        }
                                }
                            }
                        }
                    }
#endif
                }
            }
            __syncwarp();
#if WINO_NOPROD
            if (lane == 0) {
                // the last warp to release stage s refills it with stage g + STAGES
                if (atomicAdd(&cnt[2 * s], 1u) == NCW - 1) {
                    cnt[2 * s] = 0;
                    issue(g + WINO_STAGES);
                }
            }
#else
            if (lane == 0) mbar_arrive(&empty[s]);
#endif
        }

#if WINO_SUM == 1 || WINO_SUM == 3
        // fold the occupied slots (set bits of the chunk count), smallest block first
        acc_t acc[WINO_TM][NJ];
        {
            const long long Q = Cp / WINO_BK;  // number of stages = counter pushes
            bool have = false;
#pragma unroll
            for (int L = 0; L < WINO_LEVELS; ++L) {
                if ((Q >> L) & 1) {
#pragma unroll
                    for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j)
                            acc[i][j] = have ? AADD(SLOT(L, i, j), acc[i][j]) : SLOT(L, i, j);
                    have = true;
                }
            }
        }
#endif

#if WINO_FUSE_P
        // park this point's microtile in the thread's TMEM columns, [pair][point]-major
        static_assert(GM == 1 && GN == 1, "fused output: one 16-byte vector per microtile side");
#pragma unroll
        for (int i = 0; i < WINO_TM; ++i)
#pragma unroll
            for (int jj = 0; jj < WINO_TN; ++jj) {
#if WINO_PACK
                float lo, hi;
                asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i][jj >> 1]));
                const float val = (jj & 1) ? hi : lo;
#else
                const float val = acc[i][jj];
#endif
                tmem_st1(tcol0 + (unsigned)((i * WINO_TN + jj) * WINO_FUSE_PS) + (unsigned)pp, __float_as_uint(val));
            }
#else
        DT* gM = M + (p * Kp + (long long)kb * BM) * Tp + (long long)tb * BN;
#pragma unroll
        for (int q = 0; q < GM; ++q)
#pragma unroll
            for (int v = 0; v < VW; ++v) {
                const int i = q * VW + v;
                const long long row = q * (WINO_THM * VW) + tm * VW + v;
#pragma unroll
                for (int h = 0; h < GN; ++h) {
                    vec_t w4;
                    DT* ww = reinterpret_cast<DT*>(&w4);
#if WINO_PACK
#pragma unroll
                    for (int u = 0; u < VW / 2; ++u) {
                        float lo, hi;
                        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i][h * 2 + u]));
                        ww[2 * u] = lo;
                        ww[2 * u + 1] = hi;
                    }
#else
#pragma unroll
                    for (int u = 0; u < VW; ++u) ww[u] = acc[i][h * VW + u];
#endif
                    *reinterpret_cast<vec_t*>(gM + row * Tp + h * (WINO_THN * VW) + tn * VW) = w4;
                }
            }
#endif
    }  // tiles (fused: points of the group)
#if WINO_FUSE_P
        // all points of this (filter block, tile block) are parked: output transform per pair
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll 1
        for (int q = 0; q < WINO_TM * WINO_TN; ++q) {
            unsigned mr[WINO_FUSE_PS];
            tmem_ld16(tcol0 + (unsigned)(q * WINO_FUSE_PS), mr);
            const int k = kb * BM + tm * VW + q / WINO_TN;
            const long long t = (long long)tb * BN + tn * VW + q % WINO_TN;
            if (k < K && t < T) wino_fused_out(mr, k, (int)t, Y, K, Ho, Wo, th, tw, omode);
        }
#endif
    }  // groups (fused)
#if WINO_FUSE_P
    // every consumer warp is done with tensor memory before warp 0 frees it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(NTHR) : "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
#endif
}
