/*
 * wino.h -- C-ABI of the B200-native Winograd / Toom-Cook convolution library
 * (libwino.so, built from paper_1803_10986_b200/csrc/).
 *
 * The reference (arxiv 1803.10986 toolkit, package `toomcook`) is pure
 * Python/numpy: its "plugin interface" is the Python API re-exported by
 * toomcook/__init__.py:4-27.  Each entry point below replaces one piece of
 * that API's arithmetic; the reference function it stands in for is cited on
 * each declaration.  The Python package paper_1803_10986_b200 binds these with
 * ctypes (INTEGRATION.md shows the binding a reference maintainer would add).
 *
 * Conventions
 *   - plain pointers + sizes; every device buffer is caller-owned;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *     calls are stream-ordered and never synchronise the host;
 *   - return 0 on success, a negative WINO_E* code on failure; the message is
 *     kept per thread and read with wino_last_error();
 *   - element types: precision FP32 -> inputs f32, transforms f32, Hadamard /
 *     channel sum f32, output f32; MIXED -> inputs f32 widened to f64 for the
 *     transforms, U and V narrowed (round-to-nearest) to f32, Hadamard and
 *     channel sum f32, output transform f64, output f64; FP64 -> f64 throughout
 *     (reference engine.py:27-55, 356-360, 401-423).
 */
#ifndef WINO_H
#define WINO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WINO_OK 0
#define WINO_EINVAL (-1)        /* bad argument / shape  -> Python ValueError   */
#define WINO_EUNSUPPORTED (-2)  /* size outside the generated kernels' range   */
#define WINO_ECUDA (-3)         /* CUDA runtime/driver error -> RuntimeError     */
#define WINO_ECOMPILE (-4)      /* NVRTC failed on generated source              */

/* ConvConfig enums (reference engine.py:22-24) */
#define WINO_FP32 0
#define WINO_FP64 1
#define WINO_MIXED 2
#define WINO_SUM_LINEAR 0
#define WINO_SUM_PAIRWISE 1
/* contraction arithmetic: EXACT = one rounded multiply and one rounded add per
 * channel term (bitwise equal to the reference); FFMA = fused multiply-add
 * (faster, NOT bitwise, reported with its own error statistics). */
#define WINO_CONTRACT_EXACT 0
#define WINO_CONTRACT_FFMA 1
/* tensor-core modes (tcgen05.mma kind::f16): U and V rounded to BF16 / FP16,
 * FP32 accumulation in TMEM -- NOT bitwise, reported with their own error;
 * precision must be fp32 or mixed. */
#define WINO_CONTRACT_TC_BF16 2
#define WINO_CONTRACT_TC_FP16 3
/* fused tensor-core modes: the same BF16 / FP16 products, but the contraction
 * and the output transform run as one kernel (wino_contract_output): all
 * alpha^2 accumulators of a (128 tiles x NK filters) block sit in TMEM and the
 * epilogue writes y directly -- M never exists.  Needs alpha^2 <= 32. */
#define WINO_CONTRACT_TCF_BF16 4
#define WINO_CONTRACT_TCF_FP16 5

/* One postfix op of a row program (reference engine.py:153-208 compiled
 * programs, flattened): LEAF pushes coeff * in[col] (one rounded product;
 * coeff = +1 / -1 are applied exactly without a multiply), ADD pops b, a and
 * pushes a + b (one rounded sum). An empty row evaluates to +0. */
#define WINO_OP_LEAF 0
#define WINO_OP_ADD 1
typedef struct {
    int32_t kind;
    int32_t col;
    double coeff; /* already rounded to the plan's coefficient table */
} wino_op;

typedef struct {
    int32_t rows;             /* matrix rows = number of programs              */
    int32_t cols;             /* matrix columns = input length                 */
    const int32_t* row_start; /* rows + 1 offsets into ops                     */
    const wino_op* ops;
} wino_prog;

typedef struct wino_plan wino_plan;

/* Layer geometry: x[N][C][H][W], w[K][C][r][r], stride 1, zero padding `pad`,
 * y[N][K][Ho][Wo] with Ho = H + 2 pad - r + 1 (Wo likewise). */
typedef struct {
    int32_t N, C, H, W, K, pad;
} wino_layer_shape;

/* Device layout of the Winograd-domain tensors for one layer (HBM):
 *   U [P][Kp/bm][Cp][bm]  filter transform, blocked by the contraction's
 *                         k-tile (P = alpha^2)
 *   V [P][Tp/bn][Cp][bn]  input-tile transform, blocked by the t-tile
 *                         (T = N * th * tw tiles, t = (n, i, j))
 *   M [P][Kp][Tp]         channel contraction
 * so one pipeline stage of a contraction tile is one contiguous block.
 * Cp/Kp/Tp are padded to the contraction kernel's tile sizes; padded channels
 * hold +0 (U) and -0 (V) so their products are -0 and leave every sum
 * bit-identical.  M's padded rows (k >= K) and columns (t >= T) are scratch:
 * the output transform never reads them and the tensor-core contraction
 * leaves the padded rows unwritten. */
typedef struct {
    int32_t P, th, tw, Ho, Wo;
    int32_t bm, bn; /* U / V block widths */
    int64_t T, Tp, Cp, Kp;
    int32_t elem_bytes_uv;  /* 4 (fp32, mixed) or 8 (fp64) */
    int32_t elem_bytes_y;   /* 4 (fp32) or 8 (mixed, fp64) */
    size_t u_bytes, v_bytes, m_bytes, workspace_bytes;
} wino_layer_layout;

/* ---- plans (mirror TransformSet + ConvConfig; reference transforms.py:41-145,
 *      engine.py:27-55) ---------------------------------------------------- */

/* Generate and NVRTC-compile the straight-line sm_100a kernels for one
 * transform triple (G: n x r, BT: n x n, AT: m x n programs, already ordered
 * huffman/linear and rounded to `precision`'s coefficient table).  Works
 * without a GPU (compilation only); modules are loaded on first launch. */
int wino_plan_create(int r, int m, int precision, int channel_sum, int contract_mode,
                     const wino_prog* G, const wino_prog* BT, const wino_prog* AT,
                     wino_plan** out);
void wino_plan_destroy(wino_plan* plan);

/* CUDA source of a generated kernel family (0 = layer transforms, 1 = tile
 * transforms) -- for inspection and the SASS gate. */
int wino_plan_source(const wino_plan* plan, int which, char* buf, size_t cap, size_t* len);
/* cubin of a generated module (0 = layer transforms, 1 = tile transforms,
 * 2 = contraction kernel for a C-channel layer, 3 = the fused exact contraction +
 * output-transform kernel of wino_conv2d_fused, alpha^2 <= 16 only); CPU-only OK. */
int wino_plan_cubin(wino_plan* plan, int which, int channels, void* buf, size_t cap, size_t* len);

/* Compile, concurrently on host threads, the generated kernels a layer shape
 * will launch (flags: WINO_PREPARE_*).  Optional -- every entry point compiles
 * what it needs on first use; this only overlaps the NVRTC work.  CPU-only OK.
 * Compiled cubins are cached on disk ($WINO_CACHE_DIR, else kcache/ next to
 * libwino.so), keyed by a hash of the generated source and NVRTC options. */
#define WINO_PREPARE_CONV 1   /* K1+K2, K3, K4 of wino_conv2d */
#define WINO_PREPARE_ACT 2    /* K4 with ReLU / max-pool (wino_output_transform_act) */
#define WINO_PREPARE_STAGES 4 /* wino_filter_transform / wino_input_transform alone */
#define WINO_PREPARE_NHWC 8   /* K2, K1, K3, K4 of wino_conv2d_nhwc */
#define WINO_PREPARE_K4K1 16  /* s as the second layer of wino_output_input_transform (+ K2 alone) */
int wino_plan_prepare(wino_plan* plan, const wino_layer_shape* s, int flags);

/* ---- layer-level Winograd convolution (new entry point; the reference
 *      composes it from engine.py:401-429 per tile) --------- */
int wino_layer_layout_query(const wino_plan* plan, const wino_layer_shape* s,
                            wino_layer_layout* out);
/* K2: U = (G w) G^T per (k, c)                 -- engine.py:409,411
 * U's blocking ([P][Kp/bm][Cp][bm]) follows the contraction tile the plan picks
 * for the WHOLE shape, batch size N included (wino_layer_layout_query: bm, Cp,
 * Kp).  A U computed for one shape may be reused with wino_contract for another
 * shape only if both layout queries report the same (bm, Cp, Kp).  The library
 * remembers, per device pointer, the blocking its transforms last wrote there,
 * and wino_contract returns WINO_EINVAL for a U recorded with another blocking
 * (a pointer it never wrote is taken on trust).  HostPipeline keeps one U per
 * blocking for this reason. */
int wino_filter_transform(wino_plan* plan, const wino_layer_shape* s, const void* w,
                          void* U, void* stream);
/* K1: V = (B^T d) B per (tile, c), tile gather + zero padding fused -- engine.py:410,412 */
int wino_input_transform(wino_plan* plan, const wino_layer_shape* s, const void* x,
                         void* V, void* stream);
/* K1 + K2 in one launch (the filter transform's blocks ride along) */
int wino_transforms(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w,
                    void* U, void* V, void* stream);
/* wino_transforms for a layer whose contraction is wino_contract_output_smallc (shapes with
 * wino_smallc_supported() == 2): the same U and the same values in V's C real channel rows, but
 * the rows that pad C up to the contraction's channel stage are left unwritten -- that kernel
 * never reads them (VGG-16 layer 1: 5 of 8 rows, 473 MB per batch of 256).  V is NOT valid input
 * for wino_contract. */
int wino_transforms_smallc(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w,
                           void* U, void* V, void* stream);
/* K3: M_p = sum_c U_p[c] * V_p[c] for the alpha^2 points, channel order
 * linear or pairwise (halving tree) -- engine.py:415, 252-278, 336-338 */
int wino_contract(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V,
                  void* M, void* stream);
/* K4: y = A^T M A per (k, tile), crop + NCHW write-back -- engine.py:418-423 */
int wino_output_transform(wino_plan* plan, const wino_layer_shape* s, const void* M,
                          void* y, void* stream);
/* K4 with the activation fused (conv stacks, BASELINE config 5; plans with an fp32
 * M and an fp32 y: fp32 precision with the exact, ffma, tc_bf16 or tc_fp16
 * contraction): act = relu(y) (pool = 0, act [N][K][Ho][Wo]) or the 2x2
 * max-pool of relu(y) (pool = 1, even m only, act [N][K][Ho/2][Wo/2]); the same
 * values as wino_output_transform followed by wino_relu_pool, y never stored. */
int wino_output_transform_act(wino_plan* plan, const wino_layer_shape* s, const void* M,
                              void* act, int pool, void* stream);
/* K4 of layer s + activation + K1 of the next layer s2 in ONE kernel (conv stacks; fp32 plans
 * with an FP32 contraction): a block owns whole (image, channel) planes of the activation
 * between the layers, runs layer s's output transform + ReLU (+ 2x2 max-pool, pool = 1) into
 * shared memory and layer s2's input transform from there, so the activation is never written
 * to or read from HBM -- engine.py:418-423 then engine.py:410,412 per tile.  V2 gets exactly
 * what wino_output_transform_act followed by wino_input_transform(s2) would write (same
 * rounded operations).  Needs s2 = (N, K, Ho[/2], Wo[/2]) of s, unpadded channels in s2's
 * layout (Cp == C) and PL planes in shared memory; wino_output_input_supported() says so. */
int wino_output_input_supported(wino_plan* plan, const wino_layer_shape* s, int pool,
                                const wino_layer_shape* s2);
int wino_output_input_transform(wino_plan* plan, const wino_layer_shape* s, const void* M, int pool,
                                const wino_layer_shape* s2, void* V2, void* stream);
/* K3 + K4 fused (TCF modes only): y = A^T (sum_c U_p[c] V_p[c]) A straight
 * from the tensor-memory accumulators -- engine.py:415-423 */
int wino_contract_output(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V,
                         void* y, void* stream);
/* K3 + K4 (+ activation) in one launch for small channel counts (C <= 8, e.g.
 * VGG-16 layer 1): M never goes to memory.  mode 0: y (as wino_output_transform),
 * 1: ReLU (as wino_output_transform_act pool=0), 2: ReLU + 2x2 max-pool (even m).
 * Bitwise equal to the unfused kernels.  Exact fp32 plans.  wino_smallc_supported()
 * returns 0 (shape does not qualify), 1 (first design: works, but slower than K3 + K4)
 * or 2 (C <= 4 and U, one V block and the store buffers fit in shared memory: a CTA
 * stages them with bulk copies, a thread contracts one tile x two filters column by
 * column of the point grid straight into the output transform, and the warp stores whole
 * output rows, the filter pair as packed f32x2 lanes -- VGG-16 layer 1: 1.43 ms against 2.73 ms for
 * K3 + K4). */
int wino_smallc_supported(wino_plan* plan, const wino_layer_shape* s);
int wino_contract_output_smallc(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V,
                                void* out, int mode, void* stream);

/* K2 + K1, then K3 + K4 (+ activation) in ONE exact kernel for alpha^2 <= 16 (F(2x2,3x3),
 * F(2x2,2x2), ...; fp32 plans, exact or ffma contraction): a CTA contracts all alpha^2
 * points of a 64-filter x 64-tile block and parks the accumulators in tensor memory
 * (each thread's private TMEM columns), then runs the output transform from there, so M
 * never exists in shared or global memory -- engine.py:415-423 composed per (filter,
 * tile) as engine.py:426-429.  mode 0: y, 1: ReLU, 2: ReLU + 2x2 max-pool (even m).
 * Bitwise equal to wino_conv2d (+ wino_relu_pool).  The workspace holds U and V only
 * (wino_fused_workspace bytes, 256-byte aligned). */
int wino_fused_supported(wino_plan* plan, const wino_layer_shape* s);
int wino_fused_workspace(wino_plan* plan, const wino_layer_shape* s, size_t* bytes);
int wino_conv2d_fused(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w,
                      void* out, int mode, void* workspace, size_t workspace_bytes, void* stream);

/* K2 -> K1 -> K3 -> K4 with a caller-provided workspace of
 * layout.workspace_bytes bytes (256-byte aligned). */
int wino_conv2d(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w,
                void* y, void* workspace, size_t workspace_bytes, void* stream);

/* ---- NHWC activations: x[N][H][W][C], y[N][Ho][Wo][K] (w, U, V, M and the
 * contraction are layout-independent).  Native gather / store kernels: the
 * same straight-line transforms, hence the same bits, as the NCHW entry points
 * (engine.py:401-423 per (filter, tile)).  FP32-pipe contraction modes only
 * (exact, ffma); tensor-core plans return WINO_EUNSUPPORTED. */
int wino_input_transform_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* x,
                              void* V, void* stream);
int wino_output_transform_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* M,
                               void* y, void* stream);
int wino_conv2d_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w,
                     void* y, void* workspace, size_t workspace_bytes, void* stream);

/* ---- tile-level drop-in (reference public API on (..., C, n) tiles) ------ */
/* hadamard_2d: z[B][C][n][n] = (G h G^T) o (B^T x B)      -- engine.py:401-415 */
int wino_tile_hadamard2d(wino_plan* plan, int64_t B, int C, const void* h, const void* x,
                         void* z, void* stream);
/* output_2d: out[B][m][m] = A^T y A                        -- engine.py:418-423 */
int wino_tile_output2d(wino_plan* plan, int64_t B, const void* y, void* out, void* stream);
/* hadamard_1d / output_1d                                  -- engine.py:363-387 */
int wino_tile_hadamard1d(wino_plan* plan, int64_t B, int C, const void* h, const void* x,
                         void* z, void* stream);
int wino_tile_output1d(wino_plan* plan, int64_t B, const void* y, void* out, void* stream);

/* channel_reduce: in[outer][C][inner] -> out[outer][inner], left-to-right or
 * halving-tree order (dtype 0 = f32, 1 = f64)               -- engine.py:252-287, 336-338 */
int wino_channel_reduce(int dtype, int strategy, int64_t outer, int64_t C, int64_t inner,
                        const void* in, void* out, void* stream);

/* direct_products: per-channel valid correlation, taps in kernel-index order
 * (dims 1|2; dtype 0 = f32 math, 1 = f64 math; inputs f32 or f64 per in_dtype)
 * out[B][C][o(^2)]                                          -- engine.py:309-333 */
int wino_direct_products(int dims, int dtype, int in_dtype, int64_t B, int C, int r, int n,
                         const void* h, const void* x, void* out, void* stream);

/* dot_with_order: evaluate ONE postfix row program (device array of nops
 * wino_op, coefficients already rounded) on in[count][cols] -> out[count]
 * (dtype 0 = f32, 1 = f64)                                   -- engine.py:235-246 */
int wino_program_eval(int dtype, const void* ops, int nops, int cols, int64_t count,
                      const void* in, void* out, void* stream);

/* ReLU, optionally fused with a 2x2/stride-2 max-pool, over planes[H][W]
 * (dtype 0 = f32, 1 = f64) -- the activation between layers of the VGG-16
 * conv stack (BASELINE.json config 5; not part of the reference toolkit). */
int wino_relu_pool(int dtype, int64_t planes, int H, int W, int pool, const void* in, void* out,
                   void* stream);

/* ---- fp64 oracle side and error statistics ------------------------------ */
/* Layer fp64 direct correlation (taps row-major per channel, channels left to
 * right; zero padding), x/w f32 -> y64 f64. */
int wino_direct_layer_f64(const wino_layer_shape* s, int r, const float* x, const float* w,
                          double* y64, void* stream);
/* Per-image partials stats[N][4] = {sum|y - y64|, sum|y64|, count, max|y - y64|}
 * (y dtype 0 = f32, 1 = f64), sequential order within each image. */
int wino_layer_error_stats(int64_t N, int64_t per_image, int y_dtype, const void* y,
                           const double* y64, double* stats, void* stream);

/* harness.trial_inputs on the device: the numpy Philox4x64-10 stream keyed by
 * (seed, trial), h then x, uniform(-1, 1) as random(float32) * 2 - 1
 * (harness.py:97-107), for trials t0 .. t0 + B - 1. */
int wino_trial_inputs(uint64_t seed, int64_t t0, int64_t B, int dims, int r, int n, int C,
                      float* h, float* x, void* stream);
/* Per-trial L1: per_trial[b] = sum_i |out[b][i] - ref[b][i]| summed in numpy's
 * pairwise order (harness.py:143-151); out dtype 0 = f32, 1 = f64. */
int wino_trial_l1(int64_t B, int64_t per, int out_dtype, const void* out, const double* ref,
                  double* per_trial, void* stream);
/* numpy-ordered mean of a f64 vector (ErrorReport.total_l1_mean, harness.py:155). */
int wino_mean_f64(int64_t n, const double* v, double* out, void* stream);

/* Arithmetic-throughput probe for roofline denominators: `blocks` x 256
 * threads, each running 8 independent chains of `iters` steps of
 * mode 0 FFMA | 1 FMUL+FADD | 2 DFMA | 3 DMUL+DADD (immediate multiplier
 * and addend) | 4 FMUL+FADD with register operands (read from out[2], out[3];
 * the operand form of the exact contraction) | 5 packed exact FFMA2(a, m, -0) +
 * FADD2 | 6 packed FFMA2; flops = 2 per lane step (packed steps carry 2 lanes). */
int wino_peak_probe(int mode, int blocks, int iters, float* out, void* stream);

/* number of kernels this library has launched in the calling process */
int64_t wino_launch_count(void);
const char* wino_last_error(void);
/* Tuning hooks for tools/ sweeps and variant tests (the product never sets them):
 * key "gemm" = contraction tile "tm,tn,thm,thn,bk,stages,maxreg[,ku,noprod,pack]"
 * (plans created afterwards), "dbuf", "tcf_nk" (same), "k1" = "tile" | "gather" (K1 from
 * global memory only) | "bulk<KB>" (shared-memory cap of the bulk-staged K1), "k1order" =
 * "t", "k4" = "staged", "k1tc" = "4x8", "tile_interp" = "0|1", "cpt" / "kpt" =
 * 1|2|4|8, "tcf_dbg", "tc_epi", "tc_epw" (epilogue warps per TMEM lane quarter: 1|2|4),
 * "k1tc_staged" (0: off, 2: every image size) / "k1tc_blocks", "k1rowwise" / "k4rowwise", "sc2_kg" (filter-pair warp groups
 * of the small-C fused kernel), "k4k1_ks" (read once per process, before the first launch).
 * value NULL or "" clears the key.  Unknown keys -> WINO_EINVAL. */
int wino_tuning_set(const char* key, const char* value);
const char* wino_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WINO_H */
