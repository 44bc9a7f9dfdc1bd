// CUDA source generation for the transform kernels of one transform triple.
//
// Each matrix row is a postfix program (wino_op).  The emitter turns it into
// straight-line SSA code with explicit round-to-nearest intrinsics
// (__fmul_rn/__fadd_rn/__fsub_rn or their f64 forms) so that every product and
// every sum rounds exactly once, exactly as the reference's numpy evaluation
// (engine.py:191-232).  Exact rewrites only:
//   * coefficient +1: the operand itself (1*x == x);
//   * coefficient -1: a pending negation, folded into the consuming add as a
//     subtraction (a + (-1*x) == a - x bit for bit; (-x) + (-y) == (-x) - y);
//   * a row with no nonzero coefficient yields +0 (np.zeros_like).
#pragma once
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/wino.h"

namespace wino {

struct RowProg {
    std::vector<wino_op> ops;
};

struct MatProg {
    int rows = 0, cols = 0;
    std::vector<RowProg> row;
};

struct GenTypes {
    bool compute_double;  // transform arithmetic type
    bool in_double;       // layer / tile inputs (x, w, h)
    bool uv_double;       // U, V, M, z (working precision of the Hadamard stage)
    bool y_double;        // outputs
};

// validate the stack discipline of a program; returns "" or an error message
std::string validate(const MatProg& m, int expect_rows, int expect_cols, const char* name);

// U and V are written in the contraction's blocked layout:
//   U[p][k / bm][c][k % bm],  V[p][t / bn][c][t % bn]
// so one pipeline stage of a contraction tile is a single contiguous block.
std::string gen_layer_source(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                             const GenTypes& ty, int bm, int bn);
// tensor-core variant: 16-bit U/V in the UMMA K-major core-matrix layout (see codegen.cpp);
// fused_nk > 0: the fused K3t+K4 layouts and kernel (wino_tcf, NK filters per tile)
std::string gen_layer_source_tc(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                                const GenTypes& ty, bool fp16, int fused_nk = 0);
std::string gen_tile_source(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                            const GenTypes& ty);
// wino_fused_out(): output transform of one (filter, tile) pair from registers, for the fused
// exact contraction (contract_template.cuh WINO_FUSE_P); fp32 plans
std::string gen_fused_out_source(int r, int m, const MatProg& AT);

// Gather transforms: channels per K1 thread / output channels per K4 thread (the
// tile index math is amortised over them).  Must divide every channel padding
// (Cp is a multiple of 8).  Tuning keys "cpt" / "kpt" override (1, 2, 4 or 8; read
// once per process, before the first plan, so generated code and launch grids agree).  A rolled
// loop over channels is slower (tools/sweeps/sweep_xpt.sh: fewer loads in flight --
// cfg3 m=6 K4 38.9 / 65.8 / 77.1 us at 1 / 4 / 8 filters per thread); K4 keeps 1.
std::string tuning(const char* key);  // wino_host.cu registry (wino_tuning_set)
inline int tuning_pow2(const char* name, int dflt) {
    const std::string e = tuning(name);
    const int v = e.empty() ? dflt : std::atoi(e.c_str());
    return (v == 1 || v == 2 || v == 4 || v == 8) ? v : dflt;
}
// channels per K1 thread: 2 for alpha^2 <= 16 (the two windows are gathered and
// transformed in one unrolled body: more loads in flight, half the index math;
// cfg2 K1 14.7 -> 12.7 us), 1 for larger alpha (register pressure: cfg3 m=6
// 39 -> 54 us at 2).  Tuning key "cpt" overrides.
inline int gather_cpt(int P) {
    static const int v = tuning_pow2("cpt", 0);
    return v ? v : (P <= 16 ? 2 : 1);
}
inline int gather_kpt() {
    static const int v = tuning_pow2("kpt", 1);
    return v;
}

}  // namespace wino
