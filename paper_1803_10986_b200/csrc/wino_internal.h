// Internal helpers shared by the libwino translation units.
#pragma once
#include <string>

#include "../../include/wino.h"

namespace wino {
// Tuning registry (wino_tuning_set): alternative kernel forms and tile configs for
// tools/ sweeps and variant tests.  Empty string = not set (the default path).
std::string tuning(const char* key);
// record an error message for wino_last_error() and return `code`
int fail(int code, const std::string& msg);
// check the last CUDA launch, count it, translate errors
int after_launch(const char* what);
void count_launch();
// K3t: tcgen05 tensor-core contraction (tc_contract.cu)
int tc_contract_launch(const void* U, const void* V, void* M, long long Kp, long long Tp, long long Cp, int P,
                       int fp16, int K, void* stream);
// the tcgen05 contraction's dynamic smem opt-in, once per device
int tc_contract_prepare_device(int dev);
// device copies of a plan's row programs (postfix ops + row starts) for the
// interpreted tile transforms (wino_static.cu)
struct DevProgs {
    const wino_op *G, *BT, *AT;
    const int *Grs, *BTrs, *ATrs;
};
int tile_hadamard_interp_launch(int precision, int dims, const DevProgs& pg, int r, int n, long long BC,
                                const void* h, const void* x, void* z, void* stream);
int tile_output_interp_launch(int precision, int dims, const DevProgs& pg, int n, int m, long long B, const void* y,
                              void* out, void* stream);
}  // namespace wino
