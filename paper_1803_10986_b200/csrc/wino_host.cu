// libwino host side: plans, NVRTC JIT of generated sm_100a kernels, driver-API
// module loading and launches, and the C-ABI entry points of include/wino.h.
//
// A plan mirrors (TransformSet, ConvConfig) of the reference (transforms.py:41-145,
// engine.py:27-55): it owns the row programs of G, B^T and A^T, the generated
// transform source, and lazily compiled contraction variants.  Nothing here
// falls back to the CPU: every compute entry point launches device kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "codegen.h"
#include "wino_internal.h"

namespace wino {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::mutex g_tune_mu;
static std::map<std::string, std::string> g_tune;

std::string tuning(const char* key) {
    std::lock_guard<std::mutex> g(g_tune_mu);
    auto it = g_tune.find(key);
    return it == g_tune.end() ? std::string() : it->second;
}

int after_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(WINO_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    count_launch();
    return WINO_OK;
}

// ------------------------------------------------------------------ driver API
struct Driver {
    CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**) = nullptr;
    CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
    CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t) = nullptr;
    bool ok = false;
    std::string err;
};

static Driver& driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) -> bool {
            cudaDriverEntryPointQueryResult q;
            cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
            return e == cudaSuccess && q == cudaDriverEntryPointSuccess && *fn;
        };
        bool ok = get("cuModuleLoadData", (void**)&d.ModuleLoadData) &&
                  get("cuModuleGetFunction", (void**)&d.ModuleGetFunction) &&
                  get("cuLaunchKernel", (void**)&d.LaunchKernel) &&
                  get("cuFuncSetAttribute", (void**)&d.FuncSetAttribute) &&
                  get("cuGetErrorString", (void**)&d.GetErrorString) &&
                  get("cuOccupancyMaxActiveBlocksPerMultiprocessor",
                      (void**)&d.OccupancyMaxActiveBlocksPerMultiprocessor);
        d.ok = ok;
        if (!ok) d.err = "CUDA driver entry points unavailable (no GPU driver?)";
    });
    return d;
}

static std::string cu_err(CUresult r) {
    const char* s = nullptr;
    if (driver().GetErrorString) driver().GetErrorString(r, &s);
    return s ? s : ("CUresult " + std::to_string((int)r));
}

// ------------------------------------------------------------------ NVRTC
struct Compiled {
    std::vector<char> cubin;
    std::string log;
};

static const char* const kNvrtcOpts[] = {"-arch=sm_100a", "-fmad=false", "-lineinfo", "-std=c++17",
                                         "-default-device", "--ptxas-options=-v"};

// ---- on-disk cubin cache: <dir>/<module>-<128-bit FNV-1a of (options, source)>.cubin.
// dir = $WINO_CACHE_DIR, else kcache/ next to libwino.so (in-tree, git-ignored, so a
// cache filled here by build() travels with the snapshot to the GPU box).  Entries
// are written atomically (temp file + rename); unreadable or short files are ignored.
static std::string cache_dir() {
    static const std::string dir = [] {
        if (const char* e = std::getenv("WINO_CACHE_DIR")) return std::string(e);
        Dl_info info;
        if (dladdr((void*)&cache_dir, &info) && info.dli_fname) {
            std::string so = info.dli_fname;
            const size_t k = so.rfind('/');
            return (k == std::string::npos ? std::string(".") : so.substr(0, k)) + "/kcache";
        }
        return std::string();
    }();
    return dir;
}

static std::string cache_key(const std::string& text) {
    uint64_t a = 1469598103934665603ull, b = 0x9ae16a3b2f90404full;
    for (unsigned char c : text) {
        a = (a ^ c) * 1099511628211ull;
        b = (b ^ c) * 0x100000001b3ull + 0x2545f4914f6cdd1dull;
    }
    char buf[40];
    std::snprintf(buf, sizeof buf, "%016llx%016llx", (unsigned long long)a, (unsigned long long)b);
    return buf;
}

static bool cache_load(const std::string& path, std::vector<char>* out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    std::vector<char> data;
    char tmp[1 << 16];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof tmp, f)) > 0) data.insert(data.end(), tmp, tmp + k);
    std::fclose(f);
    // ELF magic + a sane size: a torn or foreign file is recompiled
    if (data.size() < 64 || data[0] != 0x7f || data[1] != 'E' || data[2] != 'L' || data[3] != 'F') return false;
    out->swap(data);
    return true;
}

static void cache_store(const std::string& path, const std::vector<char>& cubin) {
    const std::string dir = path.substr(0, path.rfind('/'));
    mkdir(dir.c_str(), 0775);
    const std::string tmp = path + ".tmp" + std::to_string((long long)getpid()) + "_" +
                            std::to_string((unsigned long long)std::hash<std::thread::id>{}(std::this_thread::get_id()));
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    if (std::fclose(f) == 0 && ok) {
        std::rename(tmp.c_str(), path.c_str());
    } else {
        std::remove(tmp.c_str());
    }
}

static int nvrtc_compile(const std::string& src, const std::string& name, Compiled* out, int maxreg = 0) {
    std::vector<const char*> opts(std::begin(kNvrtcOpts), std::end(kNvrtcOpts));
    std::string mr = "-maxrregcount=" + std::to_string(maxreg);
    if (maxreg > 0) opts.push_back(mr.c_str());
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    std::string keytext = "nvrtc " + std::to_string(major) + "." + std::to_string(minor);
    for (const char* o : opts) keytext += std::string(" ") + o;
    keytext += "\n" + src;
    const std::string dir = cache_dir();
    const std::string path = dir.empty() ? std::string() : dir + "/" + name + "-" + cache_key(keytext) + ".cubin";
    if (!path.empty() && cache_load(path, &out->cubin)) {
        out->log = "(cubin cache: " + path + ")";
        return WINO_OK;
    }
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), name.c_str(), 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(WINO_ECOMPILE, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    out->log.assign(ls, '\0');
    if (ls) nvrtcGetProgramLog(prog, &out->log[0]);
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return fail(WINO_ECOMPILE, "NVRTC failed on " + name + ": " + out->log.substr(0, 4000));
    }
    size_t cs = 0;
    nvrtcGetCUBINSize(prog, &cs);
    out->cubin.resize(cs);
    nvrtcGetCUBIN(prog, out->cubin.data());
    nvrtcDestroyProgram(&prog);
    if (!path.empty()) cache_store(path, out->cubin);
    return WINO_OK;
}

// Wrap every `extern "C" __global__` definition of a generated source in
//   #if defined(WINO_KALL) || defined(WINO_K_<name>) ... #endif
// so one NVRTC program per kernel compiles only that kernel (the shared device
// functions are static inline: unreferenced ones cost nothing).  Straight-line
// transform code makes NVRTC time grow steeply with alpha, and a layer source
// holds up to nine kernel variants of which a call path uses two or three.
static std::string wrap_kernels(const std::string& s) {
    static const std::string tag = "extern \"C\" __global__";
    std::string out;
    out.reserve(s.size() + 4096);
    size_t i = 0;
    while (true) {
        const size_t j = s.find(tag, i);
        if (j == std::string::npos) {
            out.append(s, i, std::string::npos);
            break;
        }
        out.append(s, i, j - i);
        size_t p = s.find('(', j + tag.size());
        // `__launch_bounds__(...)` precedes the kernel name
        const size_t lb = s.find("__launch_bounds__", j);
        if (lb != std::string::npos && lb < p) {
            int d = 0;
            size_t q = p;
            for (; q < s.size(); ++q) {
                if (s[q] == '(') ++d;
                if (s[q] == ')' && --d == 0) break;
            }
            p = s.find('(', q + 1);
        }
        size_t ne = p;
        while (ne > 0 && (s[ne - 1] == ' ' || s[ne - 1] == '\n')) --ne;
        size_t nb = ne;
        while (nb > 0 && (std::isalnum((unsigned char)s[nb - 1]) || s[nb - 1] == '_')) --nb;
        const std::string name = s.substr(nb, ne - nb);
        int d = 0;
        size_t q = p;
        for (; q < s.size(); ++q) {  // end of the parameter list
            if (s[q] == '(') ++d;
            if (s[q] == ')' && --d == 0) break;
        }
        size_t e = s.find('{', q);
        d = 0;
        for (; e < s.size(); ++e) {  // matching brace of the body (generated code: no braces in comments)
            if (s[e] == '/' && e + 1 < s.size() && s[e + 1] == '/') {
                e = s.find('\n', e);
                continue;
            }
            if (s[e] == '{') ++d;
            if (s[e] == '}' && --d == 0) break;
        }
        out += "#if defined(WINO_KALL) || defined(WINO_K_" + name + ")\n";
        out.append(s, j, e + 1 - j);
        out += "\n#endif\n";
        i = e + 1;
    }
    return out;
}

// A generated module: source, and one cubin per kernel (compiled on first use,
// concurrently for different kernels), loaded per device.
struct Module {
    std::string name, source;
    int maxreg = 0;  // NVRTC -maxrregcount (0 = compiler default)
    struct Bin {
        std::mutex mu;
        bool done = false;
        Compiled bin;
    };
    std::mutex mu;  // guards the maps below (never held while compiling)
    std::string wrapped;
    std::map<std::string, std::unique_ptr<Bin>> bins;  // kernel name ("*": all kernels)
    std::map<std::pair<int, std::string>, CUmodule> mods;
    std::map<std::pair<int, std::string>, CUfunction> fns;

    Bin* bin_of(const std::string& kernel) {
        std::lock_guard<std::mutex> g(mu);
        if (wrapped.empty()) wrapped = wrap_kernels(source);
        auto& b = bins[kernel];
        if (!b) b = std::make_unique<Bin>();
        return b.get();
    }

    // cubin holding `kernel` ("*": every kernel of the source)
    int ensure_compiled(const std::string& kernel, const Compiled** out = nullptr) {
        Bin* b = bin_of(kernel);
        std::lock_guard<std::mutex> g(b->mu);
        if (!b->done) {
            const std::string def = kernel == "*" ? std::string("#define WINO_KALL 1\n")
                                                  : "#define WINO_K_" + kernel + " 1\n";
            const std::string nm = name.substr(0, name.size() - 3) + (kernel == "*" ? "" : "." + kernel) + ".cu";
            int rc = nvrtc_compile(def + wrapped, nm, &b->bin, maxreg);
            if (rc) return rc;
            b->done = true;
        }
        if (out) *out = &b->bin;
        return WINO_OK;
    }

    int function(const char* fname, CUfunction* f) {
        const Compiled* bin = nullptr;
        int rc = ensure_compiled(fname, &bin);
        if (rc) return rc;
        Driver& d = driver();
        if (!d.ok) return fail(WINO_ECUDA, d.err);
        int dev = 0;
        cudaError_t ce = cudaGetDevice(&dev);
        if (ce != cudaSuccess) return fail(WINO_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(ce));
        std::lock_guard<std::mutex> g(mu);
        auto key = std::make_pair(dev, std::string(fname));
        auto it = fns.find(key);
        if (it != fns.end()) {
            *f = it->second;
            return WINO_OK;
        }
        if (!mods.count(key)) {
            cudaFree(nullptr);  // make the runtime's primary context current
            CUmodule mod;
            CUresult cr = d.ModuleLoadData(&mod, bin->cubin.data());
            if (cr != CUDA_SUCCESS) return fail(WINO_ECUDA, "cuModuleLoadData(" + name + "): " + cu_err(cr));
            mods[key] = mod;
        }
        CUfunction fn;
        CUresult cr = d.ModuleGetFunction(&fn, mods[key], fname);
        if (cr != CUDA_SUCCESS) return fail(WINO_ECUDA, std::string("cuModuleGetFunction(") + fname + "): " + cu_err(cr));
        fns[key] = fn;
        *f = fn;
        return WINO_OK;
    }
};

// Compile (module, kernel) pairs concurrently, one host thread each (NVRTC is
// thread-safe; a layer plan needs two to four kernels whose compile times add up).
static int compile_all(const std::vector<std::pair<Module*, std::string>>& work) {
    if (work.size() <= 1) return work.empty() ? WINO_OK : work[0].first->ensure_compiled(work[0].second);
    std::vector<int> rcs(work.size(), WINO_OK);
    std::vector<std::string> errs(work.size());
    std::vector<std::thread> th;
    for (size_t i = 0; i < work.size(); ++i)
        th.emplace_back([&, i] {
            rcs[i] = work[i].first->ensure_compiled(work[i].second);
            if (rcs[i]) errs[i] = g_last_error;  // thread-local: carry it to the caller's thread
        });
    for (auto& t : th) t.join();
    for (size_t i = 0; i < work.size(); ++i)
        if (rcs[i]) return fail(rcs[i], errs[i]);
    return WINO_OK;
}

static int launch(CUfunction f, dim3 grid, dim3 block, unsigned smem, void* stream, void** args, const char* what) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return WINO_OK;
    if (smem > 48 * 1024) {
        CUresult cr = driver().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
        if (cr != CUDA_SUCCESS) return fail(WINO_ECUDA, std::string(what) + ": set smem: " + cu_err(cr));
    }
    CUresult cr = driver().LaunchKernel(f, grid.x, grid.y, grid.z, block.x, block.y, block.z, smem,
                                        (CUstream)stream, args, nullptr);
    if (cr != CUDA_SUCCESS)
        return fail(WINO_ECUDA, std::string(what) + ": " + cu_err(cr) + " (grid " + std::to_string(grid.x) + "x" +
                                    std::to_string(grid.y) + ", block " + std::to_string(block.x) + ", dynamic smem " +
                                    std::to_string(smem) + ")");
    count_launch();
    return WINO_OK;
}

// ------------------------------------------------------------------ contraction template
static const char* kContractTemplate =
#include "contract_src.inc"
    ;

struct GemmCfg {
    int tm, tn, thm, thn, bk, stages, maxreg, ku = 0;  // ku: k-steps unrolled per inner loop (0 = bk)
    int noprod = 0;  // 1: no producer warp (last consumer warp to release a stage refills it)
    int pack = 0;    // 1: packed f32x2 arithmetic (float U/V only)
    int wn = 0;      // > 0: warp-tiled thread map, wn lanes along t x 32/wn lanes along k
    // Dynamic shared memory of a contraction kernel: the operand ring, 2 mbarriers per
    // stage, and (pairwise, when it fits) the dynamic-counter slots -- `levels` x the
    // consumer threads' accumulator tiles -- which otherwise live in registers.
    // Returns the byte count; *slots_smem tells which form the module is generated in.
    long long smem_bytes(int levels, int eb, bool* slots_smem) const {
        const long long ring = (long long)stages * bk * (bm() + bn()) * eb + 2LL * stages * 8;
        const long long slots = (long long)levels * tm * tn * eb * threads();
        *slots_smem = levels > 0 && ring + slots <= 232448 - 1024;  // B200: 227 KB of opt-in smem per CTA
        return ring + (*slots_smem ? slots : 0);
    }
    int bm() const { return thm * tm; }
    int bn() const { return thn * tn; }
    int threads() const { return thm * thn; }
    int block() const { return thm * thn + (noprod ? 0 : 32); }
};

}  // namespace wino

// The fused exact path (wino_conv2d_fused) runs the regular transforms with the tile config
// of its own contraction: while a ForceCand guard is alive on this thread, wino_plan::pick()
// returns that candidate instead of choosing by shape.
static thread_local int g_force_cand = -1;
struct ForceCand {
    int prev;
    explicit ForceCand(int ci) : prev(g_force_cand) { g_force_cand = ci; }
    ~ForceCand() { g_force_cand = prev; }
};

// ------------------------------------------------------------------ plan
struct wino_plan {
    int r, m, n, precision, chsum, mode;
    int nk = 0;  // fused tensor-core modes: filters per TMEM block (P * nk <= 512)
    bool fused() const { return mode >= WINO_CONTRACT_TCF_BF16; }
    wino::MatProg G, BT, AT;
    wino::GenTypes ty;
    wino::GemmCfg gemm;                 // cands[0]
    std::vector<wino::GemmCfg> cands;   // contraction tile configs a layer shape picks from
    int fused_ci = -1;                  // candidate of the fused exact K3 + K4 kernel (never picked by shape)
    wino::Module layer, tile;           // layer: transforms blocked for cands[0]
    std::mutex mu;
    std::map<int, std::unique_ptr<wino::Module>> contract;  // key: counter levels * 16 + candidate
    std::map<int, std::unique_ptr<wino::Module>> layer_x;   // transforms for other (bm, bn) blockings
    std::map<int, wino::DevProgs> dprogs;                     // per device: programs for the tile interpreter

    ~wino_plan() {  // device program copies (errors ignored: the context may already be gone at exit)
        int cur = 0;
        if (dprogs.empty() || cudaGetDevice(&cur) != cudaSuccess) return;
        for (auto& kv : dprogs) {
            if (cudaSetDevice(kv.first) == cudaSuccess) cudaFree(const_cast<wino_op*>(kv.second.G));
        }
        cudaSetDevice(cur);
        cudaGetLastError();
    }

    // Device copies of G / B^T / A^T (postfix ops + row starts), uploaded once per
    // device on first use by the interpreted tile transforms.
    int dev_progs(wino::DevProgs* out) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return wino::fail(WINO_ECUDA, "dev_progs: no CUDA device");
        std::lock_guard<std::mutex> g(mu);
        auto it = dprogs.find(dev);
        if (it != dprogs.end()) {
            *out = it->second;
            return WINO_OK;
        }
        std::vector<wino_op> ops;
        std::vector<int> rs;
        size_t off_op[3], off_rs[3];
        const wino::MatProg* mats[3] = {&G, &BT, &AT};
        for (int q = 0; q < 3; ++q) {
            off_op[q] = ops.size();
            off_rs[q] = rs.size();
            int pos = 0;
            for (const auto& row : mats[q]->row) {
                rs.push_back(pos);
                ops.insert(ops.end(), row.ops.begin(), row.ops.end());
                pos += (int)row.ops.size();
            }
            rs.push_back(pos);
        }
        const size_t ob = ops.size() * sizeof(wino_op), rb = rs.size() * sizeof(int);
        char* d = nullptr;
        if (cudaMalloc(&d, ob + rb + 16) != cudaSuccess) return wino::fail(WINO_ECUDA, "dev_progs: cudaMalloc");
        if (cudaMemcpy(d, ops.data(), ob, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(d + ob, rs.data(), rb, cudaMemcpyHostToDevice) != cudaSuccess)
            return wino::fail(WINO_ECUDA, "dev_progs: upload");
        const wino_op* dops = reinterpret_cast<const wino_op*>(d);
        const int* drs = reinterpret_cast<const int*>(d + ob);
        wino::DevProgs pg{dops + off_op[0], dops + off_op[1], dops + off_op[2],
                          drs + off_rs[0], drs + off_rs[1], drs + off_rs[2]};
        dprogs[dev] = pg;
        *out = pg;
        return WINO_OK;
    }

    // Tile config for a layer shape: the candidate with the least padded work per
    // persistent wave.  cost = ceil(tiles / slots) * bm * bn * Cp / eff, slots = 148 SMs x 3
    // co-resident CTAs (a fixed B200 constant, so the layout never depends on which
    // device answers); ties keep the earlier candidate.
    static long long rup(long long v, long long q) { return (v + q - 1) / q * q; }
    int pick(const wino_layer_shape* s) const {
        if (g_force_cand >= 0 && g_force_cand < (int)cands.size()) return g_force_cand;
        if (cands.size() < 2) return 0;
        const int Ho = s->H + 2 * s->pad - r + 1, Wo = s->W + 2 * s->pad - r + 1;
        const long long T = (long long)s->N * ((Ho + m - 1) / m) * ((Wo + m - 1) / m);
        const long long slots = 148 * 3;
        int best = 0;
        double best_cost = 0;
        for (size_t i = 0; i < cands.size(); ++i) {
            if ((int)i == fused_ci) continue;
            const long long bm = cands[i].bm(), bn = cands[i].bn();
            const long long tiles = (long long)n * n * ((s->K + bm - 1) / bm) * (((T > 0 ? T : 1) + bn - 1) / bn);
            // measured per-flop speed of the 4x8 / 4x4 microtiles vs 8x8: 0.91 / 0.92 (cfg2, cfg3)
            const double eff = cands[i].tm * cands[i].tn < 64 ? 0.91 : 1.0;
            const double cost = (double)((tiles + slots - 1) / slots) * bm * bn * rup(s->C, cands[i].bk) / eff;
            if (i == 0 || cost < best_cost * 0.97) {
                best = (int)i;
                best_cost = cost;
            }
        }
        return best;
    }

    wino::Module* layer_mod(int ci) {
        if (ci <= 0 || (cands[ci].bm() == gemm.bm() && cands[ci].bn() == gemm.bn())) return &layer;
        const int key = cands[ci].bm() * 4096 + cands[ci].bn();
        std::lock_guard<std::mutex> g(mu);
        auto it = layer_x.find(key);
        if (it != layer_x.end()) return it->second.get();
        auto mod = std::make_unique<wino::Module>();
        mod->name = layer.name.substr(0, layer.name.size() - 3) + "_b" + std::to_string(cands[ci].bm()) + "x" +
                    std::to_string(cands[ci].bn()) + ".cu";
        mod->source = wino::gen_layer_source(r, m, G, BT, AT, ty, cands[ci].bm(), cands[ci].bn());
        wino::Module* raw = mod.get();
        layer_x[key] = std::move(mod);
        return raw;
    }

    int sum_mode() const { return (mode == WINO_CONTRACT_FFMA ? 2 : 0) + (chsum == WINO_SUM_PAIRWISE ? 1 : 0); }

    wino::Module* contract_module(long long Cp, int ci = 0, bool fused_out = false) {
        const wino::GemmCfg& gemm = cands.empty() ? this->gemm : cands[ci];
        int levels = 1;
        const long long Q = Cp / gemm.bk;  // pairwise: the dynamic counter runs over stages
        while ((1LL << levels) <= Q) ++levels;  // bit_length(Q)
        if (chsum != WINO_SUM_PAIRWISE) levels = 0;
        bool slots_smem = false;
        gemm.smem_bytes(levels, ty.uv_double ? 8 : 4, &slots_smem);
        std::lock_guard<std::mutex> g(mu);
        const int key = levels * 16 + ci + (fused_out ? 1 << 20 : 0);
        auto it = contract.find(key);
        if (it != contract.end()) return it->second.get();
        auto mod = std::make_unique<wino::Module>();
        std::ostringstream os;
        const bool dbl = ty.uv_double;
        os << "#define WINO_DT " << (dbl ? "double" : "float") << "\n#define WINO_DT_IS_DOUBLE " << (dbl ? 1 : 0)
           << "\n#define WINO_TM " << gemm.tm << "\n#define WINO_TN " << gemm.tn << "\n#define WINO_THM " << gemm.thm
           << "\n#define WINO_THN " << gemm.thn << "\n#define WINO_BK " << gemm.bk << "\n#define WINO_STAGES "
           << gemm.stages << "\n#define WINO_SUM " << sum_mode() << "\n#define WINO_LEVELS "
           << (levels > 0 ? levels : 1) << "\n#define WINO_MAXREG " << gemm.maxreg << "\n#define WINO_KU " << (gemm.ku > 0 ? gemm.ku : gemm.bk) << "\n#define WINO_NOPROD " << gemm.noprod
           << "\n#define WINO_PACK " << (gemm.pack && !dbl ? 1 : 0) << "\n#define WINO_WN " << gemm.wn << "\n#define WINO_SLOTS_SMEM " << slots_smem << "\n"
           << (!wino::tuning("dbuf").empty() ? "#define WINO_DBUF " + wino::tuning("dbuf") + "\n" : std::string())
           << (fused_out ? std::string(wino::tuning("dbuf").empty() ? "#define WINO_DBUF 1\n" : "") + "#define WINO_FUSE_P " +
                               std::to_string(n * n) + "\n" + wino::gen_fused_out_source(r, m, AT)
                         : std::string())
           << wino::kContractTemplate;
        mod->source = os.str();
        mod->name = std::string(fused_out ? "wino_contract_fused_r" + std::to_string(r) + "m" + std::to_string(m) + "_s"
                                          : "wino_contract_s") +
                    std::to_string(sum_mode()) + "_L" + std::to_string(levels) + "_c" + std::to_string(ci) + ".cu";
        wino::Module* raw = mod.get();
        contract[key] = std::move(mod);
        return raw;
    }
};

namespace {

int convert_prog(const wino_prog* p, wino::MatProg* out) {
    if (!p || p->rows < 1 || p->cols < 1 || !p->row_start) return -1;
    out->rows = p->rows;
    out->cols = p->cols;
    out->row.resize(p->rows);
    for (int i = 0; i < p->rows; ++i) {
        const int a = p->row_start[i], b = p->row_start[i + 1];
        if (a < 0 || b < a || (b > a && !p->ops)) return -1;
        out->row[i].ops.assign(p->ops + a, p->ops + b);
    }
    return 0;
}

long long round_up(long long v, long long q) { return (v + q - 1) / q * q; }

int layout_of(const wino_plan* p, const wino_layer_shape* s, wino_layer_layout* L) {
    if (!p || !s || !L) return wino::fail(WINO_EINVAL, "null argument");
    if (s->N < 0 || s->C < 1 || s->K < 1 || s->H < 1 || s->W < 1 || s->pad < 0)
        return wino::fail(WINO_EINVAL, "layer shape: N >= 0, C, K, H, W >= 1, pad >= 0 required");
    const int Ho = s->H + 2 * s->pad - p->r + 1, Wo = s->W + 2 * s->pad - p->r + 1;
    if (Ho < 1 || Wo < 1) return wino::fail(WINO_EINVAL, "input smaller than kernel");
    if (p->n > 16) return wino::fail(WINO_EUNSUPPORTED, "layer path: alpha = r + m - 1 > 16 is not generated");
    std::memset(L, 0, sizeof *L);
    L->P = p->n * p->n;
    const wino::GemmCfg& g = p->cands.empty() ? p->gemm : p->cands[p->pick(s)];
    L->bm = g.bm();
    L->bn = g.bn();
    L->Ho = Ho;
    L->Wo = Wo;
    L->th = (Ho + p->m - 1) / p->m;
    L->tw = (Wo + p->m - 1) / p->m;
    L->T = (long long)s->N * L->th * L->tw;
    if (L->T > (1LL << 30) || (long long)s->H * s->W > (1LL << 30) || s->K > (1 << 30))
        return wino::fail(WINO_EUNSUPPORTED, "layer too large for 32-bit tile indexing; split the batch");
    L->Tp = round_up(L->T > 0 ? L->T : 1, g.bn());
    L->Cp = round_up(s->C, g.bk);
    L->Kp = round_up(s->K, g.bm());
    if (p->fused()) {  // wino_tcf blocking: 128 tiles x nk filters x 16 channels
        L->bm = p->nk;
        L->bn = 128;
        L->Tp = round_up(L->T > 0 ? L->T : 1, 128);
        L->Cp = round_up(s->C, 16);
        L->Kp = round_up(s->K, p->nk);
    }
    const bool tc = p->mode >= WINO_CONTRACT_TC_BF16;
    L->elem_bytes_uv = tc ? 2 : p->ty.uv_double ? 8 : 4;  // tc: 16-bit U/V, fp32 M
    L->elem_bytes_y = p->ty.y_double ? 8 : 4;
    L->u_bytes = (size_t)L->P * L->Cp * L->Kp * L->elem_bytes_uv;
    L->v_bytes = (size_t)L->P * L->Cp * L->Tp * L->elem_bytes_uv;
    L->m_bytes = p->fused() ? 0 : (size_t)L->P * L->Kp * L->Tp * (tc ? 4 : L->elem_bytes_uv);
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    L->workspace_bytes = al(L->u_bytes) + al(L->v_bytes) + al(L->m_bytes);
    return WINO_OK;
}

// ---- U layout registry.  U is blocked [P][Kp/bm][Cp][bm] for the contraction tile the plan
// picks for the WHOLE layer shape (batch size included), and a caller-owned device pointer
// carries no layout.  The transforms record, per (device, U pointer), the blocking they
// wrote; wino_contract rejects a U recorded with a different blocking instead of silently
// reading it with the wrong one (e.g. a U computed once for the weights and reused at
// another batch size).  Pointers the library never wrote are not checked.
struct ULayout {
    long long bm, Cp, Kp;
    int P;
};
static std::mutex g_u_mu;
static std::map<std::pair<int, const void*>, ULayout> g_u_layouts;

void u_layout_record(const void* U, const wino_layer_layout& L) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_u_mu);
    if (g_u_layouts.size() > 4096) g_u_layouts.clear();  // bounded: stale entries only cost a missed check
    g_u_layouts[{dev, U}] = ULayout{L.bm, L.Cp, L.Kp, L.P};
}

int u_layout_check(const void* U, const wino_layer_layout& L, const char* what) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_u_mu);
    auto it = g_u_layouts.find({dev, U});
    if (it == g_u_layouts.end()) return WINO_OK;
    const ULayout& r = it->second;
    if (r.bm == L.bm && r.Cp == L.Cp && r.Kp == L.Kp && r.P == L.P) return WINO_OK;
    return wino::fail(WINO_EINVAL, std::string(what) + ": U was transformed with blocking (bm " + std::to_string(r.bm) +
                                       ", Cp " + std::to_string(r.Cp) + ", Kp " + std::to_string(r.Kp) +
                                       ") but this layer shape contracts with (bm " + std::to_string(L.bm) + ", Cp " +
                                       std::to_string(L.Cp) + ", Kp " + std::to_string(L.Kp) +
                                       "): transform the filters again for this shape (wino_layer_layout_query)");
}

inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// K1 / K4 block size (must match codegen.cpp): 128 tiles, halved while the
// P x TB smem staging buffer exceeds 64 KB.
int xform_block(const wino_plan* p, int* smem) {
    const int P = p->n * p->n, es = (p->ty.uv_double && p->mode < WINO_CONTRACT_TC_BF16) ? 8 : 4;
    int tb = 128;
    while (tb > 32 && (long long)P * tb * es > 64 * 1024) tb /= 2;
    *smem = P * tb * es;
    return tb;
}

// K1 variant: "gather" (codegen.cpp emit_input_gather: windows gathered from
// global memory, values stored straight from registers; default) or "tile"
// (input_body: values parked in smem, 16-byte stores; also the fallback when
// the gather grid (Cp, n_tb + n_kb) exceeds 65535 rows).  WINO_K1=tile selects
// the latter for A/B timing.
// block order of the tile kernel: channel fastest (default) or tile chunk fastest (WINO_K1ORDER=t)
int k1_cfast() {
    static const int v = [] {
        const std::string es = wino::tuning("k1order");
        const char* e = es.empty() ? nullptr : es.c_str();
        return (e && std::string(e) == "t") ? 0 : 1;
    }();
    return v;
}

// K4 variant: "gather" (codegen.cpp emit_output_gather; default) or the
// smem-staged kernels (wino_output_flat for m <= 2, banded wino_output_xform
// otherwise; WINO_K4=staged)
bool k4_gather() {
    static const bool v = [] {
        const std::string es = wino::tuning("k4");
        const char* e = es.empty() ? nullptr : es.c_str();
        return !(e && std::string(e) == "staged");
    }();
    return v;
}

// Tensor-core K1 at 16 < P <= 96: the warp-per-channel kernel that parks its 16-bit results in shared
// memory (codegen.cpp input_tcs) for images of more than 32 x 32 pixels; smaller planes keep the
// 4-tiles x 8-channels map, whose eight adjacent channel planes are one contiguous run of x
// (VGG-16 batch 256, tc_bf16: 224^2 2.18 -> 1.62 ms, 112^2 1.17 -> 0.89, 56^2 0.68 -> 0.50, 28^2 equal,
// 14^2 0.100 -> 0.137; tuning key k1tc_staged = 0: off, 2: every size)
bool k1tc_staged(int P, const wino_layer_shape* s) {
    const std::string e = wino::tuning("k1tc_staged");
    if (P <= 16 || P > 96 || e == "0") return false;
    return e == "2" || (long long)s->H * s->W > 32 * 32;
}

// K2 with cooperative weight loads (codegen.cpp wino_filter_coop): filters of 5 x 5 and larger, where the
// per-thread loads are bound by L1 line requests (cfg4 K1 + K2 55.6 -> 46.0 us); its staging buffer is
// static shared memory, so it exists only while 128 (r^2 | 1) input elements fit 48 KB
bool k2_coop(const wino_plan* p) {
    return p->r >= 5 && wino::tuning("k2coop") != "0" &&
           128 * ((p->r * p->r) | 1) * (p->ty.in_double ? 8 : 4) <= 48 * 1024;
}

bool k1_no8() {  // WINO_K1TC=4x8: use the 4-tiles x 8-channels TC kernel also for P <= 16
    static const bool v = [] {
        const std::string es = wino::tuning("k1tc");
        const char* e = es.empty() ? nullptr : es.c_str();
        return e && std::string(e) == "4x8";
    }();
    return v;
}

// Tile-level API: generated straight-line kernels up to alpha = 10 (NVRTC compile
// time grows steeply: ~4 s at alpha 10, ~40 s at 14), the program interpreter
// above that (alpha <= 24) or everywhere with WINO_TILE_INTERP=1.
bool tile_interp(const wino_plan* p) {
    static const int force = [] {
        const std::string e = wino::tuning("tile_interp");
        return e.empty() ? -1 : std::atoi(e.c_str());
    }();
    if (force >= 0) return force > 0 || p->n > 16;
    return p->n > 10;
}

bool k1_gather() {
    static const bool v = [] {
        const std::string es = wino::tuning("k1");
        const char* e = es.empty() ? nullptr : es.c_str();
        return !(e && std::string(e) == "tile");
    }();
    return v;
}

// K1 from shared-memory copies of the image planes (codegen.cpp input_gather_body<true>): f32 inputs,
// planes of a multiple of 16 bytes, and the planes a 128-tile block can touch must fit (several
// blocks per SM).  On by default where it applies (VGG-16 batch 256: 14 x 14 layers 119.5 -> 103.2 us,
// 28 x 28 289 -> 245 us, 56 x 56 494 -> 455 us; single small layers unchanged); tuning key "k1" =
// "gather" turns it off, "bulk<KB>" changes the shared-memory cap.
bool k1_staged(const wino_plan* p, const wino_layer_shape* s, const wino_layer_layout& L, const void* x, int tb,
               unsigned* smem) {
    const std::string e = wino::tuning("k1");
    if (e == "gather" || e == "tile" || p->ty.in_double) return false;
    const long long hw = (long long)s->H * s->W, per = (long long)L.th * L.tw;
    if (hw % 4 || ((uintptr_t)x & 15) || per <= 0) return false;
    const long long planes = ((tb - 1) / per + 2) * wino::gather_cpt(L.P);
    const long long bytes = planes * hw * 4;
    *smem = (unsigned)bytes;
    const long long cap = e.rfind("bulk", 0) == 0 && e.size() > 4 ? std::atoll(e.c_str() + 4) * 1024 : 96 * 1024;
    return bytes <= cap;  // "bulk<KB>" overrides the cap (sweeps)
}

}  // namespace

// ================================================================== C-ABI
extern "C" {

const char* wino_last_error(void) { return wino::g_last_error.c_str(); }

int wino_tuning_set(const char* key, const char* value) {
    static const char* const keys[] = {"gemm", "dbuf", "k1", "k1order", "k4", "k1tc", "tile_interp",
                                       "cpt", "kpt", "tcf_nk", "tcf_dbg", "tc_epi", "k1rowwise", "k4rowwise", "sc2_kg", "k4k1_ks", "k1st_blocks", "k1_blocks", "k4_blocks", "k1tc_staged", "k1tc_blocks", "tc_epw", "k2coop"};
    if (!key) return wino::fail(WINO_EINVAL, "tuning_set: null key");
    bool known = false;
    for (const char* k : keys) known = known || std::strcmp(k, key) == 0;
    if (!known) return wino::fail(WINO_EINVAL, std::string("tuning_set: unknown key '") + key + "'");
    std::lock_guard<std::mutex> g(wino::g_tune_mu);
    if (value && *value) {
        wino::g_tune[key] = value;
    } else {
        wino::g_tune.erase(key);
    }
    return WINO_OK;
}
const char* wino_version(void) { return "libwino 0.1 (sm_100a)"; }
int64_t wino_launch_count(void) { return wino::g_launches.load(); }

int wino_plan_create(int r, int m, int precision, int channel_sum, int contract_mode, const wino_prog* G,
                     const wino_prog* BT, const wino_prog* AT, wino_plan** out) {
    if (!out) return wino::fail(WINO_EINVAL, "plan_create: null out");
    *out = nullptr;
    if (r < 1 || m < 1) return wino::fail(WINO_EINVAL, "kernel and output sizes must be >= 1");
    if (precision < 0 || precision > 2) return wino::fail(WINO_EINVAL, "precision must be fp32, fp64 or mixed");
    if (channel_sum < 0 || channel_sum > 1) return wino::fail(WINO_EINVAL, "channel_sum must be linear or pairwise");
    if (contract_mode < 0 || contract_mode > 5)
        return wino::fail(WINO_EINVAL, "contract mode must be exact, ffma, tc_bf16, tc_fp16, tcf_bf16 or tcf_fp16");
    if (contract_mode >= WINO_CONTRACT_TC_BF16 && precision == WINO_FP64)
        return wino::fail(WINO_EINVAL, "tensor-core contraction needs fp32 or mixed precision");
    const int n = r + m - 1;
    if (n > 24) return wino::fail(WINO_EUNSUPPORTED, "alpha = r + m - 1 > 24 is not supported");
    auto p = std::make_unique<wino_plan>();
    p->r = r;
    p->m = m;
    p->n = n;
    p->precision = precision;
    p->chsum = channel_sum;
    p->mode = contract_mode;
    if (p->fused()) {
        const int P = n * n;
        p->nk = std::min(256, (512 / P) / 16 * 16);
        const std::string e = wino::tuning("tcf_nk");  // smaller blocks (16 x P <= 256: double-buffered TMEM)
        if (!e.empty()) {
            const int v = atoi(e.c_str());
            if (v >= 16 && v % 16 == 0 && v <= p->nk) p->nk = v;
        }
        if (p->nk < 16) return wino::fail(WINO_EUNSUPPORTED, "fused tensor-core mode needs alpha^2 <= 32");
    }
    if (convert_prog(G, &p->G) || convert_prog(BT, &p->BT) || convert_prog(AT, &p->AT))
        return wino::fail(WINO_EINVAL, "malformed program table");
    std::string e = wino::validate(p->G, n, r, "G");
    if (e.empty()) e = wino::validate(p->BT, n, n, "B_T");
    if (e.empty()) e = wino::validate(p->AT, m, n, "A_T");
    if (!e.empty()) return wino::fail(WINO_EINVAL, e);
    const bool dbl64 = precision == WINO_FP64;
    p->ty.compute_double = precision != WINO_FP32;
    p->ty.in_double = dbl64;
    p->ty.uv_double = dbl64;
    p->ty.y_double = precision != WINO_FP32;
    // Tile configs {tm, tn, thm, thn, bk, stages, maxreg, ku, noprod, pack} picked by
    // tools/contract_bench.py sweeps on B200 (profiles/): 4 consumer warps + 1 producer
    // warp per CTA, so three CTAs (15 warps) fit per SM within the per-SMSP register
    // file; float U/V use packed f32x2 arithmetic (FFMA2(a, b, -0) + FADD2 in exact
    // modes: cfg2 27.4 -> 31.1 TFLOP/s, cfg3 m=6 29.1 -> 33.6, pairwise 25.6 -> 27.7).
    if (contract_mode >= WINO_CONTRACT_TC_BF16)
        p->gemm = {8, 8, 16, 16, 32, 3, 0};  // only the 128/128/32 blocking matters (tc_contract.cu)
    else if (dbl64 && channel_sum == WINO_SUM_PAIRWISE)
        p->gemm = {4, 4, 16, 16, 32, 3, 168, 8};  // DMUL/DADD pairwise, 64x64: 12.3 -> 13.1 TFLOP/s (cfg2 shape)
    else if (dbl64)
        p->gemm = {4, 4, 8, 16, 16, 4, 0};       // DMUL/DADD linear: 14.8 TFLOP/s = 84% of the DMUL+DADD ceiling
    else if (channel_sum == WINO_SUM_PAIRWISE)
        // 8 consumer warps, 64x64, 64-channel stages x 2 (VGG-16 layer 6: 30.5 -> 33.0 TFLOP/s vs
        // 32 x 3, tools/probes/vgg_l6_k3_sweep.sh)
        p->gemm = {4, 4, 16, 16, 64, 2, 168, 8, 0, 1};
    else
        p->gemm = {8, 8, 16, 8, 16, 4, 0, 16, 0, 1};
    bool env_gemm = false;
    const std::string tg = wino::tuning("gemm");  // tuning override: tm,tn,thm,thn,bk,stages,maxreg[,ku,noprod,pack,wn]
    if (!tg.empty()) {
        wino::GemmCfg g{};
        const int got = sscanf(tg.c_str(), "%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d", &g.tm, &g.tn, &g.thm, &g.thn, &g.bk,
                               &g.stages, &g.maxreg, &g.ku, &g.noprod, &g.pack, &g.wn);
        const bool wn_ok = g.wn == 0 || (g.wn > 0 && 32 % g.wn == 0 && g.thn % g.wn == 0 && g.thm % (32 / g.wn) == 0);
        // the pairwise in-stage counter (contract_template.cuh) covers stages of 8, 16, 32 or 64 channels
        const bool bk_ok = channel_sum != WINO_SUM_PAIRWISE || g.bk == 8 || g.bk == 16 || g.bk == 32 || g.bk == 64;
        if (got < 7 || g.bk % 8 || g.tm % 4 || g.tn % 4 || (g.ku != 0 && g.bk % g.ku) || !bk_ok || !wn_ok ||
            g.noprod < 0 || g.noprod > 1 || (g.thm * g.thn) % 32)
            return wino::fail(WINO_EINVAL, "tuning gemm: bad tile config '" + tg + "'");
        p->gemm = g;
        env_gemm = true;
    }
    p->cands = {p->gemm};
    if (!env_gemm && contract_mode < WINO_CONTRACT_TC_BF16 && !dbl64 && channel_sum != WINO_SUM_PAIRWISE) {
        // same 8x8 microtile transposed (64 filters x 128 tiles) and a 4x8 microtile
        // (64 x 64): small K or T layers pad less and fill the persistent wave better
        p->cands.push_back({8, 8, 8, 16, 16, 4, 0, 16, 0, 1});
        p->cands.push_back({4, 8, 16, 8, 16, 4, 0, 16, 0, 1});
        p->cands.push_back({4, 4, 16, 8, 16, 4, 0, 16, 0, 1});  // 64 x 32 (4x4): small layers (cfg1 20.4 -> 22.3)
        p->cands.push_back({8, 8, 16, 8, 8, 4, 0, 8, 0, 1});  // C <= 8 (first layers): 8-channel stages
    } else if (!env_gemm && contract_mode < WINO_CONTRACT_TC_BF16 && !dbl64) {
        // pairwise, C <= 8: 4x8 microtiles, 64 x 128 tiles (VGG-16 layer 1, M-store bound:
        // 1.57 -> 1.24 ms vs 4x4 / 64 x 64, tools/probes/layer1_k3_sweep.sh)
        p->cands.push_back({4, 8, 16, 16, 8, 4, 168, 8, 0, 1});
        // C not a multiple of 64: 32-channel stages pad less
        p->cands.push_back({4, 4, 16, 16, 32, 3, 168, 8, 0, 1});
    }
    if (!env_gemm && contract_mode < WINO_CONTRACT_TC_BF16 && precision == WINO_FP32 && n * n <= 16) {
        // fused exact K3 + K4 (wino_conv2d_fused): 64 x 64 tile, 8 consumer warps x 4x4 microtile,
        // alpha^2 x 16 accumulators per thread parked in tensor memory (contract_template.cuh)
        p->fused_ci = (int)p->cands.size();
        // (the linear sum uses the pairwise kernel's pipeline shape too: 64-channel stages x 2,
        // 8-step unrolled blocks with the explicit fragment double buffer)
        p->cands.push_back({4, 4, 16, 16, 64, 2, 168, 8, 0, 1});
    }
    const std::string tag = "r" + std::to_string(r) + "m" + std::to_string(m) + "p" + std::to_string(precision);
    p->layer.name = "wino_layer_" + tag + ".cu";
    p->layer.source = contract_mode >= WINO_CONTRACT_TC_BF16
                          ? wino::gen_layer_source_tc(r, m, p->G, p->BT, p->AT, p->ty,
                                                      contract_mode == WINO_CONTRACT_TC_FP16 ||
                                                          contract_mode == WINO_CONTRACT_TCF_FP16,
                                                      p->nk)
                          : wino::gen_layer_source(r, m, p->G, p->BT, p->AT, p->ty, p->gemm.bm(), p->gemm.bn());
    p->tile.name = "wino_tile_" + tag + ".cu";
    p->tile.source = wino::gen_tile_source(r, m, p->G, p->BT, p->AT, p->ty);
    // modules are compiled on first use: the tile-level path (measure_error) never
    // needs the layer kernels, whose straight-line code for large alpha takes
    // NVRTC minutes
    *out = p.release();
    return WINO_OK;
}

void wino_plan_destroy(wino_plan* plan) { delete plan; }  // modules unload with their context

int wino_plan_source(const wino_plan* plan, int which, char* buf, size_t cap, size_t* len) {
    if (!plan || (which != 0 && which != 1)) return wino::fail(WINO_EINVAL, "plan_source: bad arguments");
    const std::string& s = which == 0 ? plan->layer.source : plan->tile.source;
    if (len) *len = s.size();
    if (buf && cap) {
        const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(buf, s.data(), k);
        buf[k] = '\0';
    }
    return WINO_OK;
}

int wino_plan_cubin(wino_plan* plan, int which, int channels, void* buf, size_t cap, size_t* len) {
    if (!plan || which < 0 || which > 3) return wino::fail(WINO_EINVAL, "plan_cubin: bad arguments");
    if (which == 3 && plan->fused_ci < 0) return wino::fail(WINO_EUNSUPPORTED, "plan_cubin: no fused exact kernel for this plan");
    wino::Module* mod = which == 0 ? &plan->layer
                        : which == 1 ? &plan->tile
                        : which == 2 ? plan->contract_module(round_up(channels > 0 ? channels : 1, plan->gemm.bk))
                                     : plan->contract_module(round_up(channels > 0 ? channels : 1,
                                                                      plan->cands[plan->fused_ci].bk),
                                                             plan->fused_ci, true);
    const wino::Compiled* bin = nullptr;
    int rc = mod->ensure_compiled("*", &bin);
    if (rc) return rc;
    if (len) *len = bin->cubin.size();
    if (buf && cap >= bin->cubin.size()) std::memcpy(buf, bin->cubin.data(), bin->cubin.size());
    return WINO_OK;
}

// codegen.cpp emit_smallc2 (C <= 4): CTA = the bn tiles of one V block x all filters, threads = bn * KG
static int smallc2_kg() {
    const int v = std::atoi(wino::tuning("sc2_kg").c_str());
    return v >= 1 && v <= 8 ? v : 2;
}
static size_t smallc2_smem(const wino_layer_layout& L, int C, int m) {
    // sU[P][Kp/bm][C][bm] + sV[P][C][bn] + (even m) one m x 32 x m/2 float2 store buffer per warp
    const size_t wbuf = m % 2 == 0 ? (size_t)(L.bn * smallc2_kg() / 32) * m * 32 * (m / 2) * 8 : 0;
    return ((size_t)L.P * L.Kp * C + (size_t)L.P * C * L.bn) * 4 + wbuf;
}
static bool smallc2_ok(const wino_layer_layout& L, int C, int m) {
    return C <= 4 && L.bn % 32 == 0 && L.bm % 4 == 0 && L.bn * smallc2_kg() <= 1024 &&
           smallc2_smem(L, C, m) <= 232448 - 1024;
}

static bool smallc_v2(wino_plan* plan, const wino_layer_shape* s) {
    wino_layer_layout L;
    return !layout_of(plan, s, &L) && smallc2_ok(L, s->C, plan->m);
}

int wino_plan_prepare(wino_plan* plan, const wino_layer_shape* s, int flags) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->mode >= WINO_CONTRACT_TC_BF16) return WINO_OK;  // tensor-core plans compile on first use
    const int ci = plan->pick(s);
    wino::Module* lm = plan->layer_mod(ci);
    std::vector<std::pair<wino::Module*, std::string>> work;
    int smem = 0;
    const int tb = xform_block(plan, &smem);
    const long long n_tb = (L.Tp + tb - 1) / tb, n_kb = (L.Kp + tb - 1) / tb;
    if (flags & WINO_PREPARE_CONV) {
        work.push_back({lm, k1_gather() && n_tb + n_kb <= 65535 && L.Cp <= 65535 ? "wino_transforms_gather"
                                                                                  : "wino_transforms"});
        if (k2_coop(plan) && k1_gather() && L.Cp <= 65535) {  // r >= 5: K2 and K1 are two launches
            work.push_back({lm, "wino_filter_coop"});
            work.push_back({lm, "wino_input_gather"});
        }
        work.push_back({plan->contract_module(L.Cp, ci), "wino_contract"});
        work.push_back({lm, k4_gather() && s->K <= 65535 ? "wino_output_gather"
                            : plan->m <= 2               ? "wino_output_flat"
                                                         : "wino_output_xform"});
    }
    if ((flags & WINO_PREPARE_ACT) && !plan->ty.y_double) work.push_back({lm, "wino_output_gather_act"});
    if ((flags & WINO_PREPARE_K4K1) && plan->precision == WINO_FP32 && plan->mode < WINO_CONTRACT_TC_BF16) {
        work.push_back({lm, "wino_k4k1"});       // as the SECOND layer of wino_output_input_transform
        work.push_back({lm, "wino_filter_xform"});
    }
    if ((flags & WINO_PREPARE_ACT) && wino_smallc_supported(plan, s)) {
        const std::string suf = std::to_string(s->C) + (plan->chsum == WINO_SUM_PAIRWISE ? "p" : "l");
        if (smallc_v2(plan, s)) {  // one kernel per store mode; the ReLU-only one is what a first layer uses
            work.push_back({lm, "wino_smallc2_c" + suf + "_m1"});
        } else {
            work.push_back({lm, "wino_smallc_c" + suf});
        }
    }
    if (flags & WINO_PREPARE_NHWC) {
        work.push_back({lm, "wino_filter_xform"});
        work.push_back({lm, "wino_input_gather_nhwc"});
        work.push_back({plan->contract_module(L.Cp, ci), "wino_contract"});
        work.push_back({lm, "wino_output_gather_nhwc"});
    }
    if (flags & WINO_PREPARE_STAGES) {
        work.push_back({lm, "wino_filter_xform"});
        work.push_back({lm, k1_gather() && n_tb <= 65535 && L.Cp <= 65535 ? "wino_input_gather" : "wino_input_xform"});
    }
    return wino::compile_all(work);
}

int wino_layer_layout_query(const wino_plan* plan, const wino_layer_shape* s, wino_layer_layout* out) {
    return layout_of(plan, s, out);
}

int wino_filter_transform(wino_plan* plan, const wino_layer_shape* s, const void* w, void* U, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    CUfunction f;
    int K = s->K, C = s->C;
    long long Kp = L.Kp, Cp = L.Cp;
    u_layout_record(U, L);
    if (plan->mode >= WINO_CONTRACT_TC_BF16 && (k1_gather() || plan->fused()) && Cp / 8 <= 65535) {
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_filter_tcg", &f))) return rc;
        void* args[] = {(void*)&w, &U, &K, &C, &Kp, &Cp};
        return wino::launch(f, dim3(cdiv(Kp, 32), (unsigned)(Cp / 8), 1), dim3(256), 0, stream, args,
                            "filter_transform");
    }
    if (plan->fused()) return wino::fail(WINO_EUNSUPPORTED, "filter_transform: grid too large for the fused layout");
    if (plan->mode < WINO_CONTRACT_TC_BF16 && k2_coop(plan) && Cp <= 65535) {
        // large filters: cooperative weight loads through shared memory (codegen.cpp wino_filter_coop)
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_filter_coop", &f))) return rc;
        void* args[] = {(void*)&w, &U, &K, &C, &Kp, &Cp};
        return wino::launch(f, dim3((unsigned)cdiv(Kp, 128), (unsigned)Cp, 1), dim3(128), 0, stream, args,
                            "filter_transform");
    }
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_filter_xform", &f))) return rc;
    int smem = 0;
    const int tb = plan->mode >= WINO_CONTRACT_TC_BF16 ? 64 : xform_block(plan, &smem);
    void* args[] = {(void*)&w, &U, &K, &C, &Kp, &Cp};
    return wino::launch(f, dim3(cdiv(Kp, tb), (unsigned)Cp, 1), dim3(tb), 0, stream, args, "filter_transform");
}

static int transforms_impl(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* U, void* V,
                           void* stream, bool skip_pad);

int wino_transforms(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* U, void* V,
                    void* stream) {
    return transforms_impl(plan, s, x, w, U, V, stream, false);
}

int wino_transforms_smallc(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* U, void* V,
                           void* stream) {
    if (wino_smallc_supported(plan, s) != 2)
        return wino::fail(WINO_EUNSUPPORTED, "transforms_smallc: the fast small-C kernel does not apply to this shape");
    return transforms_impl(plan, s, x, w, U, V, stream, true);
}

static int transforms_impl(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* U, void* V,
                           void* stream, bool skip_pad) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if ((uintptr_t)V & 15) return wino::fail(WINO_EINVAL, "transforms: V must be 16-byte aligned");
    u_layout_record(U, L);
    CUfunction f;
    int C = s->C, H = s->H, W = s->W, pad = s->pad, th = L.th, tw = L.tw, K = s->K;
    long long T = L.T, Tp = L.Tp, Cp = L.Cp, Kp = L.Kp;
    int smem = 0;
    const bool tc = plan->mode >= WINO_CONTRACT_TC_BF16;
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_transforms", &f))) return rc;
    const int tb = tc ? 64 : xform_block(plan, &smem);
    if (tc) smem = L.P * 64 * 8 * 2;
    int n_tb = (int)cdiv(Tp, tb), n_kb = (int)cdiv(Kp, tb);
    const long long blocks = (long long)n_tb * (tc ? Cp / 8 : Cp) + (long long)n_kb * Cp;
    if (blocks >= (1LL << 31)) return wino::fail(WINO_EUNSUPPORTED, "transforms: grid too large");
    int cfast = k1_cfast(), Wl = skip_pad ? 1 : 0;  // gather kernels: 1 = leave V's padded channel rows unwritten
    if (tc && (k1_gather() || plan->fused()) && Cp / 8 <= 65535 && L.P <= 16 && !k1_no8()) {
        CUfunction fg;
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_transforms_tcg8", &fg))) return rc;
        float rtw = 1.0f / tw, rth = 1.0f / th;
        int nt128 = (int)cdiv(Tp, 128), nk16 = (int)cdiv(Kp, 16);
        void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &nt128, (void*)&w, &U, &K, &Kp,
                        &rtw, &rth};
        return wino::launch(fg, dim3((unsigned)(nt128 + nk16), (unsigned)(Cp / 8)), dim3(128), 0, stream, args,
                            "transforms");
    }
    if (tc && (k1_gather() || plan->fused()) && Cp / 8 <= 65535) {
        CUfunction fg;
        if ((rc = plan->layer_mod(plan->pick(s))->function(k1tc_staged(L.P, s) ? "wino_transforms_tcs" : "wino_transforms_tcg",
                                                           &fg)))
            return rc;
        float rtw = 1.0f / tw, rth = 1.0f / th;
        int nt32 = (int)cdiv(Tp, 32), nk32 = (int)cdiv(Kp, 32);
        void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &nt32, (void*)&w, &U, &K, &Kp,
                        &rtw, &rth};
        return wino::launch(fg, dim3((unsigned)(nt32 + nk32), (unsigned)(Cp / 8)), dim3(256), 0, stream, args,
                            "transforms");
    }
    if (!tc && k1_gather() && (long long)n_tb + n_kb <= 65535 && Cp <= 65535) {
        CUfunction fg;
        unsigned st_smem = 0;
        const bool st = k1_staged(plan, s, L, x, tb, &st_smem);
        float rtw = 1.0f / tw, rth = 1.0f / th;
        if (k2_coop(plan) && Cp <= 65535) {
            // large filters: K2 as its own kernel with cooperative weight loads (codegen.cpp wino_filter_coop:
            // cfg4 K2 35 -> see profiles/r2_experiments.md), then K1 alone
            CUfunction fk;
            if ((rc = plan->layer_mod(plan->pick(s))->function("wino_filter_coop", &fk))) return rc;
            void* kargs[] = {(void*)&w, &U, &K, &C, &Kp, &Cp};
            if ((rc = wino::launch(fk, dim3((unsigned)cdiv(Kp, 128), (unsigned)Cp), dim3(128), 0, stream, kargs,
                                   "filter_transform")))
                return rc;
            if ((rc = plan->layer_mod(plan->pick(s))->function(st ? "wino_input_gather_st" : "wino_input_gather", &fg)))
                return rc;
            void* iargs[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &Wl, &rtw, &rth};
            return wino::launch(fg, dim3((unsigned)(Cp / wino::gather_cpt(L.P)), (unsigned)n_tb), dim3(tb),
                                st ? st_smem : 0, stream, iargs, "input_transform");
        }
        if ((rc = plan->layer_mod(plan->pick(s))->function(st ? "wino_transforms_gather_st" : "wino_transforms_gather",
                                                           &fg)))
            return rc;
        void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &n_tb, (void*)&w, &U, &K, &Kp,
                        &Wl, &rtw, &rth};
        return wino::launch(fg, dim3((unsigned)(Cp / wino::gather_cpt(L.P)), (unsigned)(n_tb + n_kb)), dim3(tb),
                            st ? st_smem : 0, stream, args, "transforms");
    }
    if (plan->fused()) return wino::fail(WINO_EUNSUPPORTED, "transforms: grid too large for the fused layout");
    void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &n_tb, (void*)&w, &U, &K, &Kp, &n_kb, &cfast};
    return wino::launch(f, dim3((unsigned)blocks, 1, 1), dim3(tb), (unsigned)smem, stream, args, "transforms");
}

int wino_input_transform(wino_plan* plan, const wino_layer_shape* s, const void* x, void* V, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if ((uintptr_t)V & 15) return wino::fail(WINO_EINVAL, "input_transform: V must be 16-byte aligned");
    CUfunction f;
    int C = s->C, H = s->H, W = s->W, pad = s->pad, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Cp = L.Cp;
    int smem = 0;
    if (plan->mode < WINO_CONTRACT_TC_BF16 && k1_gather()) {
        const int tb = xform_block(plan, &smem);
        int Wl = 0, n_tb = (int)cdiv(Tp, tb);
        if (n_tb <= 65535 && Cp <= 65535) {
            unsigned st_smem = 0;
            const bool st = k1_staged(plan, s, L, x, tb, &st_smem);
            if ((rc = plan->layer_mod(plan->pick(s))->function(st ? "wino_input_gather_st" : "wino_input_gather", &f)))
                return rc;
            float rtw = 1.0f / tw, rth = 1.0f / th;
            void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &Wl, &rtw, &rth};
            return wino::launch(f, dim3((unsigned)(Cp / wino::gather_cpt(L.P)), (unsigned)n_tb), dim3(tb),
                                st ? st_smem : 0, stream, args, "input_transform");
        }
    }
    if (plan->mode >= WINO_CONTRACT_TC_BF16 && (k1_gather() || plan->fused()) && Cp / 8 <= 65535 && L.P <= 16 &&
        !k1_no8()) {
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_input_tcg8", &f))) return rc;
        float rtw = 1.0f / tw, rth = 1.0f / th;
        void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &rtw, &rth};
        return wino::launch(f, dim3((unsigned)cdiv(Tp, 128), (unsigned)(Cp / 8)), dim3(128), 0, stream, args,
                            "input_transform");
    }
    if (plan->mode >= WINO_CONTRACT_TC_BF16 && (k1_gather() || plan->fused()) && Cp / 8 <= 65535) {
        if ((rc = plan->layer_mod(plan->pick(s))->function(k1tc_staged(L.P, s) ? "wino_input_tcs" : "wino_input_tcg", &f)))
            return rc;
        float rtw = 1.0f / tw, rth = 1.0f / th;
        void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp, &rtw, &rth};
        return wino::launch(f, dim3((unsigned)cdiv(Tp, 32), (unsigned)(Cp / 8)), dim3(256), 0, stream, args,
                            "input_transform");
    }
    if (plan->fused()) return wino::fail(WINO_EUNSUPPORTED, "input_transform: grid too large for the fused layout");
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_input_xform", &f))) return rc;
    void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp};
    if (plan->mode >= WINO_CONTRACT_TC_BF16)
        return wino::launch(f, dim3(cdiv(Tp, 64), (unsigned)(Cp / 8), 1), dim3(64), (unsigned)(L.P * 64 * 16),
                            stream, args, "input_transform");
    const int tb = xform_block(plan, &smem);
    return wino::launch(f, dim3(cdiv(Tp, tb), (unsigned)Cp, 1), dim3(tb), (unsigned)smem, stream, args,
                        "input_transform");
}

int wino_contract(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V, void* M, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (((uintptr_t)U | (uintptr_t)V | (uintptr_t)M) & 15)
        return wino::fail(WINO_EINVAL, "contract: U, V, M must be 16-byte aligned");
    if ((rc = u_layout_check(U, L, "contract"))) return rc;
    if (plan->fused())
        return wino::fail(WINO_EINVAL, "contract: fused tensor-core plan has no M; use wino_contract_output");
    if (plan->mode >= WINO_CONTRACT_TC_BF16)
        return wino::tc_contract_launch(U, V, M, L.Kp, L.Tp, L.Cp, L.P, plan->mode == WINO_CONTRACT_TC_FP16,
                                        s->K, stream);
    const int ci = plan->pick(s);
    wino::Module* mod = plan->contract_module(L.Cp, ci);
    CUfunction f;
    if ((rc = mod->function("wino_contract", &f))) return rc;
    const wino::GemmCfg& g = plan->cands.empty() ? plan->gemm : plan->cands[ci];
    long long Kp = L.Kp, Tp = L.Tp, Cp = L.Cp;
    const long long tiles = (long long)L.P * (Kp / g.bm()) * (Tp / g.bn());
    if (tiles > (1LL << 30)) return wino::fail(WINO_EUNSUPPORTED, "contract: too many tiles");
    int n_tiles = (int)tiles;
    int levels = 1;  // must match contract_module()
    while ((1LL << levels) <= Cp / g.bk) ++levels;
    if (plan->chsum != WINO_SUM_PAIRWISE) levels = 0;
    bool slots_smem = false;
    const unsigned smem = (unsigned)g.smem_bytes(levels, L.elem_bytes_uv, &slots_smem);
    const int threads = g.block();
    // persistent grid: as many CTAs as can be co-resident (one wave), each walks tiles
    int per_sm = 0, sms = 0, dev = 0;
    if (smem > 48 * 1024) {
        CUresult cr = wino::driver().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
        if (cr != CUDA_SUCCESS) return wino::fail(WINO_ECUDA, "contract: set smem: " + wino::cu_err(cr));
    }
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (wino::driver().OccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem) != CUDA_SUCCESS ||
        per_sm < 1)
        per_sm = 1;
    const long long grid = std::min<long long>(tiles, (long long)per_sm * (sms > 0 ? sms : 148));
    unsigned long long nz2 = 0x8000000080000000ull;  // (-0, -0): exact packed products (contract_template.cuh)
    void* args[] = {(void*)&U, (void*)&V, &M, &Kp, &Tp, &Cp, &n_tiles, &nz2};
    return wino::launch(f, dim3((unsigned)grid, 1, 1), dim3(threads), smem, stream, args, "contract");
}

int wino_output_transform_act(wino_plan* plan, const wino_layer_shape* s, const void* M, void* act, int pool,
                              void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->fused() || plan->ty.y_double)
        return wino::fail(WINO_EUNSUPPORTED, "output_transform_act: plans with an fp32 M and an fp32 y only");
    if (pool != 0 && pool != 1) return wino::fail(WINO_EINVAL, "output_transform_act: pool must be 0 or 1");
    if (pool && (plan->m & 1)) return wino::fail(WINO_EUNSUPPORTED, "output_transform_act: pooling needs an even m");
    if (s->K > 65535) return wino::fail(WINO_EUNSUPPORTED, "output_transform_act: K > 65535");
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_output_gather_act", &f))) return rc;
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Kp = L.Kp;
    float rtw = 1.0f / tw, rth = 1.0f / th;
    void* args[] = {(void*)&M, &act, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &rtw, &rth, &pool};
    return wino::launch(f, dim3(cdiv(T, 128), (unsigned)K, 1), dim3(128), 0, stream, args, "output_transform_act");
}

// K4 of layer `s` + activation + K1 of layer `s2` in one kernel (codegen.cpp emit_k4k1)
static int k4k1_geometry(wino_plan* plan, const wino_layer_shape* s, int pool, const wino_layer_shape* s2,
                         wino_layer_layout* L, wino_layer_layout* L2, int* PL, unsigned* smem) {
    int rc;
    if (!plan || !s || !s2) return wino::fail(WINO_EINVAL, "output_input_transform: null argument");
    if ((rc = layout_of(plan, s, L)) || (rc = layout_of(plan, s2, L2))) return rc;
    if (plan->mode >= WINO_CONTRACT_TC_BF16 || plan->precision != WINO_FP32)
        return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: fp32 plans with an FP32 contraction only");
    if (pool != 0 && pool != 1) return wino::fail(WINO_EINVAL, "output_input_transform: pool must be 0 or 1");
    if (pool && (plan->m & 1)) return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: pooling needs an even m");
    const int H2 = pool ? L->Ho / 2 : L->Ho, W2 = pool ? L->Wo / 2 : L->Wo;
    if (s2->N != s->N || s2->C != s->K || s2->H != H2 || s2->W != W2)
        return wino::fail(WINO_EINVAL, "output_input_transform: the second layer does not take the first one's activation");
    if (L2->Cp != s2->C)  // padded channels of V are K1's job
        return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: the second layer's channels are padded");
    if (s->K > 65535) return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: K > 65535");
    const long long per1 = (long long)L->th * L->tw, hw2 = (long long)H2 * W2;
    *PL = (int)std::max(1LL, 128 / per1);
    const long long bytes = (long long)*PL * hw2 * 4;
    if (hw2 <= 0 || bytes > 200 * 1024) return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: plane too large for shared memory");
    *smem = (unsigned)bytes;
    return WINO_OK;
}

int wino_output_input_supported(wino_plan* plan, const wino_layer_shape* s, int pool, const wino_layer_shape* s2) {
    wino_layer_layout L, L2;
    int PL;
    unsigned smem;
    return k4k1_geometry(plan, s, pool, s2, &L, &L2, &PL, &smem) == WINO_OK ? 1 : 0;
}

int wino_output_input_transform(wino_plan* plan, const wino_layer_shape* s, const void* M, int pool,
                                const wino_layer_shape* s2, void* V2, void* stream) {
    wino_layer_layout L, L2;
    int PL, rc;
    unsigned smem;
    if ((rc = k4k1_geometry(plan, s, pool, s2, &L, &L2, &PL, &smem))) return rc;
    if ((uintptr_t)V2 & 15) return wino::fail(WINO_EINVAL, "output_input_transform: V must be 16-byte aligned");
    if (s->N == 0) return WINO_OK;
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s2))->function("wino_k4k1", &f))) return rc;
    int N = s->N, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw, H2 = s2->H, W2 = s2->W, pad2 = s2->pad, th2 = L2.th,
        tw2 = L2.tw;
    long long Tp = L.Tp, Kp = L.Kp, T2 = L2.T, Tp2 = L2.Tp, Cp2 = L2.Cp;
    int K = s->K, G = (int)cdiv(N, PL), KS = 8;
    const std::string ks = wino::tuning("k4k1_ks");
    if (!ks.empty() && std::atoi(ks.c_str()) > 0) KS = std::atoi(ks.c_str());
    const long long blocks = (long long)G * cdiv(K, KS) * KS;
    if (blocks >= (1LL << 31)) return wino::fail(WINO_EUNSUPPORTED, "output_input_transform: grid too large");
    void* args[] = {(void*)&M, &V2, &N, &PL, &pool, &K, &G, &KS, &Ho, &Wo, &th, &tw, &Tp, &Kp,
                    &H2, &W2, &pad2, &th2, &tw2, &T2, &Tp2, &Cp2};
    return wino::launch(f, dim3((unsigned)blocks, 1, 1), dim3(128), smem, stream, args, "output_input_transform");
}

int wino_output_transform(wino_plan* plan, const wino_layer_shape* s, const void* M, void* y, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->fused())
        return wino::fail(WINO_EINVAL, "output_transform: fused tensor-core plan has no M; use wino_contract_output");
    CUfunction f;
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Kp = L.Kp;
    if (k4_gather() && K <= 65535) {
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_output_gather", &f))) return rc;
        float rtw = 1.0f / tw, rth = 1.0f / th;
        void* gargs[] = {(void*)&M, &y, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &rtw, &rth};
        return wino::launch(f, dim3(cdiv(T, 128), cdiv(K, wino::gather_kpt()), 1), dim3(128), 0, stream, gargs,
                            "output_transform");
    }
    if (plan->m <= 2) {
        // small output blocks: one thread per (k, tile), M staged per 128 tiles,
        // per-thread m x m stores (rows of m <= 2 values)
        if ((rc = plan->layer_mod(plan->pick(s))->function("wino_output_flat", &f))) return rc;
        int smem = 0;
        const int tb = xform_block(plan, &smem);
        void* fargs[] = {(void*)&M, &y, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp};
        return wino::launch(f, dim3(cdiv(T, tb), (unsigned)K, 1), dim3(tb), (unsigned)smem, stream, fargs,
                            "output_transform");
    }
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_output_xform", &f))) return rc;
    // block = R tile rows of one image x KB output channels (~256 tiles), output
    // band staged in smem (<= 96 KB)
    const int es = L.elem_bytes_y, m = plan->m;
    int R = th * tw <= 256 ? th : (256 / tw > 0 ? 256 / tw : 1);
    int KB = th * tw <= 256 ? std::max(1, std::min(K, 256 / (th * tw))) : 1;
    auto smem_of = [&](int kb, int rr) { return (long long)kb * rr * m * Wo * es; };
    while (KB > 1 && smem_of(KB, R) > 96 * 1024) --KB;
    while (R > 1 && smem_of(KB, R) > 96 * 1024) --R;
    if (smem_of(KB, R) > 200 * 1024) return wino::fail(WINO_EUNSUPPORTED, "output_transform: image too wide");
    const int nbands = (th + R - 1) / R;
    const unsigned smem = (unsigned)smem_of(KB, R);
    void* args[] = {(void*)&M, &y, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &R, &KB};
    if (s->N > 65535) return wino::fail(WINO_EUNSUPPORTED, "output_transform: N > 65535");
    return wino::launch(f, dim3((unsigned)nbands, (unsigned)((K + KB - 1) / KB), (unsigned)s->N), dim3(128), smem,
                        stream, args, "output_transform");
}

int wino_conv2d(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* y, void* workspace,
                size_t workspace_bytes, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (s->N == 0) return WINO_OK;
    if (!workspace || workspace_bytes < L.workspace_bytes || ((uintptr_t)workspace & 255))
        return wino::fail(WINO_EINVAL, "conv2d: workspace missing, too small or not 256-byte aligned");
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    char* U = (char*)workspace;
    char* V = U + al(L.u_bytes);
    char* M = V + al(L.v_bytes);
    if ((rc = wino_transforms(plan, s, x, w, U, V, stream))) return rc;
    if (plan->fused()) return wino_contract_output(plan, s, U, V, y, stream);
    if ((rc = wino_contract(plan, s, U, V, M, stream))) return rc;
    return wino_output_transform(plan, s, M, y, stream);
}

int wino_input_transform_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* x, void* V, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->mode >= WINO_CONTRACT_TC_BF16)
        return wino::fail(WINO_EUNSUPPORTED, "input_transform_nhwc: FP32-pipe contraction modes only");
    if ((uintptr_t)V & 15) return wino::fail(WINO_EINVAL, "input_transform_nhwc: V must be 16-byte aligned");
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_input_gather_nhwc", &f))) return rc;
    int C = s->C, H = s->H, W = s->W, pad = s->pad, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Cp = L.Cp;
    if (cdiv(Cp, 16) > 65535) return wino::fail(WINO_EUNSUPPORTED, "input_transform_nhwc: too many channels");
    void* args[] = {(void*)&x, &V, &C, &H, &W, &pad, &th, &tw, &T, &Tp, &Cp};
    // block = 8 tiles x 16 channels (codegen.cpp emit_nhwc)
    return wino::launch(f, dim3(cdiv(Tp, 8), cdiv(Cp, 16), 1), dim3(128), 0, stream, args, "input_transform_nhwc");
}

int wino_output_transform_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* M, void* y, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->mode >= WINO_CONTRACT_TC_BF16)
        return wino::fail(WINO_EUNSUPPORTED, "output_transform_nhwc: FP32-pipe contraction modes only");
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_output_gather_nhwc", &f))) return rc;
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Kp = L.Kp;
    if (cdiv(K, 16) > 65535) return wino::fail(WINO_EUNSUPPORTED, "output_transform_nhwc: too many filters");
    void* args[] = {(void*)&M, &y, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp};
    return wino::launch(f, dim3(cdiv(T, 8), cdiv(K, 16), 1), dim3(128), 0, stream, args, "output_transform_nhwc");
}

int wino_conv2d_nhwc(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* y,
                     void* workspace, size_t workspace_bytes, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (plan->mode >= WINO_CONTRACT_TC_BF16)
        return wino::fail(WINO_EUNSUPPORTED, "conv2d_nhwc: FP32-pipe contraction modes only");
    if (s->N == 0) return WINO_OK;
    if (!workspace || workspace_bytes < L.workspace_bytes || ((uintptr_t)workspace & 255))
        return wino::fail(WINO_EINVAL, "conv2d_nhwc: workspace missing, too small or not 256-byte aligned");
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    char* U = (char*)workspace;
    char* V = U + al(L.u_bytes);
    char* M = V + al(L.v_bytes);
    if ((rc = wino_filter_transform(plan, s, w, U, stream))) return rc;
    if ((rc = wino_input_transform_nhwc(plan, s, x, V, stream))) return rc;
    if ((rc = wino_contract(plan, s, U, V, M, stream))) return rc;
    return wino_output_transform_nhwc(plan, s, M, y, stream);
}

int wino_fused_supported(wino_plan* plan, const wino_layer_shape* s) {
    wino_layer_layout L;
    if (!plan || !s || plan->fused_ci < 0) return 0;
    ForceCand guard(plan->fused_ci);
    if (layout_of(plan, s, &L)) return 0;
    const long long groups = (L.Kp / L.bm) * (L.Tp / L.bn);
    return groups > 0 && groups * L.P < (1LL << 30);
}

int wino_fused_workspace(wino_plan* plan, const wino_layer_shape* s, size_t* bytes) {
    if (!bytes) return wino::fail(WINO_EINVAL, "fused_workspace: null bytes");
    if (!wino_fused_supported(plan, s))
        return wino::fail(WINO_EUNSUPPORTED, "fused: needs an fp32 plan with an FP32-pipe contraction and alpha^2 <= 16");
    ForceCand guard(plan->fused_ci);
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    *bytes = al(L.u_bytes) + al(L.v_bytes);
    return WINO_OK;
}

int wino_conv2d_fused(wino_plan* plan, const wino_layer_shape* s, const void* x, const void* w, void* out, int mode,
                      void* workspace, size_t workspace_bytes, void* stream) {
    if (!wino_fused_supported(plan, s))
        return wino::fail(WINO_EUNSUPPORTED, "conv2d_fused: needs an fp32 plan with an FP32-pipe contraction and alpha^2 <= 16");
    if (mode < 0 || mode > 2) return wino::fail(WINO_EINVAL, "conv2d_fused: mode must be 0 (y), 1 (ReLU) or 2 (ReLU + 2x2 max-pool)");
    if (mode == 2 && (plan->m & 1)) return wino::fail(WINO_EUNSUPPORTED, "conv2d_fused: pooling needs an even m");
    ForceCand guard(plan->fused_ci);  // transforms and layout follow the fused kernel's 64 x 64 blocking
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (s->N == 0) return WINO_OK;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    if (!workspace || workspace_bytes < al(L.u_bytes) + al(L.v_bytes) || ((uintptr_t)workspace & 255))
        return wino::fail(WINO_EINVAL, "conv2d_fused: workspace missing, too small or not 256-byte aligned");
    char* U = (char*)workspace;
    char* V = U + al(L.u_bytes);
    if ((rc = wino_transforms(plan, s, x, w, U, V, stream))) return rc;
    const int ci = plan->fused_ci;
    const wino::GemmCfg& g = plan->cands[ci];
    wino::Module* mod = plan->contract_module(L.Cp, ci, true);
    CUfunction f;
    if ((rc = mod->function("wino_contract", &f))) return rc;
    long long Kp = L.Kp, Tp = L.Tp, Cp = L.Cp, T = L.T;
    const long long groups = (Kp / g.bm()) * (Tp / g.bn());
    int n_tiles = (int)(groups * L.P);
    int levels = 1;
    while ((1LL << levels) <= Cp / g.bk) ++levels;
    if (plan->chsum != WINO_SUM_PAIRWISE) levels = 0;
    bool slots_smem = false;
    unsigned smem = (unsigned)g.smem_bytes(levels, 4, &slots_smem);
    // the CTA owns all 512 TMEM columns of its SM: ask for more than half of the shared memory so
    // that no second CTA of this kernel can become co-resident (and block in tcgen05.alloc)
    if (smem < 120 * 1024) smem = 120 * 1024;
    CUresult cr = wino::driver().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
    if (cr != CUDA_SUCCESS) return wino::fail(WINO_ECUDA, "conv2d_fused: set smem: " + wino::cu_err(cr));
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long grid = std::min<long long>(groups, sms > 0 ? sms : 148);
    unsigned long long nz2 = 0x8000000080000000ull;
    void* M = nullptr;
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw;
    const void* Uc = U;
    const void* Vc = V;
    void* args[] = {(void*)&Uc, (void*)&Vc, &M, &Kp, &Tp, &Cp, &n_tiles, &nz2, &out, &K, &Ho, &Wo, &th, &tw, &T, &mode};
    return wino::launch(f, dim3((unsigned)grid, 1, 1), dim3(g.block()), smem, stream, args, "conv2d_fused");
}

int wino_smallc_supported(wino_plan* plan, const wino_layer_shape* s) {
    wino_layer_layout L;
    if (!plan || !s || layout_of(plan, s, &L)) return 0;
    if (plan->mode != WINO_CONTRACT_EXACT || plan->precision != WINO_FP32 || s->C > 8) return 0;
    if (smallc2_ok(L, s->C, plan->m)) return 2;
    const long long cw = s->C <= 4 ? 4 : 8;
    const long long tt = s->C <= 4 ? 96 : 32;  // codegen.cpp emit_smallc: SC_TT
    return (L.P * cw + 4) * (L.Kp + tt) * 4 <= 232448 ? 1 : 0;
}

int wino_contract_output_smallc(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V, void* out,
                                int mode, void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (!wino_smallc_supported(plan, s))
        return wino::fail(WINO_EUNSUPPORTED, "contract_output_smallc: needs an exact fp32 plan, C <= 8 and U in smem");
    if (mode < 0 || mode > 2) return wino::fail(WINO_EINVAL, "contract_output_smallc: mode must be 0, 1 or 2");
    if (mode == 2 && (plan->m & 1)) return wino::fail(WINO_EUNSUPPORTED, "contract_output_smallc: pooling needs an even m");
    if (((uintptr_t)U | (uintptr_t)V) & 15) return wino::fail(WINO_EINVAL, "contract_output_smallc: U, V must be 16-byte aligned");
    if ((rc = u_layout_check(U, L, "contract_output_smallc"))) return rc;
    if (s->N == 0) return WINO_OK;
    const bool v2 = smallc2_ok(L, s->C, plan->m);
    const std::string kname = std::string(v2 ? "wino_smallc2_c" : "wino_smallc_c") + std::to_string(s->C) +
                              (plan->chsum == WINO_SUM_PAIRWISE ? "p" : "l") + (v2 ? "_m" + std::to_string(mode) : "");
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s))->function(kname.c_str(), &f))) return rc;
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw, bm = L.bm, bn = L.bn;
    long long T = L.T, Tp = L.Tp, Kp = L.Kp, Cp = L.Cp;
    if (v2) {
        const unsigned smem = (unsigned)smallc2_smem(L, s->C, plan->m);
        const long long nb = (T + bn - 1) / bn;
        if (nb > (1LL << 30)) return wino::fail(WINO_EUNSUPPORTED, "contract_output_smallc: too many tiles");
        if (smem + 1024 > 48 * 1024) {  // the kernel also has static shared memory (its mbarriers)
            CUresult cr = wino::driver().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
            if (cr != CUDA_SUCCESS) return wino::fail(WINO_ECUDA, "contract_output_smallc: set smem: " + wino::cu_err(cr));
        }
        unsigned long long nz2 = 0x8000000080000000ull;  // (-0, -0): exact packed products (codegen.cpp k2_mul)
        void* args[] = {(void*)&U, (void*)&V, &out, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &Cp, &nz2};
        return wino::launch(f, dim3((unsigned)nb), dim3((unsigned)(bn * smallc2_kg())), smem, stream, args,
                            "contract_output_smallc");
    }
    const long long cw = s->C <= 4 ? 4 : 8;
    const long long tt = s->C <= 4 ? 96 : 32;  // tiles per block (SC_TT); threads = 4 * tt
    const unsigned smem = (unsigned)((L.P * cw + 4) * (L.Kp + tt) * 4);  // codegen.cpp emit_smallc: [Kp + TT][P*CW + 4]
    float rtw = 1.0f / tw, rth = 1.0f / th;
    const long long nb = (T + tt - 1) / tt;
    if (nb > (1LL << 30)) return wino::fail(WINO_EUNSUPPORTED, "contract_output_smallc: too many tiles");
    int n_blocks = (int)nb, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void* args[] = {(void*)&U, (void*)&V, &out, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &Cp, &bm, &bn, &rtw, &rth,
                    &mode, &n_blocks};
    int per_sm = 1;  // persistent: as many CTAs as fit (2 per SM for C <= 4)
    if (smem > 48 * 1024) {
        CUresult cr = wino::driver().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
        if (cr != CUDA_SUCCESS) return wino::fail(WINO_ECUDA, "contract_output_smallc: set smem: " + wino::cu_err(cr));
    }
    const int threads = (int)(4 * tt);
    if (wino::driver().OccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem) != CUDA_SUCCESS ||
        per_sm < 1)
        per_sm = 1;
    return wino::launch(f, dim3((unsigned)std::min<long long>(nb, (long long)sms * per_sm)), dim3(threads), smem,
                        stream, args, "contract_output_smallc");
}

int wino_contract_output(wino_plan* plan, const wino_layer_shape* s, const void* U, const void* V, void* y,
                         void* stream) {
    wino_layer_layout L;
    int rc = layout_of(plan, s, &L);
    if (rc) return rc;
    if (!plan->fused()) return wino::fail(WINO_EINVAL, "contract_output: needs a fused tensor-core plan (tcf_*)");
    if (((uintptr_t)U | (uintptr_t)V) & 15) return wino::fail(WINO_EINVAL, "contract_output: U, V must be 16-byte aligned");
    if (s->N == 0) return WINO_OK;
    CUfunction f;
    if ((rc = plan->layer_mod(plan->pick(s))->function("wino_tcf", &f))) return rc;
    // must match codegen.cpp emit_tcf_kernel
    const long long P = L.P, NK = plan->nk;
    const long long stb = P * 4096 + P * NK * 32;
    const long long st = std::max(1LL, std::min(4LL, (232448 - 256) / stb));
    const unsigned smem = (unsigned)(st * stb + 256);
    long long tiles = (L.Tp / 128) * (L.Kp / NK);
    if (tiles > (1LL << 30)) return wino::fail(WINO_EUNSUPPORTED, "contract_output: too many tiles");
    int n_tiles = (int)tiles, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int K = s->K, Ho = L.Ho, Wo = L.Wo, th = L.th, tw = L.tw;
    long long T = L.T, Tp = L.Tp, Kp = L.Kp, Cp = L.Cp;
    float rtw = 1.0f / tw, rth = 1.0f / th;
    static const int dbg = [] {  // timing experiments only: 1 = no MMAs, 2 = no epilogue, 4 = no y stores
        const std::string e = wino::tuning("tcf_dbg");
        return e.empty() ? 0 : atoi(e.c_str());
    }();
    int dbgv = dbg;
    void* args[] = {(void*)&U, (void*)&V, &y, &K, &Ho, &Wo, &th, &tw, &T, &Tp, &Kp, &Cp, &n_tiles, &rtw, &rth, &dbgv};
    return wino::launch(f, dim3((unsigned)std::min<long long>(tiles, sms)), dim3(192), smem, stream, args,
                        "contract_output");
}

int wino_tile_hadamard2d(wino_plan* plan, int64_t B, int C, const void* h, const void* x, void* z, void* stream) {
    if (!plan || B < 0 || C < 1) return wino::fail(WINO_EINVAL, "tile_hadamard2d: bad arguments");
    if (tile_interp(plan)) {
        wino::DevProgs pg;
        int rc = plan->dev_progs(&pg);
        return rc ? rc : wino::tile_hadamard_interp_launch(plan->precision, 2, pg, plan->r, plan->n, B * (long long)C,
                                                           h, x, z, stream);
    }
    CUfunction f;
    int rc = plan->tile.function("wino_tile_h2d", &f);
    if (rc) return rc;
    long long BC = B * (long long)C;
    void* args[] = {(void*)&h, (void*)&x, &z, &BC};
    return wino::launch(f, dim3(cdiv(BC, 128)), dim3(128), 0, stream, args, "tile_hadamard2d");
}

int wino_tile_output2d(wino_plan* plan, int64_t B, const void* y, void* out, void* stream) {
    if (!plan || B < 0) return wino::fail(WINO_EINVAL, "tile_output2d: bad arguments");
    if (tile_interp(plan)) {
        wino::DevProgs pg;
        int rc = plan->dev_progs(&pg);
        return rc ? rc : wino::tile_output_interp_launch(plan->precision, 2, pg, plan->n, plan->m, B, y, out, stream);
    }
    CUfunction f;
    int rc = plan->tile.function("wino_tile_o2d", &f);
    if (rc) return rc;
    long long b = B;
    void* args[] = {(void*)&y, &out, &b};
    return wino::launch(f, dim3(cdiv(b, 128)), dim3(128), 0, stream, args, "tile_output2d");
}

int wino_tile_hadamard1d(wino_plan* plan, int64_t B, int C, const void* h, const void* x, void* z, void* stream) {
    if (!plan || B < 0 || C < 1) return wino::fail(WINO_EINVAL, "tile_hadamard1d: bad arguments");
    if (tile_interp(plan)) {
        wino::DevProgs pg;
        int rc = plan->dev_progs(&pg);
        return rc ? rc : wino::tile_hadamard_interp_launch(plan->precision, 1, pg, plan->r, plan->n, B * (long long)C,
                                                           h, x, z, stream);
    }
    CUfunction f;
    int rc = plan->tile.function("wino_tile_h1d", &f);
    if (rc) return rc;
    long long BC = B * (long long)C;
    void* args[] = {(void*)&h, (void*)&x, &z, &BC};
    return wino::launch(f, dim3(cdiv(BC, 128)), dim3(128), 0, stream, args, "tile_hadamard1d");
}

int wino_tile_output1d(wino_plan* plan, int64_t B, const void* y, void* out, void* stream) {
    if (!plan || B < 0) return wino::fail(WINO_EINVAL, "tile_output1d: bad arguments");
    if (tile_interp(plan)) {
        wino::DevProgs pg;
        int rc = plan->dev_progs(&pg);
        return rc ? rc : wino::tile_output_interp_launch(plan->precision, 1, pg, plan->n, plan->m, B, y, out, stream);
    }
    CUfunction f;
    int rc = plan->tile.function("wino_tile_o1d", &f);
    if (rc) return rc;
    long long b = B;
    void* args[] = {(void*)&y, &out, &b};
    return wino::launch(f, dim3(cdiv(b, 128)), dim3(128), 0, stream, args, "tile_output1d");
}

}  // extern "C"
