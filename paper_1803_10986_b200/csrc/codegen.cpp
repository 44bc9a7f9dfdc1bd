// Straight-line CUDA generation for the transform stages (see codegen.h).
#include "codegen.h"

#include <algorithm>
#include <cstdio>
#include <map>
#include <sstream>

namespace wino {

namespace {

struct Ref {
    std::string name;
    bool neg;
};

class Emitter {
  public:
    // packed: every value is an f32x2 pair (two independent problems, e.g. two filters) held in a
    // 64-bit register; one add.rn.f32x2 / sub.rn.f32x2 per sum and fma.rn.f32x2(c, x, -0) per product
    // (k2_mul; the -0 pair `nz2` is a kernel parameter so ptxas can neither fold it away nor fuse
    // the product into the consuming sum -- the contraction kernel's exact packed product)
    Emitter(std::ostringstream& os, bool dbl, int& counter, bool packed = false)
        : os_(os), dbl_(dbl), packed_(packed), ctr_(counter) {}

    const char* type() const { return packed_ ? "unsigned long long" : dbl_ ? "double" : "float"; }

    std::string lit(double c) const {
        char buf[64];
        if (packed_) {
            std::snprintf(buf, sizeof buf, "k2_dup(%af)", c);
            return buf;
        }
        if (dbl_)
            std::snprintf(buf, sizeof buf, "(%a)", c);
        else
            std::snprintf(buf, sizeof buf, "(%af)", c);
        return buf;
    }

    // Evaluate one row program over `in`; returns the name holding the result.
    // Products fl(|c| * x) are shared between the rows of one pass (products of
    // +c and -c differ only in sign: fl(-c*x) == -fl(c*x) exactly, and the sign
    // is folded into the consuming add/sub).
    std::string row(const RowProg& p, const std::vector<std::string>& in) {
        if (p.ops.empty()) return packed_ ? "0ull" : dbl_ ? "0.0" : "0.0f";
        std::vector<Ref> st;
        for (const wino_op& op : p.ops) {
            if (op.kind == WINO_OP_LEAF) {
                const std::string& x = in[op.col];
                const double mag = op.coeff < 0 ? -op.coeff : op.coeff;
                const bool neg = op.coeff < 0;
                if (mag == 1.0) {
                    st.push_back({x, neg});
                } else {
                    const std::string key = x + "*" + lit(mag);
                    auto it = products_.find(key);
                    std::string t;
                    if (it != products_.end()) {
                        t = it->second;
                    } else {
                        t = fresh();
                        os_ << "  const " << type() << " " << t << " = " << mul(lit(mag), x) << ";\n";
                        products_[key] = t;
                    }
                    st.push_back({t, neg});
                }
            } else {
                Ref b = st.back();
                st.pop_back();
                Ref a = st.back();
                st.pop_back();
                std::string e;
                if (!a.neg && !b.neg)
                    e = add(a.name, b.name);
                else if (a.neg && !b.neg)
                    e = sub(b.name, a.name);
                else if (!a.neg && b.neg)
                    e = sub(a.name, b.name);
                else
                    e = sub(neg(a.name), b.name);  // fl(-a + -b) == fl(-a - b)
                std::string t = fresh();
                os_ << "  const " << type() << " " << t << " = " << e << ";\n";
                st.push_back({t, false});
            }
        }
        Ref r = st.back();
        if (!r.neg) return r.name;
        std::string t = fresh();
        os_ << "  const " << type() << " " << t << " = " << neg(r.name) << ";\n";
        return t;
    }

    // out[i] = row_i(in) for every row of `mp`
    std::vector<std::string> apply(const MatProg& mp, const std::vector<std::string>& in) {
        std::vector<std::string> out;
        out.reserve(mp.rows);
        for (int i = 0; i < mp.rows; ++i) out.push_back(row(mp.row[i], in));
        return out;
    }

    // 2D: left pass (rows of `mp` against the first index) then right pass;
    // data[a][b] with a, b < mp.cols -> out[i][j] with i, j < mp.rows
    std::vector<std::vector<std::string>> apply2d(const MatProg& mp,
                                                  const std::vector<std::vector<std::string>>& data) {
        const int R = mp.rows, K = mp.cols;
        const int ncol = (int)data[0].size();
        std::vector<std::vector<std::string>> left(R, std::vector<std::string>(ncol));
        for (int b = 0; b < ncol; ++b) {
            std::vector<std::string> col(K);
            for (int a = 0; a < K; ++a) col[a] = data[a][b];
            std::vector<std::string> res = apply(mp, col);
            for (int i = 0; i < R; ++i) left[i][b] = res[i];
        }
        std::vector<std::vector<std::string>> out(R);
        for (int i = 0; i < R; ++i) out[i] = apply(mp, left[i]);
        return out;
    }

    // 2D, one output row at a time: row i of the left pass is evaluated on every column
    // (the same rounded products and sums as apply2d, but products are not shared between
    // the rows of the left pass), then the right pass of that row, then `sink(i, values)`.
    // Only one row of the intermediate is live at a time, so the inputs can stay in their
    // narrow storage type (mixed precision: 64 f32 registers instead of 64 f64 values).
    template <class Sink>
    void apply2d_rowwise(const MatProg& mp, const std::vector<std::vector<std::string>>& data, Sink sink) {
        const int R = mp.rows, K = mp.cols;
        const int ncol = (int)data[0].size();
        for (int i = 0; i < R; ++i) {
            os_ << "  {\n";
            std::vector<std::string> left(ncol);
            for (int b = 0; b < ncol; ++b) {
                std::vector<std::string> col(K);
                for (int a = 0; a < K; ++a) col[a] = data[a][b];
                products_.clear();
                left[b] = row(mp.row[i], col);
            }
            products_.clear();
            sink(i, apply(mp, left));
            os_ << "  }\n";
            products_.clear();
        }
    }

  private:
    std::string fresh() { return "t" + std::to_string(ctr_++); }
    std::string neg(const std::string& a) const {
        return packed_ ? "(" + a + " ^ 0x8000000080000000ull)" : "(-" + a + ")";
    }
    std::string mul(const std::string& a, const std::string& b) const {
        if (packed_) return "k2_mul(" + a + ", " + b + ", nz2)";
        return std::string(dbl_ ? "__dmul_rn(" : "__fmul_rn(") + a + ", " + b + ")";
    }
    std::string add(const std::string& a, const std::string& b) const {
        if (packed_) return "k2_add(" + a + ", " + b + ")";
        return std::string(dbl_ ? "__dadd_rn(" : "__fadd_rn(") + a + ", " + b + ")";
    }
    std::string sub(const std::string& a, const std::string& b) const {
        if (packed_) return "k2_sub(" + a + ", " + b + ")";
        return std::string(dbl_ ? "__dsub_rn(" : "__fsub_rn(") + a + ", " + b + ")";
    }

    std::ostringstream& os_;
    bool dbl_, packed_;
    int& ctr_;
    std::map<std::string, std::string> products_;  // "x*|c|" -> SSA name (per emitter)
};

// q = a / b for 0 <= a < 2^22 (rb = 1/b rounded): float estimate, then exact correction
static const char* kIdivSmall =
    "static __device__ __forceinline__ int idiv_small(int a, int b, float rb) {\n"
    "  int q = (int)((float)a * rb);\n"
    "  q -= (q * b > a);\n"
    "  q += ((q + 1) * b <= a);\n"
    "  return q;\n"
    "}\n\n";

const char* tname(bool d) { return d ? "double" : "float"; }

// value conversion from compute type to a storage type
std::string store_cvt(bool compute_double, bool store_double, const std::string& v) {
    if (compute_double && !store_double) return "__double2float_rn(" + v + ")";
    return v;
}

std::string header(const GenTypes& ty) {
    std::ostringstream os;
    os << "// generated by libwino codegen -- do not edit\n"
       << "typedef " << tname(ty.in_double) << " in_t;\n"
       << "typedef " << tname(ty.compute_double) << " ct_t;\n"
       << "typedef " << tname(ty.uv_double) << " uv_t;\n"
       << "typedef " << tname(ty.y_double) << " y_t;\n"
       << kIdivSmall
       // f32 -> f64 at the point of use: volatile, so the compiler does not hoist one widened
       // copy of every input and keep all of them live (row-wise mixed-precision transforms)
       << "static __device__ __forceinline__ double wino_widen(float v) {\n"
          "  double d;\n"
          "  asm volatile(\"cvt.f64.f32 %0, %1;\" : \"=d\"(d) : \"f\"(v));\n"
          "  return d;\n"
          "}\n\n";
    return os.str();
}

}  // namespace

std::string validate(const MatProg& m, int expect_rows, int expect_cols, const char* name) {
    if (m.rows != expect_rows || m.cols != expect_cols)
        return std::string(name) + ": wrong matrix shape";
    if ((int)m.row.size() != m.rows) return std::string(name) + ": row count mismatch";
    for (int i = 0; i < m.rows; ++i) {
        int depth = 0;
        for (const wino_op& op : m.row[i].ops) {
            if (op.kind == WINO_OP_LEAF) {
                if (op.col < 0 || op.col >= m.cols) return std::string(name) + ": column out of range";
                if (!(op.coeff == op.coeff) || op.coeff == 0.0)
                    return std::string(name) + ": zero or NaN coefficient";
                ++depth;
            } else if (op.kind == WINO_OP_ADD) {
                if (depth < 2) return std::string(name) + ": ADD on a short stack";
                --depth;
            } else {
                return std::string(name) + ": unknown op kind";
            }
        }
        if (!m.row[i].ops.empty() && depth != 1) return std::string(name) + ": malformed program";
    }
    return "";
}

// K4: output transform y = A^T M A, crop, NCHW (M is [P][Kp][Tp] in uv_t, or
// fp32 for the tensor-core modes).  The block stages M[.][k][t0 .. t0+TB) for
// all P points through shared memory with 16-byte coalesced loads, then each
// thread transforms one tile.
static void emit_output_flat(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty, int TB,
                               int& ctr, const char* mt = "uv_t", int mes = 0) {
    const int n = r + m - 1, P = n * n;
    const int es = mes ? mes : (ty.uv_double ? 8 : 4);
    const int VEC = 16 / es;
    const char* VT = es == 8 ? "double2" : "float4";
    {
        os << "extern \"C\" __global__ void __launch_bounds__(" << TB << ") wino_output_flat(\n"
              "    const " << mt << "* __restrict__ Mm, y_t* __restrict__ y, int K, int Ho, int Wo, int th, int tw,\n"
              "    long long T, long long Tp, long long Kp) {\n"
              "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
              "  " << mt << "* sm = reinterpret_cast<" << mt << "*>(smem_raw);  // [P][TB]\n"
           << "  const int t0 = blockIdx.x * " << TB << ";\n"
              "  const int k = blockIdx.y;\n"
              "  const long long plane = Kp * Tp;\n"
           << "  constexpr int NV = " << TB / VEC << ";\n"
           << "#pragma unroll 4\n"
           << "  for (int i = threadIdx.x; i < " << P << " * NV; i += " << TB << ") {\n"
           << "    const int p = i / NV, q = i - p * NV;\n"
           << "    const int tt = t0 + q * " << VEC << ";\n"
           << "    if (tt < Tp)\n"
           << "      *reinterpret_cast<" << VT << "*>(sm + p * " << TB << " + q * " << VEC << ") = __ldg(reinterpret_cast<const "
           << VT << "*>(Mm + p * plane + (long long)k * Tp + tt));\n"
           << "  }\n"
              "  __syncthreads();\n"
              "  const int t = t0 + threadIdx.x;\n"
              "  if (t >= T) return;\n";
        std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << mm[a][b] << " = (ct_t)sm[" << (a * n + b) * TB << " + threadIdx.x];\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto yv = em.apply2d(AT, mm);
        os << "  const int per = th * tw;\n"
              "  const int img = t / per;\n"
              "  const int rem = t - img * per;\n"
              "  const int ti = rem / tw, tj = rem - ti * tw;\n"
           << "  const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
           << "  y_t* dst = y + ((long long)img * K + k) * ((long long)Ho * Wo) + y0 * Wo + x0;\n"
           << "  if (y0 + " << m << " <= Ho && x0 + " << m << " <= Wo) {\n";
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b)
                os << "    dst[" << a << " * Wo + " << b << "] = " << store_cvt(ty.compute_double, ty.y_double, yv[a][b])
                   << ";\n";
        os << "  } else {\n";
        for (int a = 0; a < m; ++a) {
            os << "    if (y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; ++b)
                os << "      if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b
                   << "] = " << store_cvt(ty.compute_double, ty.y_double, yv[a][b]) << ";\n";
            os << "    }\n";
        }
        os << "  }\n}\n";
    }
}
static void emit_output_kernel(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty, int TB,
                               int& ctr, const char* mt = "uv_t", int mes = 0) {
    (void)TB;
    (void)mes;
    const int n = r + m - 1;
    // Block = (band of R tile rows of one image) x (KB output channels); 128
    // threads loop over its KB*R*tw tiles.  Each tile's m x m outputs are
    // parked in shared memory as image rows, then the block writes the band's
    // rows -- contiguous in y[img][k] -- with coalesced stores (per-thread m x m
    // patches would scatter each warp store over ~m rows).
    os << "extern \"C\" __global__ void __launch_bounds__(128, 4) wino_output_xform(\n"
          "    const " << mt << "* __restrict__ Mm, y_t* __restrict__ y, int K, int Ho, int Wo, int th, int tw,\n"
          "    long long T, long long Tp, long long Kp, int R, int KB) {\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  y_t* so = reinterpret_cast<y_t*>(smem_raw);  // [KB][R*m][Wo]\n"
          "  const int band = blockIdx.x, kg = blockIdx.y, img = blockIdx.z;\n"
       << "  const int rows = min(R * " << m << ", Ho - band * R * " << m << ");\n"
          "  const int items = KB * R * tw;\n"
          "  const long long plane = Kp * Tp;\n"
          "  const int per = th * tw;\n"
          "#pragma unroll 1\n"
          "  for (int it = threadIdx.x; it < items; it += 128) {\n"
          "    const int kk = it / (R * tw);\n"
          "    const int rem = it - kk * (R * tw);\n"
          "    const int til = rem / tw, tj = rem - til * tw;\n"
          "    const int k = kg * KB + kk, ti = band * R + til;\n"
          "    if (k >= K || ti >= th) continue;\n"
          "    const " << mt << "* src = Mm + (long long)k * Tp + ((long long)img * per + ti * tw + tj);\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "    const ct_t " << mm[a][b] << " = (ct_t)__ldg(src + " << (a * n + b) << " * plane);\n";
        }
    Emitter em(os, ty.compute_double, ctr);
    auto yv = em.apply2d(AT, mm);
    os << "    y_t* d = so + ((long long)kk * R * " << m << " + til * " << m << ") * Wo + tj * " << m << ";\n"
       << "    const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
       << "    if (y0 + " << m << " <= Ho && x0 + " << m << " <= Wo) {\n";
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b)
            os << "      d[" << a << " * Wo + " << b << "] = " << store_cvt(ty.compute_double, ty.y_double, yv[a][b])
               << ";\n";
    os << "    } else {\n";
    for (int a = 0; a < m; ++a) {
        os << "      if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "        if (x0 + " << b << " < Wo) d[" << a << " * Wo + " << b
               << "] = " << store_cvt(ty.compute_double, ty.y_double, yv[a][b]) << ";\n";
        os << "      }\n";
    }
    os << "    }\n  }\n"
          "  __syncthreads();\n"
          "  // the band's rows of each output channel are contiguous in y\n"
          "#pragma unroll 1\n"
          "  for (int kk = 0; kk < KB; ++kk) {\n"
          "    const int k = kg * KB + kk;\n"
          "    if (k >= K) break;\n"
       << "    y_t* dst = y + (((long long)img * K + k) * Ho + band * R * " << m << ") * Wo;\n"
       << "    const y_t* sb = so + (long long)kk * R * " << m << " * Wo;\n"
          "    const int cnt = rows * Wo;\n"
          "    for (int i = threadIdx.x; i < cnt; i += 128) dst[i] = sb[i];\n"
          "  }\n}\n";
}

// K1, gather form with direct stores: thread = one tile x CPT consecutive
// channels (the tile index math -- two divisions, padding predicates -- is done
// once per thread, then a channel loop); the alpha x alpha window is gathered
// from global memory (zero padding fused, unpredicated interior path) and the P
// values are stored straight from registers -- a warp's store of one p covers
// 32 consecutive t of the blocked V, one aligned 128-byte line.
// Grid (Cp / CPT, n_tb [+ n_kb filter rows]).
static void emit_input_gather(std::ostringstream& os, int r, int m, const MatProg& BT, const GenTypes& ty, int bn,
                              int TB, int& ctr) {
    const int n = r + m - 1, P = n * n;
    // ST: the image planes this block's tiles read (consecutive images of channels c0 .. c0 + CPT - 1,
    // each a contiguous H x W run of x) are first copied to shared memory with one cp.async.bulk
    // per plane (completion on an mbarrier: no staging loop, no registers), and the windows are
    // gathered from there -- for small images, where a warp's 32 tiles span several tile rows and
    // every window load from global memory touches 7-13 L1 lines.
    os << "template <bool ST> static __device__ __forceinline__ in_t k1_ld(const in_t* p) {\n"
          "  if constexpr (ST) return *p; else return __ldg(p);\n}\n"
          "template <bool ST> static __device__ __forceinline__ float2 k1_ld2(const float2* p) {\n"
          "  if constexpr (ST) return *p; else return __ldg(p);\n}\n"
          "template <bool ST>\n"
          "static __device__ __forceinline__ void input_gather_body(const in_t* __restrict__ x, uv_t* __restrict__ V,\n"
          "    int C, int H, int W, int pad, int th, int tw, long long T, long long Tp, long long Cp,\n"
          "    float rtw, float rth, int t0, int cb) {\n"
          "  const long long plane = Cp * Tp;\n"
          "  const long long tt = (long long)t0 + threadIdx.x;\n"
       << "  const int c0 = cb * " << gather_cpt(P) << ";\n"
       << "  extern __shared__ __align__(16) unsigned char k1_smem[];\n"
          "  __shared__ __align__(8) unsigned long long k1_bar;\n"
          "  int img_lo = 0;\n"
          "  if constexpr (ST) {\n"
          "    if (c0 < C && t0 < T) {  // block-uniform\n"
          "      const int per = th * tw, HWi = H * W;\n"
          "      img_lo = t0 / per;\n"
       << "      const long long tl = (T < (long long)t0 + " << TB << " ? T : (long long)t0 + " << TB << ") - 1;\n"
       << "      const int nc = C - c0 < " << gather_cpt(P) << " ? C - c0 : " << gather_cpt(P) << ";\n"
          "      const int ncp = ((int)(tl / per) - img_lo + 1) * nc;\n"
          "      const unsigned bar = (unsigned)__cvta_generic_to_shared(&k1_bar);\n"
          "      if (threadIdx.x == 0) {\n"
          "        asm volatile(\"mbarrier.init.shared::cta.b64 [%0], %1;\" ::\"r\"(bar), \"r\"(1u) : \"memory\");\n"
          "        asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
          "      }\n"
          "      __syncthreads();\n"
          "      if (threadIdx.x < 32) {\n"
          "        if (threadIdx.x == 0)\n"
          "          asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" ::\"r\"(bar),\n"
          "                       \"r\"((unsigned)(ncp * HWi * (int)sizeof(in_t))) : \"memory\");\n"
          "        __syncwarp();\n"
          "        for (int j = threadIdx.x; j < ncp; j += 32) {\n"
          "          const int ii = j / nc, cc = j - ii * nc;\n"
       << "          const in_t* gp = x + ((long long)(img_lo + ii) * C + c0 + cc) * HWi;\n"
       << "          in_t* sp = reinterpret_cast<in_t*>(k1_smem) + (long long)(ii * " << gather_cpt(P) << " + cc) * HWi;\n"
          "          asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "                       ::\"r\"((unsigned)__cvta_generic_to_shared(sp)), \"l\"(gp),\n"
          "                         \"r\"((unsigned)(HWi * (int)sizeof(in_t))), \"r\"(bar) : \"memory\");\n"
          "        }\n"
          "      }\n"
          "      asm volatile(\"{\\n\\t.reg .pred P1;\\nK1_WAIT_%=:\\n\\t\"\n"
          "                   \"mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\\n\\t\"\n"
          "                   \"@!P1 bra K1_WAIT_%=;\\n}\\n\" ::\"r\"(bar), \"r\"(0u) : \"memory\");\n"
          "    }\n"
          "  }\n"
       << "  if (tt >= Tp) return;\n"
       << "  uv_t* op = V + ((tt / " << bn << ") * Cp + c0) * " << bn << " + (tt % " << bn << ");\n"
       << "  if (tt >= T || c0 >= C) {\n"
       << "    for (int cc = 0; cc < " << gather_cpt(P) << "; ++cc, op += " << bn << ") {\n"
          "      const uv_t z = (c0 + cc >= C) ? (uv_t)(-0.0) : (uv_t)0;\n"
          "#pragma unroll\n"
       << "      for (int p = 0; p < " << P << "; ++p) op[p * plane] = z;\n"
          "    }\n"
          "    return;\n"
          "  }\n"
          "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
          "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
          "  const int off = off0 + threadIdx.x;\n"
          "  const int k = idiv_small(off, tw, rtw), tj = off - k * tw;\n"
          "  const int di = idiv_small(ti0 + k, th, rth);\n"
          "  const int ti = ti0 + k - di * th;\n"
       << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
       << "  const long long HW = (long long)H * W;\n"
       << "  const in_t* src = ST ? reinterpret_cast<const in_t*>(k1_smem) + (long long)(img0 + di - img_lo) * "
       << gather_cpt(P) << " * HW\n"
          "                       : x + ((long long)(img0 + di) * C + c0) * HW;\n"
       << "  const bool interior = h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W;\n"
       << (gather_cpt(P) > 1 && P <= 16 ? "#pragma unroll\n" : "#pragma unroll 1\n")
       << "  for (int cc = 0; cc < " << gather_cpt(P) << "; ++cc, src += HW, op += " << bn << ") {\n"
       << "  if (c0 + cc >= C) {\n"
          "#pragma unroll\n"
       << "    for (int p = 0; p < " << P << "; ++p) op[p * plane] = (uv_t)(-0.0);\n"
          "    continue;\n"
          "  }\n";
    // mixed precision (f32 tensors, f64 transforms): keep the window in its 64 f32 registers and
    // evaluate one output row at a time (Emitter::apply2d_rowwise) instead of holding alpha^2
    // f64 intermediates (166 registers, 16% occupancy at alpha = 8); same products, same sums
    const bool rowwise = ty.compute_double && !ty.in_double && n >= 6 && tuning("k1rowwise") != "0";
    const char* wt = rowwise ? "in_t" : "ct_t";
    std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
            os << "  " << wt << " " << d[a][b] << ";\n";
        }
    if (m % 2 == 0 && !ty.in_double) {
        // even m: every window starts at the same parity (w0 = m*tj - pad), so with an
        // even row length each row of the window is read with 8-byte loads from the
        // even column at or below w0 -- fewer, fuller load wavefronts than scalar
        // gathers; the parity branch is warp-uniform.
        for (int sh = 0; sh < 2; ++sh) {
            const int nl = (n + sh + 1) / 2;
            os << "  " << (sh == 0 ? "if" : "else if") << " (interior && (W & 1) == 0 && (pad & 1) == " << sh
               << " && (reinterpret_cast<size_t>(src) & 7) == 0) {\n"
               << "    const float2* rp = reinterpret_cast<const float2*>(src + h0 * W + w0 - " << sh << ");\n"
               << "    const int W2 = W >> 1;\n";
            for (int a = 0; a < n; ++a) {
                for (int q = 0; q < nl; ++q)
                    os << "    const float2 f" << a << "_" << q << " = k1_ld2<ST>(rp + " << a << " * W2 + " << q << ");\n";
                for (int b = 0; b < n; ++b) {
                    const int e = b + sh;
                    os << "    " << d[a][b] << " = (" << wt << ")f" << a << "_" << e / 2 << (e % 2 ? ".y" : ".x") << ";\n";
                }
            }
            os << "  }\n";
        }
        os << "  else if (interior) {\n";
    } else {
        os << "  if (interior) {\n";
    }
    os << "    const in_t* rp = src + h0 * W + w0;\n";
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            os << "    " << d[a][b] << " = (" << wt << ")k1_ld<ST>(rp + " << a << " * W + " << b << ");\n";
    os << "  } else {\n";
    for (int a = 0; a < n; ++a)
        os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
    for (int b = 0; b < n; ++b)
        os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            os << "    " << d[a][b] << " = (r" << a << " && c" << b << ") ? (" << wt << ")k1_ld<ST>(src + (h0 + " << a
               << ") * W + (w0 + " << b << ")) : (" << wt << ")0;\n";
    os << "  }\n";
    Emitter em(os, ty.compute_double, ctr);
    if (rowwise) {
        std::vector<std::vector<std::string>> dw(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) dw[a][b] = "wino_widen(" + d[a][b] + ")";
        em.apply2d_rowwise(BT, dw, [&](int i, const std::vector<std::string>& row) {
            for (int j = 0; j < n; ++j)
                os << "  op[" << (i * n + j) << " * plane] = " << store_cvt(ty.compute_double, ty.uv_double, row[j])
                   << ";\n";
        });
    } else {
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                os << "  op[" << (i * n + j) << " * plane] = " << store_cvt(ty.compute_double, ty.uv_double, v[i][j])
                   << ";\n";
    }
    os << "  }\n}\n\n";
    // register cap through the minimum-blocks launch bound: 384 threads per SM (<= 168 registers:
    // no spills; cfg3 mixed K1 79.9 -> 51.1 us, against 69.8 / 131.8 us at 512 / 640 threads, which
    // spill); tuning key k1rowwise = 2..6 selects another bound (0: row-wise off)
    const int rw_blocks = std::atoi(tuning("k1rowwise").c_str()) >= 2 ? std::atoi(tuning("k1rowwise").c_str()) : 3;
    const std::string lb = rowwise ? std::to_string(TB) + ", " + std::to_string(rw_blocks * 128 / TB) : std::to_string(TB);
    // bulk-staged variants: tuning key "k1st_blocks" = minimum blocks per SM (register cap), default none
    // minimum blocks per SM = register cap.  alpha = 8: 6 blocks (<= 85 registers, a few spilled values)
    // beat the unconstrained 106 registers / 4 blocks on every VGG-16 layer -- bulk-staged K1 at 14 x 14
    // 103.1 -> 98.8 us, 28 x 28 246 -> 231, 56 x 56 456 -> 420; global gather at 112 x 112 865 -> 832,
    // 224 x 224 1665 -> 1626 (7 and 8 blocks spill too much: 56 x 56 547 / 759 us); alpha = 4 loses
    // (cfg2 15.0 -> 16.8 us), so only P = 64 gets the bound (tools/sweeps/sweep_k1st_blocks.sh)
    auto blocks_of = [&](const char* key) {
        const std::string e = tuning(key);
        return e.empty() ? (P == 64 ? 6 : 0) : std::atoi(e.c_str());
    };
    const int st_blocks = blocks_of("k1st_blocks"), pl_blocks = blocks_of("k1_blocks");
    const std::string lb_plain = lb;
    for (int st = 0; st < 2; ++st) {
        const std::string sfx = st ? "_st" : "", tp = st ? "<true>" : "<false>";
        const int nb = st ? st_blocks : pl_blocks;
        const std::string lb = !rowwise && nb > 0 ? std::to_string(TB) + ", " + std::to_string(nb) : lb_plain;
        os << "extern \"C\" __global__ void __launch_bounds__(" << lb << ") wino_input_gather" << sfx << "(\n"
              "    const in_t* __restrict__ x, uv_t* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, int Wl, float rtw, float rth) {\n"
           << "  input_gather_body" << tp << "(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.y * " << TB
           << ", blockIdx.x);\n"
           << "}\n\n"
           << "extern \"C\" __global__ void __launch_bounds__(" << lb << ") wino_transforms_gather" << sfx << "(\n"
              "    const in_t* __restrict__ x, uv_t* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
              "    const in_t* __restrict__ w, uv_t* __restrict__ U, int K, long long Kp, int Wl, float rtw, float rth) {\n"
              "  if ((int)blockIdx.y < n_tb) {\n"
           << "    if (Wl && (int)blockIdx.x * " << gather_cpt(P) << " >= C) return;  // consumer reads the C real rows only\n"
           << "    input_gather_body" << tp << "(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.y * " << TB
           << ", blockIdx.x);\n"
           << "  } else {\n"
           << "    for (int cc = 0; cc < " << gather_cpt(P) << "; ++cc)\n"
           << "      filter_body(w, U, K, C, Kp, Cp, (blockIdx.y - n_tb) * " << TB << " + threadIdx.x, blockIdx.x * "
           << gather_cpt(P) << " + cc);\n"
              "  }\n"
              "}\n\n";
    }
}

// K4, gather form: thread = (tile t, output channel k).  Its P values
// M[p][k][t] are read straight from global memory (a warp's load of one p is
// 32 consecutive t: one coalesced 128-byte line), transformed in registers and
// the m x m block is stored to NCHW y -- as 8/16-byte pairs when m and Wo are
// even, so a warp's row store covers a contiguous stretch of the output row.
// Each thread loops over KPT output channels (tile index math done once).
// Grid (ceil(T / TB), ceil(K / KPT)).
static void emit_output_gather(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty, int TB,
                               int& ctr, const char* mt = "uv_t") {
    const int n = r + m - 1;
    const char* PT = ty.y_double ? "double2" : "float2";
    const bool rowwise = ty.compute_double && !ty.uv_double && std::string(mt) == "uv_t" && n >= 6 &&
                         tuning("k4rowwise") != "0";
    const int rw_blocks = std::atoi(tuning("k4rowwise").c_str()) >= 2 ? std::atoi(tuning("k4rowwise").c_str()) : 3;  // cfg3 mixed K4 65.8 -> 47.2 us at 2..4 blocks, 61.5 at 5 (spills)
    os << "extern \"C\" __global__ void __launch_bounds__(" << TB
       << (rowwise ? ", " + std::to_string(rw_blocks)
                   : std::atoi(tuning("k4_blocks").c_str()) > 0 ? ", " + tuning("k4_blocks") : std::string())
       << ") wino_output_gather(\n"
          "    const " << mt << "* __restrict__ Mm, y_t* __restrict__ y, int K, int Ho, int Wo, int th, int tw,\n"
          "    long long T, long long Tp, long long Kp, float rtw, float rth) {\n"
       << "  const int t0 = blockIdx.x * " << TB << ";\n"
          "  const int t = t0 + threadIdx.x;\n"
          "  if (t >= T) return;\n"
          "  const long long plane = Kp * Tp;\n"
          "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
          "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
          "  const int off = off0 + threadIdx.x;\n"
          "  const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
          "  const int di = idiv_small(ti0 + kk, th, rth);\n"
          "  const int ti = ti0 + kk - di * th;\n"
       << "  const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
       << "  const int k0 = blockIdx.y * " << gather_kpt() << ";\n"
       << "  const long long HoWo = (long long)Ho * Wo;\n"
       << "  const " << mt << "* src = Mm + (long long)k0 * Tp + t;\n"
       << "  y_t* dst = y + (((long long)(img0 + di) * K + k0) * Ho + y0) * Wo + x0;\n"
       << "  const bool full = y0 + " << m << " <= Ho && x0 + " << m << " <= Wo;\n"
       << "  const bool pair_ok = (Wo & 1) == 0 && (reinterpret_cast<size_t>(y) & (2 * sizeof(y_t) - 1)) == 0;\n"
       << "#pragma unroll 1\n"
       << "  for (int k = k0; k < k0 + " << gather_kpt() << " && k < K; ++k, src += Tp, dst += HoWo) {\n";
    // mixed precision (f32 M, f64 transform): keep the alpha^2 values in f32 registers and
    // evaluate one output row at a time (see emit_input_gather)
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            if (rowwise)
                os << "  const " << mt << " " << mm[a][b] << " = __ldg(src + " << (a * n + b) << " * plane);\n";
            else
                os << "  const ct_t " << mm[a][b] << " = (ct_t)__ldg(src + " << (a * n + b) << " * plane);\n";
        }
    Emitter em(os, ty.compute_double, ctr);
    // stores of output row a (values already in the y type)
    auto store_row = [&](int a, const std::vector<std::string>& v) {
        if (m % 2 == 0) {
            // x0 = m * tj and Wo even: a pair of columns is valid or clipped as a whole, so every
            // tile (edge tiles too) stores 8/16-byte pairs -- half the L2 store requests
            os << "  if (pair_ok) {\n"
               << "    if (full || y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; b += 2)
                os << "      if (full || x0 + " << b << " < Wo) *reinterpret_cast<" << PT << "*>(dst + " << a
                   << " * Wo + " << b << ") = make_" << PT << "(" << v[b] << ", " << v[b + 1] << ");\n";
            os << "    }\n"
               << "  } else\n";
        }
        os << "  if (full || y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "    if (full || x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = " << v[b] << ";\n";
        os << "  }\n";
    };
    if (rowwise) {
        std::vector<std::vector<std::string>> mw(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) mw[a][b] = "wino_widen(" + mm[a][b] + ")";
        em.apply2d_rowwise(AT, mw, [&](int a, const std::vector<std::string>& row) {
            std::vector<std::string> v(m);
            for (int b = 0; b < m; ++b) v[b] = store_cvt(ty.compute_double, ty.y_double, row[b]);
            store_row(a, v);
        });
    } else {
        auto yv = em.apply2d(AT, mm);
        for (int a = 0; a < m; ++a) {
            std::vector<std::string> v(m);
            for (int b = 0; b < m; ++b) v[b] = store_cvt(ty.compute_double, ty.y_double, yv[a][b]);
            store_row(a, v);
        }
    }
    os << "  }\n}\n\n";
}

// K4 with the activation fused (conv stacks, BASELINE config 5): the same
// gather output transform, then ReLU -- and with pool = 1 the 2x2 max-pool, which
// is local to a tile when m is even (tile origins are even) -- written straight
// to the activation tensor: the pre-activation y never goes to HBM.  Same
// expressions as wino_relu_pool (wino_static.cu): v = max(max(q00, q01),
// max(q10, q11)); out = v > 0 ? v : 0.  fp32 y only.
static void emit_output_gather_act(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty,
                                   int TB, int& ctr, const char* mt = "uv_t") {
    const int n = r + m - 1;
    os << "static __device__ __forceinline__ float wino_relu(float v) { return v > 0.f ? v : 0.f; }\n"
          "extern \"C\" __global__ void __launch_bounds__(" << TB
       << (std::atoi(tuning("k4_blocks").c_str()) > 0 ? ", " + tuning("k4_blocks") : std::string())
       << ") wino_output_gather_act(\n"
          "    const " << mt << "* __restrict__ Mm, float* __restrict__ act, int K, int Ho, int Wo, int th, int tw,\n"
          "    long long T, long long Tp, long long Kp, float rtw, float rth, int pool) {\n"
       << "  const int t0 = blockIdx.x * " << TB << ";\n"
          "  const int t = t0 + threadIdx.x;\n"
          "  if (t >= T) return;\n"
          "  const int k = blockIdx.y;\n"
          "  const long long plane = Kp * Tp;\n"
          "  const " << mt << "* src = Mm + (long long)k * Tp + t;\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "  const ct_t " << mm[a][b] << " = (ct_t)__ldg(src + " << (a * n + b) << " * plane);\n";
        }
    os << "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
          "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
          "  const int off = off0 + threadIdx.x;\n"
          "  const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
          "  const int di = idiv_small(ti0 + kk, th, rth);\n"
          "  const int ti = ti0 + kk - di * th;\n";
    Emitter em(os, ty.compute_double, ctr);
    auto yv = em.apply2d(AT, mm);
    auto val = [&](int a, int b) { return store_cvt(ty.compute_double, false, yv[a][b]); };
    os << "  const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
          "  if (!pool) {\n"
          "    float* dst = act + (((long long)(img0 + di) * K + k) * Ho + y0) * Wo + x0;\n";
    if (m % 2 == 0) {
        // whole tiles of an even-width output: 8-byte stores (x0 = m * tj is even), half as many
        // store requests -- the un-pooled 56 / 28 / 14-pixel layers are bound by the L2's
        // request rate for 4-byte partial-sector writes, not by bytes
        os << "    // x0 and Wo even: a pair of columns is valid or clipped as a whole\n"
              "    if ((Wo & 1) == 0 && (reinterpret_cast<size_t>(act) & 7) == 0) {\n";
        for (int a = 0; a < m; ++a) {
            os << "      if (y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; b += 2)
                os << "        if (x0 + " << b << " < Wo) *reinterpret_cast<float2*>(dst + " << a << " * Wo + " << b
                   << ") = make_float2(wino_relu(" << val(a, b) << "), wino_relu(" << val(a, b + 1) << "));\n";
            os << "      }\n";
        }
        os << "      return;\n    }\n";
    }
    for (int a = 0; a < m; ++a) {
        os << "    if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "      if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = wino_relu(" << val(a, b)
               << ");\n";
        os << "    }\n";
    }
    os << "    return;\n  }\n";
    if (m % 2 == 0) {
        os << "  const int Hp = Ho >> 1, Wp = Wo >> 1, py0 = y0 >> 1, px0 = x0 >> 1;\n"
              "  float* dst = act + (((long long)(img0 + di) * K + k) * Hp + py0) * Wp + px0;\n";
        for (int a = 0; a < m / 2; ++a) {
            os << "  if (py0 + " << a << " < Hp) {\n";
            for (int b = 0; b < m / 2; ++b)
                os << "    if (px0 + " << b << " < Wp) dst[" << a << " * Wp + " << b << "] = wino_relu(fmaxf(fmaxf("
                   << val(2 * a, 2 * b) << ", " << val(2 * a, 2 * b + 1) << "), fmaxf(" << val(2 * a + 1, 2 * b)
                   << ", " << val(2 * a + 1, 2 * b + 1) << ")));\n";
            os << "  }\n";
        }
    }
    os << "}\n\n";
}

// ---- NHWC layer kernels (activations x[N][H][W][C], y[N][Ho][Wo][K]; w, U, V, M as for NCHW)
//
// Channels are the contiguous axis of x and y, tiles the contiguous axis of V and M, so no
// thread-to-(tile, channel) map is unit-stride on both sides.  A block is 8 tiles x 16
// channels, a warp 8 tiles x 4 channels: the larger tensor (V written by K1, M read by K4;
// alpha^2 / m^2 times the activation) moves in full 32-byte sectors (8 consecutive t), the
// activation in 16-byte runs (4 consecutive channels) whose other half-sector is touched by
// the neighbouring warp of the same block (L1 for the K1 loads, merged in L2 for the K4
// stores).  Same generated straight-line transforms, same bits as the NCHW kernels.
static void emit_nhwc(std::ostringstream& os, int r, int m, const MatProg& BT, const MatProg& AT, const GenTypes& ty,
                      int bn, int& ctr) {
    const int n = r + m - 1, P = n * n;
    // K1
    os << "extern \"C\" __global__ void __launch_bounds__(128) wino_input_gather_nhwc(\n"
          "    const in_t* __restrict__ x, uv_t* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp) {\n"
          "  const long long plane = Cp * Tp;\n"
          "  const long long tt = (long long)blockIdx.x * 8 + (threadIdx.x & 7);\n"
          "  const int c = blockIdx.y * 16 + (threadIdx.x >> 3);\n"
          "  if (tt >= Tp || c >= Cp) return;\n"
       << "  uv_t* op = V + ((tt / " << bn << ") * Cp + c) * " << bn << " + (tt % " << bn << ");\n"
       << "  if (tt >= T || c >= C) {\n"
          "    const uv_t z = (c >= C) ? (uv_t)(-0.0) : (uv_t)0;\n"
          "#pragma unroll\n"
       << "    for (int p = 0; p < " << P << "; ++p) op[p * plane] = z;\n"
          "    return;\n"
          "  }\n"
          "  const int t = (int)tt;\n"
          "  const int g = t / tw, tj = t - g * tw;\n"
          "  const int img = g / th, ti = g - img * th;\n"
       << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
       << "  const in_t* src = x + (long long)img * H * W * C + c;\n"
       << "  const bool interior = h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W;\n";
    std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
            os << "  ct_t " << d[a][b] << ";\n";
        }
    os << "  if (interior) {\n"
          "    const in_t* rp = src + ((long long)h0 * W + w0) * C;\n"
          "    const long long rs = (long long)W * C;\n";
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            os << "    " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * rs + " << b << " * (long long)C);\n";
    os << "  } else {\n";
    for (int a = 0; a < n; ++a)
        os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
    for (int b = 0; b < n; ++b)
        os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            os << "    " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + ((long long)(h0 + " << a
               << ") * W + (w0 + " << b << ")) * C) : (ct_t)0;\n";
    os << "  }\n";
    {
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                os << "  op[" << (i * n + j) << " * plane] = " << store_cvt(ty.compute_double, ty.uv_double, v[i][j])
                   << ";\n";
    }
    os << "}\n\n";
    // K4
    os << "extern \"C\" __global__ void __launch_bounds__(128) wino_output_gather_nhwc(\n"
          "    const uv_t* __restrict__ Mm, y_t* __restrict__ y, int K, int Ho, int Wo, int th, int tw,\n"
          "    long long T, long long Tp, long long Kp) {\n"
          "  const long long tt = (long long)blockIdx.x * 8 + (threadIdx.x & 7);\n"
          "  const int k = blockIdx.y * 16 + (threadIdx.x >> 3);\n"
          "  if (tt >= T || k >= K) return;\n"
          "  const long long plane = Kp * Tp;\n"
          "  const uv_t* src = Mm + (long long)k * Tp + tt;\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "  const ct_t " << mm[a][b] << " = (ct_t)__ldg(src + " << (a * n + b) << " * plane);\n";
        }
    os << "  const int t = (int)tt;\n"
          "  const int g = t / tw, tj = t - g * tw;\n"
          "  const int img = g / th, ti = g - img * th;\n"
       << "  const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n";
    {
        Emitter em(os, ty.compute_double, ctr);
        auto yv = em.apply2d(AT, mm);
        os << "  y_t* dst = y + (((long long)img * Ho + y0) * Wo + x0) * K + k;\n"
           << "  const long long rs = (long long)Wo * K;\n"
           << "  if (y0 + " << m << " <= Ho && x0 + " << m << " <= Wo) {\n";
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b)
                os << "    dst[" << a << " * rs + " << b << " * (long long)K] = "
                   << store_cvt(ty.compute_double, ty.y_double, yv[a][b]) << ";\n";
        os << "  } else {\n";
        for (int a = 0; a < m; ++a) {
            os << "    if (y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; ++b)
                os << "      if (x0 + " << b << " < Wo) dst[" << a << " * rs + " << b << " * (long long)K] = "
                   << store_cvt(ty.compute_double, ty.y_double, yv[a][b]) << ";\n";
            os << "    }\n";
        }
        os << "  }\n";
    }
    os << "}\n\n";
}

// K3 + K4 (+ ReLU, + 2x2 max-pool) in one kernel for small channel counts (C <= 8,
// e.g. VGG-16 layer 1 with C = 3): the contraction is a few products per point, so
// the unfused pair is bound by writing and re-reading M (alpha^2 x K x T floats,
// 6 GB at VGG layer 1).  Persistent CTAs keep all of U in shared memory
// ([P][Kp][CW], loaded once), stage the V values of 64 tiles at a time
// ([P][64][CW]), and each thread turns one (tile, filter) pair into its P channel
// sums -- the plan's linear order, or the pairwise halving tree of the padded
// 8-channel stage with the -0 leaves pruned (x + -0 == x exactly, so the result
// is the contraction kernel's bit for bit) -- then (A^T M) A, the activation and
// the store.  A warp covers 8 tiles x 4 filters, so its shared-memory reads are
// broadcasts of 8 V vectors and 4 U vectors.  fp32 plans only.
static void emit_smallc(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty, int& ctr) {
    const int n = r + m - 1, P = n * n;
    os << "template <int L, int R, int C>\n"
          "static __device__ __forceinline__ float sc_tree(const float* z) {\n"
          "  if constexpr (R - L == 1) {\n    return z[L];\n  } else {\n"
          "    constexpr int Mid = (L + R) / 2;\n"
          "    if constexpr (Mid >= C) return sc_tree<L, Mid, C>(z);\n"
          "    else return __fadd_rn(sc_tree<L, Mid, C>(z), sc_tree<Mid, R, C>(z));\n  }\n}\n"
          "template <int C, int PW, int CW>\n"
          "static __device__ __forceinline__ float sc_sum(const float* __restrict__ u, const float* __restrict__ v) {\n"
          "  float uu[CW], vv[CW], z[8];\n"
          "#pragma unroll\n"
          "  for (int q = 0; q < CW; q += 4) {\n"
          "    const float4 a = *reinterpret_cast<const float4*>(u + q), b = *reinterpret_cast<const float4*>(v + q);\n"
          "    uu[q] = a.x; uu[q + 1] = a.y; uu[q + 2] = a.z; uu[q + 3] = a.w;\n"
          "    vv[q] = b.x; vv[q + 1] = b.y; vv[q + 2] = b.z; vv[q + 3] = b.w;\n  }\n"
          "#pragma unroll\n"
          "  for (int c = 0; c < C; ++c) z[c] = __fmul_rn(uu[c], vv[c]);\n"
          "  if constexpr (PW) {\n    return sc_tree<0, 8, C>(z);\n  } else {\n"
          "    float a = z[0];\n"
          "#pragma unroll\n"
          "    for (int c = 1; c < C; ++c) a = __fadd_rn(a, z[c]);\n    return a;\n  }\n}\n";
    os << "template <int C, int PW>\n"
          "static __device__ __forceinline__ void sc_body(const float* __restrict__ U, const float* __restrict__ V,\n"
          "    float* __restrict__ out, int K, int Ho, int Wo, int th, int tw, long long T, long long Tp, long long Kp,\n"
          "    long long Cp, int bm, int bn, float rtw, float rth, int mode, int n_blocks) {\n"
          "  constexpr int CW = C <= 4 ? 4 : 8;\n"
          "  constexpr int NW = C <= 4 ? 12 : 4;       // warps per CTA (one CTA per SM)\n"
          "  constexpr int SC_TT = 8 * NW;             // tiles per block: a warp = 8 tiles x 4 filters\n"
       << "  constexpr int P = " << P << ";\n"
          "  constexpr int STR = P * CW + 4;  // per-filter / per-tile row (+16 B: conflict-free for 8 rows)\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  float* sU = reinterpret_cast<float*>(smem_raw);   // [Kp][STR]\n"
          "  float* sV = sU + (long long)Kp * STR;             // [SC_TT][STR]\n"
          "  const long long plu = Cp * Kp, plv = Cp * Tp;\n"
          "  // U once per CTA: thread = one filter k (the blocked row offset computed once)\n"
          "  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {\n"
          "    const float* src = U + (long long)(k / bm) * Cp * bm + (k % bm);\n"
          "    float* dst = sU + (long long)k * STR;\n"
          "#pragma unroll 4\n"
          "    for (int pc = 0; pc < P * CW; ++pc) {\n"
          "      const int p = pc / CW, c = pc % CW;\n"
          "      dst[pc] = c < C ? src[p * plu + (long long)c * bm] : 0.f;\n"
          "    }\n"
          "  }\n"
          "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
          "  const int tl = warp * 8 + (lane & 7), k0 = lane >> 3;\n"
          "  // V staging: thread -> one tile column q and every (32 * NW / SC_TT)-th (p, c) row\n"
          "  const int sq = threadIdx.x % SC_TT, srow = threadIdx.x / SC_TT;\n"
          "#pragma unroll 1\n"
          "  for (int blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {\n"
          "    const long long t0 = (long long)blk * SC_TT;\n"
          "    __syncthreads();  // previous block's readers are done with sV\n"
          "    {\n"
          "      const long long ts = t0 + sq;\n"
          "      const bool ok = ts < Tp;\n"
          "      const float* src = V + (ok ? (ts / bn) * Cp * bn + (ts % bn) : 0);\n"
          "      float* dst = sV + sq * STR;\n"
          "#pragma unroll 4\n"
          "      for (int pc = srow; pc < P * CW; pc += 32 * NW / SC_TT) {\n"
          "        const int p = pc / CW, c = pc % CW;\n"
          "        dst[pc] = (ok && c < C) ? src[p * plv + (long long)c * bn] : 0.f;\n"
          "      }\n"
          "    }\n"
          "    __syncthreads();\n"
          "    const long long t = t0 + tl;\n"
          "    if (t >= T) continue;\n"
          "    const int per = th * tw;\n"
          "    const int img = (int)(t / per), rem = (int)(t - (long long)img * per);\n"
          "    const int ti = idiv_small(rem, tw, rtw), tj = rem - ti * tw;\n"
          "    const float* vp = sV + tl * STR;\n"
          "#pragma unroll 1\n"
          "    for (int k = k0; k < K; k += 4) {\n"
          "      const float* up = sU + (long long)k * STR;\n";
    // channel sums computed lazily, column by column, right before the left pass
    // consumes them (keeps the live set to one column of M + the left-pass results)
    Emitter em(os, false, ctr);
    std::vector<std::vector<std::string>> left(AT.rows, std::vector<std::string>(n));
    for (int b = 0; b < n; ++b) {
        std::vector<std::string> col(n);
        for (int a = 0; a < n; ++a) {
            col[a] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "      const float " << col[a] << " = sc_sum<C, PW, CW>(up + " << (a * n + b) << " * CW, vp + "
               << (a * n + b) << " * CW);\n";
        }
        auto res = em.apply(AT, col);
        for (int i = 0; i < AT.rows; ++i) left[i][b] = res[i];
    }
    std::vector<std::vector<std::string>> yv(AT.rows);
    for (int i = 0; i < AT.rows; ++i) yv[i] = em.apply(AT, left[i]);
    os << "      const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
          "      if (mode < 2) {\n"
          "        float* dst = out + (((long long)img * K + k) * Ho + y0) * Wo + x0;\n"
       << "        if (y0 + " << m << " <= Ho && x0 + " << m << " <= Wo) {\n";
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b)
            os << "          dst[" << a << " * Wo + " << b << "] = mode ? wino_relu(" << yv[a][b] << ") : " << yv[a][b]
               << ";\n";
    os << "        } else {\n";
    for (int a = 0; a < m; ++a) {
        os << "          if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "            if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = mode ? wino_relu("
               << yv[a][b] << ") : " << yv[a][b] << ";\n";
        os << "          }\n";
    }
    os << "        }\n        continue;\n      }\n";
    if (m % 2 == 0) {
        os << "      const int Hp = Ho >> 1, Wp = Wo >> 1, py0 = y0 >> 1, px0 = x0 >> 1;\n"
              "      float* dst = out + (((long long)img * K + k) * Hp + py0) * Wp + px0;\n";
        auto pv = [&](int a, int b) {
            return "wino_relu(fmaxf(fmaxf(" + yv[2 * a][2 * b] + ", " + yv[2 * a][2 * b + 1] + "), fmaxf(" +
                   yv[2 * a + 1][2 * b] + ", " + yv[2 * a + 1][2 * b + 1] + ")))";
        };
        os << "      if (py0 + " << m / 2 << " <= Hp && px0 + " << m / 2 << " <= Wp) {\n";
        for (int a = 0; a < m / 2; ++a)
            for (int b = 0; b < m / 2; ++b) os << "        dst[" << a << " * Wp + " << b << "] = " << pv(a, b) << ";\n";
        os << "      } else {\n";
        for (int a = 0; a < m / 2; ++a) {
            os << "        if (py0 + " << a << " < Hp) {\n";
            for (int b = 0; b < m / 2; ++b)
                os << "          if (px0 + " << b << " < Wp) dst[" << a << " * Wp + " << b << "] = " << pv(a, b)
                   << ";\n";
            os << "        }\n";
        }
        os << "      }\n";
    }
    os << "    }\n  }\n}\n";
    for (int C = 1; C <= 8; ++C)
        for (int pw = 0; pw < 2; ++pw)
            os << "extern \"C\" __global__ void __launch_bounds__(" << (C <= 4 ? 384 : 128) << ", 1) wino_smallc_c" << C
               << (pw ? "p" : "l")
               << "(\n    const float* __restrict__ U, const float* __restrict__ V, float* __restrict__ out, int K,\n"
                  "    int Ho, int Wo, int th, int tw, long long T, long long Tp, long long Kp, long long Cp, int bm,\n"
                  "    int bn, float rtw, float rth, int mode, int n_blocks) {\n"
               << "  sc_body<" << C << ", " << pw << ">(U, V, out, K, Ho, Wo, th, tw, T, Tp, Kp, Cp, bm, bn, rtw, rth,"
                  " mode, n_blocks);\n}\n";
    os << "\n";
}

// K3 + K4 (+ ReLU, + 2x2 max-pool) in one kernel for C <= 4 (an RGB first layer: VGG-16
// layer 1 moves 6 GB of M out to HBM and back in for 3 products per point).  Second design
// (the first, emit_smallc, spilled and was shared-memory bound):
//   * a CTA owns the bn tiles of one V block and all filters: U as sU[p][k/2][c][k%2] and the
//     block's V rows as sV[p][c][tile] are staged once with coalesced loads;
//   * a warp is 32 consecutive tiles (conflict-free V loads, the store pattern of the
//     gather K4) times one filter PAIR, so each V value loaded feeds two filters and the
//     filter operands are two broadcast loads per point: 2.5 shared-memory wavefronts per
//     (point, filter) against ~18 FP32-pipe cycles;
//   * channel sums are produced one column of the alpha x alpha point grid at a time and
//     consumed at once by the left pass of (A^T M) A, so the live set is the 2 x m x alpha
//     left-pass results, not 2 x alpha^2 sums;
//   * the channel sum is the contraction kernel's value bit for bit: the plan's linear order
//     ((-0 + z0) + z1 ... == (z0 + z1) ...), or the halving tree of the padded 8-channel stage
//     with its -0 leaves pruned (x + -0 == x exactly).
// KG warps-of-pairs per tile warp (tuning key "sc2_kg", default 2: 256 threads, no spills at
// 236 registers; 3 spills at the 168-register cap): threads = bn * KG.
inline int smallc2_kg() {
    static const int v = std::atoi(tuning("sc2_kg").c_str());
    return v >= 1 && v <= 8 ? v : 2;
}

static void emit_smallc2(std::ostringstream& os, int r, int m, const MatProg& AT, int bm, int bn, int& ctr) {
    const int n = r + m - 1, P = n * n, KG = smallc2_kg();
    if (bn % 32 || bm % 4 || bn * KG > 1024) return;
    const bool even = m % 2 == 0;
    // packed f32x2 helpers: lane 0 = filter 2kp, lane 1 = filter 2kp + 1 (the same arithmetic on two
    // independent filters; every product and every sum still rounds once, see Emitter `packed`)
    os << "typedef unsigned long long k2_t;\n"
          "static __device__ __forceinline__ k2_t k2_mul(k2_t a, k2_t b, k2_t nz2) {\n"
          "  k2_t r;\n  asm(\"fma.rn.f32x2 %0, %1, %2, %3;\" : \"=l\"(r) : \"l\"(a), \"l\"(b), \"l\"(nz2));\n  return r;\n}\n"
          "static __device__ __forceinline__ k2_t k2_add(k2_t a, k2_t b) {\n"
          "  k2_t r;\n  asm(\"add.rn.f32x2 %0, %1, %2;\" : \"=l\"(r) : \"l\"(a), \"l\"(b));\n  return r;\n}\n"
          "static __device__ __forceinline__ k2_t k2_sub(k2_t a, k2_t b) {\n"
          "  k2_t r;\n  asm(\"sub.rn.f32x2 %0, %1, %2;\" : \"=l\"(r) : \"l\"(a), \"l\"(b));\n  return r;\n}\n"
          "static __device__ __forceinline__ k2_t k2_dup(float a) {\n"
          "  k2_t r;\n  asm(\"mov.b64 %0, {%1, %1};\" : \"=l\"(r) : \"f\"(a));\n  return r;\n}\n"
          "static __device__ __forceinline__ float k2_lo(k2_t a) { return __uint_as_float((unsigned)a); }\n"
          "static __device__ __forceinline__ float k2_hi(k2_t a) { return __uint_as_float((unsigned)(a >> 32)); }\n"
          "template <int C, int PW>\n"
          "static __device__ __forceinline__ k2_t sc2_dot(k2_t u0, k2_t u1, k2_t u2, k2_t u3, float v0, float v1,\n"
          "                                               float v2, float v3, k2_t nz2) {\n"
          "  const k2_t z0 = k2_mul(u0, k2_dup(v0), nz2);\n"
          "  if constexpr (C == 1) return z0;\n"
          "  const k2_t z1 = k2_mul(u1, k2_dup(v1), nz2);\n"
          "  if constexpr (C == 2) return k2_add(z0, z1);\n"
          "  const k2_t z2 = k2_mul(u2, k2_dup(v2), nz2);\n"
          "  if constexpr (C == 3) return k2_add(k2_add(z0, z1), z2);\n"
          "  const k2_t z3 = k2_mul(u3, k2_dup(v3), nz2);\n"
          "  if constexpr (PW) return k2_add(k2_add(z0, z1), k2_add(z2, z3));\n"
          "  return k2_add(k2_add(k2_add(z0, z1), z2), z3);\n"
          "}\n";
    auto val = [&](int a, int b) { return "y" + std::to_string(a) + "_" + std::to_string(b); };
    // Store of one (tile, filter) result y[a][b] (registers).  MODE 0: y, 1: ReLU, 2: ReLU of the 2x2
    // max-pool.  MODE 0 / 1 with an even m and an even, 8-byte aligned output row (`coop`): the warp's
    // 32 tiles are consecutive, so one output row of the warp is (mostly) one contiguous run of
    // 32 x m floats; each lane parks its m x m values in the warp's shared-memory buffer and the
    // warp writes every row as m/2 fully coalesced 8-byte stores (lane l writes pair j*32 + l, whose
    // address and clipping -- soff / sy0 -- were computed once per thread).  Direct stores (8 bytes per
    // lane, 4 m bytes apart) touch every sector of the run m/2 times, and that request rate, not the
    // arithmetic, bounded the first version of this kernel.
    os << "template <int MODE>\n"
          "static __device__ __forceinline__ void sc2_store(float* __restrict__ out, bool coop, bool live, float2* wbuf,\n"
          "    int lane, const long long* soff, const int* sy0, int img, int K, int k, int Ho, int Wo, int y0, int x0";
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b) os << ", float y" << a << "_" << b;
    os << ") {\n"
          "  if constexpr (MODE < 2) {\n";
    if (even) {
        os << "    if (coop) {\n"
              "      float* ok = out + (long long)k * Ho * Wo;  // soff carries the image and the tile origin\n"
              "      __syncwarp();\n";
        for (int a = 0; a < m; ++a)
            for (int q = 0; q < m / 2; ++q)
                os << "      wbuf[(" << a << " * 32 + lane) * " << m / 2 << " + " << q << "] = MODE ? make_float2(wino_relu("
                   << val(a, 2 * q) << "), wino_relu(" << val(a, 2 * q + 1) << ")) : make_float2(" << val(a, 2 * q) << ", "
                   << val(a, 2 * q + 1) << ");\n";
        os << "      __syncwarp();\n";
        for (int a = 0; a < m; ++a)
            for (int j = 0; j < m / 2; ++j)
                os << "      if (sy0[" << j << "] + " << a << " < Ho) *reinterpret_cast<float2*>(ok + soff[" << j << "] + "
                   << a << " * Wo) = wbuf[" << (a * (m / 2) + j) << " * 32 + lane];\n";
        os << "      return;\n    }\n";
    }
    os << "    if (!live) return;\n"
          "    float* dst = out + ((((long long)img * K + k) * Ho + y0) * Wo + x0);\n";
    for (int a = 0; a < m; ++a) {
        os << "    if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "      if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = MODE ? wino_relu(" << val(a, b)
               << ") : " << val(a, b) << ";\n";
        os << "    }\n";
    }
    os << "  } else {\n";
    if (even) {
        os << "    if (!live) return;\n"
              "    const int Hp = Ho >> 1, Wp = Wo >> 1, py0 = y0 >> 1, px0 = x0 >> 1;\n"
              "    float* dst = out + ((((long long)img * K + k) * Hp + py0) * Wp + px0);\n";
        for (int a = 0; a < m / 2; ++a) {
            os << "    if (py0 + " << a << " < Hp) {\n";
            for (int b = 0; b < m / 2; ++b)
                os << "      if (px0 + " << b << " < Wp) dst[" << a << " * Wp + " << b << "] = wino_relu(fmaxf(fmaxf("
                   << val(2 * a, 2 * b) << ", " << val(2 * a, 2 * b + 1) << "), fmaxf(" << val(2 * a + 1, 2 * b) << ", "
                   << val(2 * a + 1, 2 * b + 1) << ")));\n";
            os << "    }\n";
        }
    }
    os << "  }\n}\n";
    os << "static __device__ __forceinline__ unsigned sc2_s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }\n"
          "static __device__ __forceinline__ void sc2_wait(unsigned long long* bar) {\n"
          "  asm volatile(\"{\\n\\t.reg .pred P1;\\nSC2_WAIT_%=:\\n\\t\"\n"
          "               \"mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\\n\\t\"\n"
          "               \"@!P1 bra SC2_WAIT_%=;\\n}\\n\" ::\"r\"(sc2_s32(bar)), \"r\"(0u) : \"memory\");\n"
          "}\n"
          "static __device__ __forceinline__ void sc2_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {\n"
          "  asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "               ::\"r\"(sc2_s32(dst)), \"l\"(src), \"r\"(bytes), \"r\"(sc2_s32(bar)) : \"memory\");\n"
          "}\n";
    os << "template <int C, int PW, int MODE>\n"
          "static __device__ __forceinline__ void sc2_body(const float* __restrict__ U, const float* __restrict__ V,\n"
          "    float* __restrict__ out, int K, int Ho, int Wo, int th, int tw, long long T, long long Tp, long long Kp,\n"
          "    long long Cp, k2_t nz2) {\n"
       << "  constexpr int N1 = " << n << ", P = " << P << ", M = " << m << ", BM = " << bm << ", BN = " << bn
       << ", KG = " << KG << ", HP = " << (even ? m / 2 : 1) << ";\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  __shared__ __align__(8) unsigned long long bar[N1];  // one per column of the point grid\n"
          "  const int KB = (int)(Kp / BM);\n"
          "  float* sU = reinterpret_cast<float*>(smem_raw);   // [P][KB][C][BM]: the first C rows of U's blocks\n"
          "  float* sV = sU + (long long)P * KB * C * BM;      // [P][C][BN]:     the first C rows of this V block\n"
          "  const long long plu = Cp * Kp, plv = Cp * Tp;\n"
          "  // Staging: one bulk copy per (point, U block) and per point of V, completing on the barrier of\n"
          "  // the point's column, so the first column's sums start while the rest streams in.\n"
          "  if (threadIdx.x == 0) {\n"
          "    for (int b = 0; b < N1; ++b)\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], %1;\" ::\"r\"(sc2_s32(&bar[b])), \"r\"(1u) : \"memory\");\n"
          "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
          "  }\n"
          "  __syncthreads();\n"
          "  if (threadIdx.x < 32) {\n"
          "    const float* vb = V + (long long)blockIdx.x * Cp * BN;\n"
          "    for (int b = 0; b < N1; ++b) {\n"
          "      if (threadIdx.x == 0)\n"
          "        asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" ::\"r\"(sc2_s32(&bar[b])),\n"
          "                     \"r\"((unsigned)(N1 * (KB * C * BM + C * BN) * 4)) : \"memory\");\n"
          "      __syncwarp();\n"
          "      for (int j = threadIdx.x; j < N1 * (KB + 1); j += 32) {\n"
          "        const int a = j / (KB + 1), kb = j - a * (KB + 1), p = a * N1 + b;\n"
          "        if (kb < KB)\n"
          "          sc2_bulk(sU + ((long long)p * KB + kb) * C * BM, U + p * plu + (long long)kb * Cp * BM, C * BM * 4, &bar[b]);\n"
          "        else\n"
          "          sc2_bulk(sV + p * C * BN, vb + p * plv, C * BN * 4, &bar[b]);\n"
          "      }\n"
          "    }\n"
          "  }\n"
          "  const int tl = threadIdx.x % BN, kg = threadIdx.x / BN, lane = threadIdx.x & 31;\n"
          "  const long long t = (long long)blockIdx.x * BN + tl;\n"
          "  const bool live = t < T;\n"
          "  const int per = th * tw;\n"
          "  int y0 = 0, x0 = 0, img = 0;\n"
          "  if (live) {\n"
          "    img = (int)(t / per);\n"
          "    const int rem = (int)(t - (long long)img * per), ti = rem / tw;\n"
          "    y0 = ti * M;\n"
          "    x0 = (rem - ti * tw) * M;\n"
          "  }\n"
          "  // warp-cooperative row stores (sc2_store): pair j * 32 + lane of a warp row belongs to lane ls\n"
          "  const bool coop = MODE < 2 && " << (even ? "true" : "false")
       << " && (Wo & 1) == 0 && (reinterpret_cast<size_t>(out) & 7) == 0;\n"
          "  float2* wbuf = reinterpret_cast<float2*>(sV + P * C * BN) + (threadIdx.x >> 5) * (M * 32 * HP);\n"
          "  long long soff[HP];\n"
          "  int sy0[HP];\n"
          "#pragma unroll\n"
          "  for (int j = 0; j < HP; ++j) {\n"
          "    const int i = j * 32 + lane, ls = i / HP, q = i - ls * HP;\n"
          "    const long long tt = t - lane + ls;\n"
          "    soff[j] = 0;\n"
          "    sy0[j] = Ho;\n"
          "    if (coop && tt < T) {\n"
          "      const int im = (int)(tt / per), rem = (int)(tt - (long long)im * per), ti = rem / tw;\n"
          "      const int xx = (rem - ti * tw) * M + 2 * q;\n"
          "      soff[j] = ((long long)im * K * Ho + ti * M) * Wo + xx;\n"
          "      if (xx < Wo) sy0[j] = ti * M;\n"
          "    }\n"
          "  }\n"
          "  const float* vp = sV + tl;\n"
          "  const int us = KB * C * BM;  // floats between the points of one filter\n"
          "  bool first = true;\n"
          "#pragma unroll 1\n"
          "  for (int kp = kg; 2 * kp < K; kp += KG) {\n"
          "    const float* up = sU + ((2 * kp) / BM) * C * BM + ((2 * kp) % BM);\n";
    Emitter em(os, false, ctr, /*packed=*/true);
    std::vector<std::vector<std::string>> left(AT.rows, std::vector<std::string>(n));
    for (int b = 0; b < n; ++b) {
        std::vector<std::string> col(n);
        os << "    if (first) sc2_wait(&bar[" << b << "]);\n";
        for (int a = 0; a < n; ++a) {
            const int p = a * n + b;
            const std::string s = std::to_string(a) + "_" + std::to_string(b);
            col[a] = "mm" + s;
            os << "    const k2_t ua" << s << " = *reinterpret_cast<const k2_t*>(up + " << p << " * us);\n"
               << "    const k2_t ub" << s << " = C > 1 ? *reinterpret_cast<const k2_t*>(up + " << p << " * us + BM) : 0ull;\n"
               << "    const k2_t uc" << s << " = C > 2 ? *reinterpret_cast<const k2_t*>(up + " << p << " * us + 2 * BM) : 0ull;\n"
               << "    const k2_t ud" << s << " = C > 3 ? *reinterpret_cast<const k2_t*>(up + " << p << " * us + 3 * BM) : 0ull;\n"
               << "    const float va" << s << " = vp[" << p << " * C * BN];\n"
               << "    const float vb" << s << " = C > 1 ? vp[(" << p << " * C + 1) * BN] : 0.f;\n"
               << "    const float vc" << s << " = C > 2 ? vp[(" << p << " * C + 2) * BN] : 0.f;\n"
               << "    const float vd" << s << " = C > 3 ? vp[(" << p << " * C + 3) * BN] : 0.f;\n"
               << "    const k2_t " << col[a] << " = sc2_dot<C, PW>(ua" << s << ", ub" << s << ", uc" << s << ", ud" << s
               << ", va" << s << ", vb" << s << ", vc" << s << ", vd" << s << ", nz2);\n";
            // keep the shared-memory loads of later points behind the sums of these (ptxas would hoist
            // all 64 points' operands and spill)
            if ((a + 1) % 2 == 0) os << "    asm volatile(\"\" ::: \"memory\");\n";
        }
        auto rr = em.apply(AT, col);
        for (int i = 0; i < AT.rows; ++i) left[i][b] = rr[i];
    }
    {
        std::vector<std::vector<std::string>> yv(AT.rows);
        for (int i = 0; i < AT.rows; ++i) yv[i] = em.apply(AT, left[i]);
        for (int half = 0; half < 2; ++half) {
            os << "    " << (half ? "if (2 * kp + 1 < K) " : "")
               << "sc2_store<MODE>(out, coop, live, wbuf, lane, soff, sy0, img, K, 2 * kp + " << half
               << ", Ho, Wo, y0, x0";
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) os << ", " << (half ? "k2_hi(" : "k2_lo(") << yv[a][b] << ")";
            os << ");\n";
        }
    }
    os << "    first = false;\n  }\n}\n";
    for (int C = 1; C <= 4; ++C)
        for (int pw = 0; pw < 2; ++pw)
            for (int mode = 0; mode < (even ? 3 : 2); ++mode)
                os << "extern \"C\" __global__ void __launch_bounds__(" << bn * KG << ", 1) wino_smallc2_c" << C
                   << (pw ? "p" : "l") << "_m" << mode
                   << "(\n    const float* __restrict__ U, const float* __restrict__ V, float* __restrict__ out, int K,\n"
                      "    int Ho, int Wo, int th, int tw, long long T, long long Tp, long long Kp, long long Cp,\n"
                      "    unsigned long long nz2) {\n"
                   << "  sc2_body<" << C << ", " << pw << ", " << mode
                   << ">(U, V, out, K, Ho, Wo, th, tw, T, Tp, Kp, Cp, nz2);\n}\n";
    os << "\n";
}

// K4 of layer i fused with K1 of layer i + 1 (conv stacks, fp32): a block owns PL whole (image,
// channel) planes of the activation between the two layers.  Phase 1 is the gather output transform
// of layer i (thread = tile: alpha^2 coalesced M loads, (A^T M) A, ReLU, optional 2x2 max-pool --
// the expressions of wino_output_gather_act) written to the planes in shared memory; phase 2 is
// the gather input transform of layer i + 1 (thread = tile: window from shared memory with the
// zero padding, (B^T d) B, V stores coalesced across tiles -- the expressions of
// input_gather_body).  The activation never goes to HBM: per (tile, channel) the pair moves
// alpha^2 + alpha^2 values instead of alpha^2 + m^2 and m^2 + alpha^2.  Planes are whole, so
// there is no halo between blocks.  Same rounded operations, hence the same bits, as the two
// kernels it replaces.  The kernel lives in the module of layer i + 1 (V blocking bn).
static void emit_k4k1(std::ostringstream& os, int r, int m, const MatProg& BT, const MatProg& AT, int bn, int& ctr) {
    const int n = r + m - 1, P = n * n;
    // Block order: KS consecutive filters innermost, then the plane groups, so the blocks resident at
    // one time read KS long contiguous runs of M (consecutive tiles of one filter) and write V in
    // runs of KS consecutive channels (2 KB for KS = 8) -- with the filter as the slow grid axis every
    // 256-byte V row landed 128 KB from the next one.
    os << "extern \"C\" __global__ void __launch_bounds__(128) wino_k4k1(\n"
          "    const float* __restrict__ Mm, float* __restrict__ V, int N, int PL, int pool, int K, int G, int KS,\n"
          "    int Ho, int Wo, int th, int tw, long long Tp, long long Kp,\n"
          "    int H2, int W2, int pad2, int th2, int tw2, long long T2, long long Tp2, long long Cp2) {\n"
          "  extern __shared__ __align__(16) float k41_plane[];  // [PL][H2][W2]\n"
          "  const int kk = blockIdx.x % KS, rest = blockIdx.x / KS, grp = rest % G;\n"
          "  const int k = (rest / G) * KS + kk, n0 = grp * PL;\n"
          "  if (k >= K) return;\n"
          "  const int np = N - n0 < PL ? N - n0 : PL;\n"
          "  const int per1 = th * tw, per2 = th2 * tw2, HW2 = H2 * W2;\n"
          "  const long long mplane = Kp * Tp;\n"
          "#pragma unroll 1\n"
          "  for (int q = threadIdx.x; q < np * per1; q += 128) {\n"
          "    const int pl = q / per1, rem = q - pl * per1, ti = rem / tw, tj = rem - ti * tw;\n"
          "    const float* src = Mm + (long long)k * Tp + (long long)n0 * per1 + q;\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "    const float " << mm[a][b] << " = __ldg(src + " << (a * n + b) << " * mplane);\n";
        }
    {
        Emitter em(os, false, ctr);
        auto yv = em.apply2d(AT, mm);
        os << "    float* dst = k41_plane + pl * HW2;\n"
           << "    const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
              "    if (!pool) {\n";
        for (int a = 0; a < m; ++a) {
            os << "      if (y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; ++b)
                os << "        if (x0 + " << b << " < Wo) dst[(y0 + " << a << ") * W2 + x0 + " << b << "] = wino_relu("
                   << yv[a][b] << ");\n";
            os << "      }\n";
        }
        os << "    } else {\n";
        if (m % 2 == 0) {
            os << "      const int py0 = y0 >> 1, px0 = x0 >> 1;\n";
            for (int a = 0; a < m / 2; ++a) {
                os << "      if (py0 + " << a << " < H2) {\n";
                for (int b = 0; b < m / 2; ++b)
                    os << "        if (px0 + " << b << " < W2) dst[(py0 + " << a << ") * W2 + px0 + " << b
                       << "] = wino_relu(fmaxf(fmaxf(" << yv[2 * a][2 * b] << ", " << yv[2 * a][2 * b + 1] << "), fmaxf("
                       << yv[2 * a + 1][2 * b] << ", " << yv[2 * a + 1][2 * b + 1] << ")));\n";
                os << "      }\n";
            }
        }
        os << "    }\n  }\n";
    }
    os << "  __syncthreads();\n"
          "  const long long vplane = Cp2 * Tp2;\n"
          "#pragma unroll 1\n"
          "  for (int q = threadIdx.x; q < np * per2; q += 128) {\n"
          "    const int pl = q / per2, rem = q - pl * per2, ti = rem / tw2, tj = rem - ti * tw2;\n"
          "    const long long t2 = (long long)n0 * per2 + q;\n"
       << "    float* op = V + ((t2 / " << bn << ") * Cp2 + k) * " << bn << " + (t2 % " << bn << ");\n"
       << "    const int h0 = ti * " << m << " - pad2, w0 = tj * " << m << " - pad2;\n"
          "    const float* sp = k41_plane + pl * HW2;\n";
    std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a) os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H2;\n";
    for (int b = 0; b < n; ++b) os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W2;\n";
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
            os << "    const float " << d[a][b] << " = (r" << a << " && c" << b << ") ? sp[(h0 + " << a << ") * W2 + (w0 + "
               << b << ")] : 0.f;\n";
        }
    {
        Emitter em(os, false, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "    op[" << (i * n + j) << " * vplane] = " << v[i][j] << ";\n";
    }
    os << "  }\n"
          "  // tiles padding T2 up to the contraction's tile: zeros, as K1 writes them\n"
          "  if (grp == G - 1)\n"
          "    for (long long tt = T2 + threadIdx.x; tt < Tp2; tt += 128) {\n"
       << "      float* op = V + ((tt / " << bn << ") * Cp2 + k) * " << bn << " + (tt % " << bn << ");\n"
       << "      for (int p = 0; p < " << P << "; ++p) op[p * vplane] = 0.f;\n"
          "    }\n"
          "}\n\n";
}

std::string gen_layer_source(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                             const GenTypes& ty, int bm, int bn) {
    const int n = r + m - 1, P = n * n;
    std::ostringstream os;
    os << header(ty);
    int ctr = 0;

    // Block size of K1 / K2 / K4: 128, fewer when the K1/K4 smem staging
    // buffer (P x TB values) would exceed 64 KB.
    const int es = ty.uv_double ? 8 : 4;
    int TB = 128;
    while (TB > 32 && (long long)P * TB * es > 64 * 1024) TB /= 2;
    const int VEC = 16 / es;  // values per 16-byte vector
    const char* VT = ty.uv_double ? "double2" : "float4";

    // ---------------- K2 body: U[p][k/bm][c][k%bm] = (G w[k,c] G^T)[p] ------------
    {
        os << "static __device__ __forceinline__ void filter_body(const in_t* __restrict__ w, uv_t* __restrict__ U,\n"
              "    int K, int C, long long Kp, long long Cp, int k, int c) {\n"
              "  if (k >= Kp) return;\n"
              "  const long long plane = Cp * Kp;\n"
           << "  uv_t* o = U + ((long long)(k / " << bm << ") * Cp + c) * " << bm << " + (k % " << bm << ");\n"
              "  if (k >= K || c >= C) {\n"
              "#pragma unroll 1\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * plane] = (uv_t)0;\n"
              "    return;\n  }\n"
           << "  const in_t* src = w + ((long long)k * C + c) * " << r * r << ";\n";
        std::vector<std::vector<std::string>> h(r, std::vector<std::string>(r));
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) {
                h[a][b] = "h" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << h[a][b] << " = (ct_t)__ldg(src + " << a * r + b << ");\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply2d(G, h);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                os << "  o[" << (i * n + j) << " * plane] = " << store_cvt(ty.compute_double, ty.uv_double, u[i][j])
                   << ";\n";
        os << "}\n\n";
    }

    // ---------------- K2, cooperative loads (large filters, r >= 5) ----------------
    // filter_body's r^2 loads each touch 32 different lines (consecutive threads are consecutive k, and
    // filters are C r^2 floats apart): at r = 5 the kernel is bound by L1 line requests, not bytes
    // (cfg4: 35 of the 55.6 us of K1 + K2).  Here the block first copies its 128 filters' r^2 weights to
    // shared memory with consecutive lanes on consecutive floats of a filter (about four lines per load
    // instruction), then every thread transforms its own filter from there (row stride r^2 | 1: no bank
    // conflicts).  Same arithmetic, same stores.  Grid (ceil(Kp / 128), Cp).
    if (128 * ((r * r) | 1) * (ty.in_double ? 8 : 4) <= 48 * 1024) {  // static shared memory (host: k2_coop())
        const int RR = r * r, RS = RR | 1;
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_filter_coop(\n"
              "    const in_t* __restrict__ w, uv_t* __restrict__ U, int K, int C, long long Kp, long long Cp) {\n"
           << "  __shared__ in_t fw[128 * " << RS << "];\n"
              "  const int k0 = blockIdx.x * 128, c = blockIdx.y, tid = threadIdx.x;\n"
              "  if (c < C) {\n"
              "#pragma unroll\n"
           << "    for (int q = 0; q < " << RR << "; ++q) {\n"
           << "      const int e = q * 128 + tid, ch = e / " << RR << ", off = e - ch * " << RR << ";\n"
           << "      fw[ch * " << RS << " + off] = k0 + ch < K ? __ldg(w + ((long long)(k0 + ch) * C + c) * " << RR
           << " + off) : (in_t)0;\n"
              "    }\n"
              "  }\n"
              "  __syncthreads();\n"
              "  const int k = k0 + tid;\n"
              "  if (k >= Kp) return;\n"
              "  const long long plane = Cp * Kp;\n"
           << "  uv_t* o = U + ((long long)(k / " << bm << ") * Cp + c) * " << bm << " + (k % " << bm << ");\n"
              "  if (k >= K || c >= C) {\n"
              "#pragma unroll 1\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * plane] = (uv_t)0;\n"
              "    return;\n  }\n";
        std::vector<std::vector<std::string>> h(r, std::vector<std::string>(r));
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) {
                h[a][b] = "g" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << h[a][b] << " = (ct_t)fw[tid * " << RS << " + " << a * r + b << "];\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply2d(G, h);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                os << "  o[" << (i * n + j) << " * plane] = " << store_cvt(ty.compute_double, ty.uv_double, u[i][j])
                   << ";\n";
        os << "}\n\n";
    }

    // ---------------- K1 body: V[p][t/bn][c][t%bn] = (B^T d B)[p] ------------
    // Each thread transforms one (tile, channel) window gathered from x (zero
    // padding fused; interior windows take an unpredicated fast path), parks its
    // P values in shared memory, and the block writes every p-row of its TB
    // tiles with 16-byte coalesced stores.
    {
        os << "static __device__ __forceinline__ void input_body(const in_t* __restrict__ x, uv_t* __restrict__ V,\n"
              "    uv_t* sv, int C, int H, int W, int pad, int th, int tw, long long T, long long Tp, long long Cp,\n"
              "    int t0, int c) {\n"
              "  const int t = t0 + threadIdx.x;\n"
              "  const long long plane = Cp * Tp;\n"
              "  if (c >= C || t >= T) {\n"
              "    const uv_t z = (c >= C) ? (uv_t)(-0.0) : (uv_t)0;\n"
              "#pragma unroll 1\n"
           << "    for (int p = 0; p < " << P << "; ++p) sv[p * " << TB << " + threadIdx.x] = z;\n"
              "  } else {\n"
              "  const int per = th * tw;\n"
              "  const int img = t / per;\n"
              "  const int rem = t - img * per;\n"
              "  const int ti = rem / tw, tj = rem - ti * tw;\n"
           << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
           << "  const in_t* src = x + ((long long)img * C + c) * ((long long)H * W);\n";
        std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "  ct_t " << d[a][b] << ";\n";
            }
        os << "  if (h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W) {\n"
           << "    const in_t* rp = src + h0 * W + w0;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * W + " << b << ");\n";
        os << "  } else {\n";
        for (int a = 0; a < n; ++a)
            os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
        for (int b = 0; b < n; ++b)
            os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + (h0 + " << a
                   << ") * W + (w0 + " << b << ")) : (ct_t)0;\n";
        os << "  }\n";
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                os << "  sv[" << (i * n + j) * TB << " + threadIdx.x] = "
                   << store_cvt(ty.compute_double, ty.uv_double, v[i][j]) << ";\n";
        os << "  }\n"
              "  __syncthreads();\n"
           << "  constexpr int NV = " << TB / VEC << ";\n"
           << "#pragma unroll 4\n"
           << "  for (int i = threadIdx.x; i < " << P << " * NV; i += " << TB << ") {\n"
           << "    const int p = i / NV, q = i - p * NV;\n"
           << "    const int tt = t0 + q * " << VEC << ";\n"
           << "    if (tt < Tp) {\n"
           << "      uv_t* o = V + p * plane + ((long long)(tt / " << bn << ") * Cp + c) * " << bn << " + (tt % " << bn
           << ");\n"
           << "      *reinterpret_cast<" << VT << "*>(o) = *reinterpret_cast<const " << VT << "*>(sv + p * " << TB
           << " + q * " << VEC << ");\n"
           << "    }\n  }\n"
           << "}\n\n";
    }

    // kernels: K2 alone, K1 alone, and K1+K2 in one launch (the filter
    // transform's blocks ride along with the input transform's)
    os << "extern \"C\" __global__ void __launch_bounds__(" << TB << ") wino_filter_xform(\n"
          "    const in_t* __restrict__ w, uv_t* __restrict__ U, int K, int C, long long Kp, long long Cp) {\n"
       << "  filter_body(w, U, K, C, Kp, Cp, blockIdx.x * " << TB << " + threadIdx.x, blockIdx.y);\n"
       << "}\n\n"
       << "extern \"C\" __global__ void __launch_bounds__(" << TB << ") wino_input_xform(\n"
          "    const in_t* __restrict__ x, uv_t* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp) {\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
       << "  input_body(x, V, reinterpret_cast<uv_t*>(smem_raw), C, H, W, pad, th, tw, T, Tp, Cp, blockIdx.x * " << TB
       << ", blockIdx.y);\n"
       << "}\n\n"
       << "extern \"C\" __global__ void __launch_bounds__(" << TB << ") wino_transforms(\n"
          "    const in_t* __restrict__ x, uv_t* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
          "    const in_t* __restrict__ w, uv_t* __restrict__ U, int K, long long Kp, int n_kb, int cfast) {\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  const int b = blockIdx.x;\n"
          "  const int n_in = n_tb * (int)Cp;\n"
          "  if (b < n_in) {\n"
          "    const int tb = cfast ? b / (int)Cp : b % n_tb, c = cfast ? b % (int)Cp : b / n_tb;\n"
       << "    input_body(x, V, reinterpret_cast<uv_t*>(smem_raw), C, H, W, pad, th, tw, T, Tp, Cp, tb * "
       << TB << ", c);\n"
          "  } else {\n"
          "    const int f = b - n_in;\n"
       << "    filter_body(w, U, K, C, Kp, Cp, (f % n_kb) * " << TB << " + threadIdx.x, f / n_kb);\n"
          "  }\n"
          "}\n\n";

    emit_input_gather(os, r, m, BT, ty, bn, TB, ctr);
    emit_output_kernel(os, r, m, AT, ty, TB, ctr);
    {
        const int es4 = ty.uv_double ? 8 : 4;
        int tbf = 128;
        while (tbf > 32 && (long long)P * tbf * es4 > 64 * 1024) tbf /= 2;
        emit_output_flat(os, r, m, AT, ty, tbf, ctr);
        emit_output_gather(os, r, m, AT, ty, 128, ctr);
        if (!ty.y_double) emit_output_gather_act(os, r, m, AT, ty, 128, ctr);
        emit_nhwc(os, r, m, BT, AT, ty, bn, ctr);
        if (!ty.compute_double && !ty.uv_double && !ty.y_double) {
            emit_smallc(os, r, m, AT, ty, ctr);
            emit_smallc2(os, r, m, AT, bm, bn, ctr);
            emit_k4k1(os, r, m, BT, AT, bn, ctr);
        }
    }
    return os.str();
}

// Output transform of ONE (filter k, tile t) pair from its alpha^2 point sums in registers
// (mr[a * n + b], raw fp32 bits), for the fused exact contraction (contract_template.cuh
// WINO_FUSE_P): (A^T M) A in the plan's order, crop, and the NCHW store -- omode 0: y,
// 1: ReLU, 2: ReLU of the 2x2 max-pool (even m; same expressions as wino_output_gather_act).
// fp32 plans only.  The text is prepended to the contraction template.
std::string gen_fused_out_source(int r, int m, const MatProg& AT) {
    const int n = r + m - 1;
    std::ostringstream os;
    int ctr = 0;
    os << "static __device__ __forceinline__ float wino_relu(float v) { return v > 0.f ? v : 0.f; }\n"
          "static __device__ __forceinline__ void wino_fused_out(const unsigned* mr, int k, int t,\n"
          "    float* __restrict__ out, int K, int Ho, int Wo, int th, int tw, int omode) {\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "  const float " << mm[a][b] << " = __uint_as_float(mr[" << (a * n + b) << "]);\n";
        }
    os << "  const int g = t / tw, tj = t - g * tw;\n"
          "  const int img = g / th, ti = g - img * th;\n"
       << "  const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n";
    Emitter em(os, false, ctr);
    auto yv = em.apply2d(AT, mm);
    os << "  if (omode < 2) {\n"
          "    float* dst = out + (((long long)img * K + k) * Ho + y0) * Wo + x0;\n";
    if (m % 2 == 0) {
        os << "    if ((Wo & 1) == 0 && (reinterpret_cast<size_t>(out) & 7) == 0) {\n";
        for (int a = 0; a < m; ++a) {
            os << "      if (y0 + " << a << " < Ho) {\n";
            for (int b = 0; b < m; b += 2)
                os << "        if (x0 + " << b << " < Wo) *reinterpret_cast<float2*>(dst + " << a << " * Wo + " << b
                   << ") = omode ? make_float2(wino_relu(" << yv[a][b] << "), wino_relu(" << yv[a][b + 1]
                   << ")) : make_float2(" << yv[a][b] << ", " << yv[a][b + 1] << ");\n";
            os << "      }\n";
        }
        os << "      return;\n    }\n";
    }
    for (int a = 0; a < m; ++a) {
        os << "    if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "      if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = omode ? wino_relu(" << yv[a][b]
               << ") : " << yv[a][b] << ";\n";
        os << "    }\n";
    }
    os << "    return;\n  }\n";
    if (m % 2 == 0) {
        os << "  const int Hp = Ho >> 1, Wp = Wo >> 1, py0 = y0 >> 1, px0 = x0 >> 1;\n"
              "  float* dst = out + (((long long)img * K + k) * Hp + py0) * Wp + px0;\n";
        for (int a = 0; a < m / 2; ++a) {
            os << "  if (py0 + " << a << " < Hp) {\n";
            for (int b = 0; b < m / 2; ++b)
                os << "    if (px0 + " << b << " < Wp) dst[" << a << " * Wp + " << b << "] = wino_relu(fmaxf(fmaxf("
                   << yv[2 * a][2 * b] << ", " << yv[2 * a][2 * b + 1] << "), fmaxf(" << yv[2 * a + 1][2 * b] << ", "
                   << yv[2 * a + 1][2 * b + 1] << ")));\n";
            os << "  }\n";
        }
    }
    os << "}\n\n";
    return os.str();
}

std::string gen_tile_source(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                            const GenTypes& ty) {
    const int n = r + m - 1, P = n * n;
    std::ostringstream os;
    os << header(ty);
    int ctr = 0;
    const char* MULW = ty.uv_double ? "__dmul_rn" : "__fmul_rn";

    // hadamard_2d: z[bc][p] = (G h G^T) o (B^T x B)
    {
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_tile_h2d(\n"
              "    const in_t* __restrict__ h, const in_t* __restrict__ x, uv_t* __restrict__ z, long long BC) {\n"
              "  const long long i = (long long)blockIdx.x * 128 + threadIdx.x;\n"
              "  if (i >= BC) return;\n"
           << "  const in_t* hs = h + i * " << r * r << ";\n"
           << "  const in_t* xs = x + i * " << P << ";\n"
           << "  uv_t* o = z + i * " << P << ";\n";
        std::vector<std::vector<std::string>> hv(r, std::vector<std::string>(r)), xv(n, std::vector<std::string>(n));
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) {
                hv[a][b] = "h" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << hv[a][b] << " = (ct_t)hs[" << a * r + b << "];\n";
            }
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                xv[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << xv[a][b] << " = (ct_t)xs[" << a * n + b << "];\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply2d(G, hv);
        auto v = em.apply2d(BT, xv);
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "  o[" << a * n + b << "] = " << MULW << "(" << store_cvt(ty.compute_double, ty.uv_double, u[a][b])
                   << ", " << store_cvt(ty.compute_double, ty.uv_double, v[a][b]) << ");\n";
        os << "}\n\n";
    }
    // output_2d: out[b] = A^T y A
    {
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_tile_o2d(\n"
              "    const uv_t* __restrict__ yin, y_t* __restrict__ out, long long B) {\n"
              "  const long long i = (long long)blockIdx.x * 128 + threadIdx.x;\n"
              "  if (i >= B) return;\n"
           << "  const uv_t* s = yin + i * " << P << ";\n"
           << "  y_t* o = out + i * " << m * m << ";\n";
        std::vector<std::vector<std::string>> yv(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                yv[a][b] = "y" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << yv[a][b] << " = (ct_t)s[" << a * n + b << "];\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto res = em.apply2d(AT, yv);
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b)
                os << "  o[" << a * m + b << "] = " << store_cvt(ty.compute_double, ty.y_double, res[a][b]) << ";\n";
        os << "}\n\n";
    }
    // hadamard_1d: z[bc][i] = (G h)[i] * (B^T x)[i]
    {
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_tile_h1d(\n"
              "    const in_t* __restrict__ h, const in_t* __restrict__ x, uv_t* __restrict__ z, long long BC) {\n"
              "  const long long i = (long long)blockIdx.x * 128 + threadIdx.x;\n"
              "  if (i >= BC) return;\n"
           << "  const in_t* hs = h + i * " << r << ";\n"
           << "  const in_t* xs = x + i * " << n << ";\n"
           << "  uv_t* o = z + i * " << n << ";\n";
        std::vector<std::string> hv(r), xv(n);
        for (int a = 0; a < r; ++a) {
            hv[a] = "h" + std::to_string(a);
            os << "  const ct_t " << hv[a] << " = (ct_t)hs[" << a << "];\n";
        }
        for (int a = 0; a < n; ++a) {
            xv[a] = "x" + std::to_string(a);
            os << "  const ct_t " << xv[a] << " = (ct_t)xs[" << a << "];\n";
        }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply(G, hv);
        auto v = em.apply(BT, xv);
        for (int a = 0; a < n; ++a)
            os << "  o[" << a << "] = " << MULW << "(" << store_cvt(ty.compute_double, ty.uv_double, u[a]) << ", "
               << store_cvt(ty.compute_double, ty.uv_double, v[a]) << ");\n";
        os << "}\n\n";
    }
    // output_1d
    {
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_tile_o1d(\n"
              "    const uv_t* __restrict__ yin, y_t* __restrict__ out, long long B) {\n"
              "  const long long i = (long long)blockIdx.x * 128 + threadIdx.x;\n"
              "  if (i >= B) return;\n"
           << "  const uv_t* s = yin + i * " << n << ";\n"
           << "  y_t* o = out + i * " << m << ";\n";
        std::vector<std::string> yv(n);
        for (int a = 0; a < n; ++a) {
            yv[a] = "y" + std::to_string(a);
            os << "  const ct_t " << yv[a] << " = (ct_t)s[" << a << "];\n";
        }
        Emitter em(os, ty.compute_double, ctr);
        auto res = em.apply(AT, yv);
        for (int a = 0; a < m; ++a)
            os << "  o[" << a << "] = " << store_cvt(ty.compute_double, ty.y_double, res[a]) << ";\n";
        os << "}\n";
    }
    return os.str();
}

// ---------------------------------------------------------------------------
// Tensor-core (K3t) variant of K1/K2: U and V written as 16-bit (BF16 / FP16)
// operands directly in the canonical UMMA K-major no-swizzle layout, blocked
// by the tc contraction's 128-row tiles and 32-channel stages:
//   X16[p][rowblock][c/32][(c/8)%4][row%128 / 8][row%8][c%8]
// (one stage of one tile = 8 KB contiguous = one bulk copy).  The transforms
// themselves are the same straight-line FP32/FP64 code; only the final store
// rounds to 16 bits (FP32 first in mixed mode).
// Fused K3t + K4 for the tensor-core modes (P * NK <= 512): one persistent CTA
// per SM walks (128-tile, NK-filter) blocks.  All P Winograd-point GEMMs of a
// block accumulate side by side in TMEM (point p in columns [p NK, p NK + NK),
// rows = tiles), so the epilogue holds every point of a (tile, filter) pair
// and applies the output transform right out of TMEM: M never reaches HBM.
//   warp 0      producer: one cp.async.bulk for the V stage (P x 128 x 16,
//               contiguous) and one for the U stage (P x NK x 16) per
//               16-channel step, ST-deep smem ring (mbarrier complete_tx)
//   warp 1      one thread issues P tcgen05.mma (M=128, N=NK, K=16) per
//               stage; tcgen05.commit frees the stage / publishes the block
//   warps 2-5   epilogue: tcgen05.ld (32 lanes = 32 tiles per warp) of every
//               point for KC filters, (A^T M) A in registers, crop, NCHW store
static void emit_tcf_kernel(std::ostringstream& os, int r, int m, const MatProg& AT, const GenTypes& ty, bool fp16,
                            int NK, int& ctr) {
    const int n = r + m - 1, P = n * n;
    const int VST = P * 4096, UST = P * NK * 32, STB = VST + UST;
    const int ST = std::max(1, std::min(4, (232448 - 256) / STB));
    const int KC = P <= 16 ? 8 : 4;  // filters per tcgen05.ld batch (P x KC registers)
    const int NB = 2 * P * NK <= 512 ? 2 : 1;  // TMEM accumulator sets (2: epilogue overlaps the next block)
    const char* PT = ty.y_double ? "double2" : "float2";
    os << "typedef unsigned long long tcf_u64;\n"
          "static __device__ __forceinline__ unsigned tcf_s(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }\n"
          "static __device__ __forceinline__ void tcf_wait(tcf_u64* b, unsigned parity) {\n"
          "  asm volatile(\"{\\n\\t.reg .pred P1;\\nTCF_WAIT_%=:\\n\\t\"\n"
          "               \"mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\\n\\t\"\n"
          "               \"@!P1 bra TCF_WAIT_%=;\\n}\\n\" :: \"r\"(tcf_s(b)), \"r\"(parity) : \"memory\");\n"
          "}\n"
          "static __device__ __forceinline__ tcf_u64 tcf_desc(unsigned addr, unsigned lbo, unsigned sbo) {\n"
          "  return (tcf_u64)((addr >> 4) & 0x3FFF) | ((tcf_u64)((lbo >> 4) & 0x3FFF) << 16) |\n"
          "         ((tcf_u64)((sbo >> 4) & 0x3FFF) << 32) | ((tcf_u64)1 << 46);\n"
          "}\n\n";
    os << "extern \"C\" __global__ void __launch_bounds__(192, 1) wino_tcf(\n"
          "    const unsigned short* __restrict__ U, const unsigned short* __restrict__ V, y_t* __restrict__ y,\n"
          "    int K, int Ho, int Wo, int th, int tw, long long T, long long Tp, long long Kp, long long Cp,\n"
          "    int n_tiles, float rtw, float rth, int dbg) {\n"
       << "  constexpr int P = " << P << ", NK = " << NK << ", ST = " << ST << ", KC = " << KC << ", NB = " << NB
       << ";\n"
       << "  constexpr unsigned VST = " << VST << "u, UST = " << UST << "u, STB = " << STB << "u;\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
          "  tcf_u64* full = reinterpret_cast<tcf_u64*>(smem + ST * STB);\n"
          "  tcf_u64* empty = full + ST;\n"
          "  tcf_u64* acc_full = empty + ST;\n"
          "  tcf_u64* acc_empty = acc_full + NB;\n"
          "  unsigned* tmem_slot = reinterpret_cast<unsigned*>(acc_empty + NB);\n"
          "  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;\n"
          "  const int nk = (int)(Cp >> 4), n_kb = (int)(Kp / NK);\n"
          "  if (tid == 0) {\n"
          "    for (int s = 0; s < ST; ++s) {\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(tcf_s(&full[s])) : \"memory\");\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(tcf_s(&empty[s])) : \"memory\");\n"
          "    }\n"
          "    for (int b = 0; b < NB; ++b) {\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 1;\" :: \"r\"(tcf_s(&acc_full[b])) : \"memory\");\n"
          "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], 4;\" :: \"r\"(tcf_s(&acc_empty[b])) : \"memory\");\n"
          "    }\n"
          "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
          "  }\n"
          "  if (warp == 1) {  // all 512 TMEM columns: P x NK fp32 accumulators x 128 lanes\n"
          "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\" :: \"r\"(tcf_s(tmem_slot)) : \"memory\");\n"
          "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\" ::: \"memory\");\n"
          "  }\n"
          "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n"
          "  __syncthreads();\n"
          "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
          "  const unsigned tmem = *tmem_slot;\n"
          "  if (warp == 0) {\n"
          "    if (lane == 0) {  // producer\n"
          "      int g = 0;\n"
          "      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {\n"
          "        const int kb = tile % n_kb, tb = tile / n_kb;\n"
          "        const unsigned short* gV = V + (long long)tb * nk * (VST / 2);\n"
          "        const unsigned short* gU = U + (long long)kb * nk * (UST / 2);\n"
          "        for (int kt = 0; kt < nk; ++kt, ++g) {\n"
          "          const int s = g % ST;\n"
          "          if (g >= ST) tcf_wait(&empty[s], (unsigned)(((g / ST) - 1) & 1));\n"
          "          unsigned char* dst = smem + s * STB;\n"
          "          asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(tcf_s(&full[s])), \"r\"(STB) : \"memory\");\n"
          "          asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "                       :: \"r\"(tcf_s(dst)), \"l\"(gV + (long long)kt * (VST / 2)), \"r\"(VST), \"r\"(tcf_s(&full[s])) : \"memory\");\n"
          "          asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\"\n"
          "                       :: \"r\"(tcf_s(dst + VST)), \"l\"(gU + (long long)kt * (UST / 2)), \"r\"(UST), \"r\"(tcf_s(&full[s])) : \"memory\");\n"
          "        }\n"
          "      }\n"
          "    }\n"
          "  } else if (warp == 1) {\n"
          "    if (lane == 0) {  // MMA issuer: D[t][k] += V_p[t][c] U_p[k][c] for every point p\n"
       << "      const unsigned idesc = (1u << 4) | (" << (fp16 ? 0 : 1) << "u << 7) | (" << (fp16 ? 0 : 1)
       << "u << 10) | ((unsigned)(NK >> 3) << 17) | (8u << 24);\n"
          "      int g = 0, it = 0;\n"
          "      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {\n"
          "        const int ab = it % NB;\n"
          "        if (it >= NB) tcf_wait(&acc_empty[ab], (unsigned)(((it / NB) - 1) & 1));\n"
          "        asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
          "        for (int kt = 0; kt < nk; ++kt, ++g) {\n"
          "          const int s = g % ST;\n"
          "          tcf_wait(&full[s], (unsigned)((g / ST) & 1));\n"
          "          asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
          "          const unsigned a0 = tcf_s(smem + s * STB), b0 = a0 + VST;\n"
          "#pragma unroll\n"
          "          for (int p = 0; p < P; ++p) {\n"
          "            if (dbg & 1) break;\n"
          "            const tcf_u64 da = tcf_desc(a0 + p * 4096, 2048, 128);\n"
          "            const tcf_u64 db = tcf_desc(b0 + p * (NK * 32), NK * 16, 128);\n"
          "            asm volatile(\"{\\n\\t.reg .pred q;\\n\\tsetp.ne.b32 q, %4, 0;\\n\\t\"\n"
          "                         \"tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\\n\\t}\\n\"\n"
          "                         :: \"r\"(tmem + (unsigned)(ab * 256 + p * NK)), \"l\"(da), \"l\"(db), \"r\"(idesc), \"r\"((unsigned)kt) : \"memory\");\n"
          "          }\n"
          "          asm volatile(\"tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\" :: \"r\"(tcf_s(&empty[s])) : \"memory\");\n"
          "        }\n"
          "        asm volatile(\"tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\" :: \"r\"(tcf_s(&acc_full[ab])) : \"memory\");\n"
          "      }\n"
          "    }\n"
          "  } else {\n"
          "    // epilogue: warp (2..5) % 4 selects TMEM lanes = tiles [32 q4, 32 q4 + 32) of the block\n"
          "    const int q4 = warp & 3;\n"
          "    int it = 0;\n"
          "    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {\n"
          "      const int kb = tile % n_kb, tb = tile / n_kb;\n"
          "      const int ab = it % NB;\n"
          "      tcf_wait(&acc_full[ab], (unsigned)((it / NB) & 1));\n"
          "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
          "      const int t0 = tb * 128;\n"
          "      const int t = t0 + q4 * 32 + lane;\n"
          "      const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
          "      const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
          "      const int off = off0 + q4 * 32 + lane;\n"
          "      const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
          "      const int di = idiv_small(ti0 + kk, th, rth);\n"
          "      const int ti = ti0 + kk - di * th;\n"
       << "      const int y0 = ti * " << m << ", x0 = tj * " << m << ";\n"
       << "      const bool live = t < T;\n"
          "      const bool inner = y0 + " << m << " <= Ho && x0 + " << m << " <= Wo;\n"
          "      y_t* ybase = y + ((long long)(img0 + di) * K) * Ho * Wo + (long long)y0 * Wo + x0;\n"
          "      const unsigned trow = tmem + ((unsigned)(q4 * 32) << 16) + (unsigned)(ab * 256);\n"
          "#pragma unroll 1\n"
          "      for (int kc = 0; kc < ((dbg & 2) ? 0 : NK); kc += KC) {\n"
          "        unsigned rr[P][KC];\n"
          "#pragma unroll\n"
          "        for (int p = 0; p < P; ++p) {\n";
    if (KC == 8)
        os << "          asm volatile(\"tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\"\n"
              "                       : \"=r\"(rr[p][0]), \"=r\"(rr[p][1]), \"=r\"(rr[p][2]), \"=r\"(rr[p][3]),\n"
              "                         \"=r\"(rr[p][4]), \"=r\"(rr[p][5]), \"=r\"(rr[p][6]), \"=r\"(rr[p][7])\n"
              "                       : \"r\"(trow + (unsigned)(p * NK + kc)));\n";
    else
        os << "          asm volatile(\"tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\"\n"
              "                       : \"=r\"(rr[p][0]), \"=r\"(rr[p][1]), \"=r\"(rr[p][2]), \"=r\"(rr[p][3])\n"
              "                       : \"r\"(trow + (unsigned)(p * NK + kc)));\n";
    os << "        }\n"
          "        asm volatile(\"tcgen05.wait::ld.sync.aligned;\" ::: \"memory\");\n"
          "#pragma unroll\n"
          "        for (int j = 0; j < KC; ++j) {\n"
          "          const int k = kb * NK + kc + j;\n"
          "          if (!live || k >= K || (dbg & 4)) continue;\n";
    std::vector<std::vector<std::string>> mm(n, std::vector<std::string>(n));
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            mm[a][b] = "m" + std::to_string(a) + "_" + std::to_string(b);
            os << "          const ct_t " << mm[a][b] << " = (ct_t)__uint_as_float(rr[" << a * n + b << "][j]);\n";
        }
    Emitter em(os, ty.compute_double, ctr);
    auto yv = em.apply2d(AT, mm);
    auto val = [&](int a, int b) { return store_cvt(ty.compute_double, ty.y_double, yv[a][b]); };
    os << "          y_t* dst = ybase + (long long)k * Ho * Wo;\n"
          "          if (inner) {\n";
    if (m % 2 == 0) {
        os << "            if ((Wo & 1) == 0) {\n";
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; b += 2)
                os << "              *reinterpret_cast<" << PT << "*>(dst + " << a << " * Wo + " << b << ") = make_" << PT
                   << "(" << val(a, b) << ", " << val(a, b + 1) << ");\n";
        os << "            } else {\n";
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) os << "              dst[" << a << " * Wo + " << b << "] = " << val(a, b) << ";\n";
        os << "            }\n";
    } else {
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) os << "            dst[" << a << " * Wo + " << b << "] = " << val(a, b) << ";\n";
    }
    os << "          } else {\n";
    for (int a = 0; a < m; ++a) {
        os << "            if (y0 + " << a << " < Ho) {\n";
        for (int b = 0; b < m; ++b)
            os << "              if (x0 + " << b << " < Wo) dst[" << a << " * Wo + " << b << "] = " << val(a, b) << ";\n";
        os << "            }\n";
    }
    os << "          }\n"
          "        }\n"
          "      }\n"
          "      asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n"
          "      __syncwarp();\n"
          "      if (lane == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(tcf_s(&acc_empty[ab])) : \"memory\");\n"
          "    }\n"
          "  }\n"
          "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n"
          "  __syncthreads();\n"
          "  if (warp == 1) {\n"
          "    asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n"
          "    asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\" :: \"r\"(tmem) : \"memory\");\n"
          "  }\n"
          "}\n\n";
}

std::string gen_layer_source_tc(int r, int m, const MatProg& G, const MatProg& BT, const MatProg& AT,
                                const GenTypes& ty, bool fp16, int fused_nk) {
    const int n = r + m - 1, P = n * n;
    std::ostringstream os;
    os << header(ty)
       << "static __device__ __forceinline__ unsigned short to16(float v) {\n"
       << "  unsigned short h;\n"
       << "  asm(\"cvt.rn." << (fp16 ? "f16" : "bf16") << ".f32 %0, %1;\" : \"=h\"(h) : \"f\"(v));\n"
       << "  return h;\n}\n"
       << "static __device__ __forceinline__ long long tc_off(long long row, long long c, long long Cp) {\n"
       << "  return ((row >> 7) * (Cp >> 5) + (c >> 5)) * 4096 + ((c >> 3) & 3) * 1024 + (row & 127) * 8 + (c & 7);\n"
       << "}\n";
    // Operand layouts written by the gather transforms.  Unfused (K3t kernel,
    // tc_contract.cu): X16[p][row/128][c/32][(c/8)%4][(row%128)/8][row%8][c%8],
    // p-stride = rows x Cp.  Fused (wino_tcf below): every pipeline stage of a
    // (128-tile | NK-filter, 16-channel) block holds all P points contiguously,
    //   V16[t/128][c/16][p][(c/8)%2][(t%128)/8][t%8][c%8]      (p-stride 2048)
    //   U16[k/NK][c/16][p][(c/8)%2][(k%NK)/8][k%8][c%8]         (p-stride 16 NK)
    if (fused_nk) {
        const int NK = fused_nk;
        os << "static __device__ __forceinline__ long long tc_voff(long long t, long long c, long long Cp) {\n"
           << "  return ((t >> 7) * (Cp >> 4) + (c >> 4)) * " << P * 2048
           << "LL + ((c >> 3) & 1) * 1024 + (t & 127) * 8 + (c & 7);\n}\n"
           << "static __device__ __forceinline__ long long tc_uoff(long long k, long long c, long long Cp) {\n"
           << "  return ((k / " << NK << ") * (Cp >> 4) + (c >> 4)) * " << (long long)P * NK * 16 << "LL + ((c >> 3) & 1) * "
           << NK * 8 << " + (k % " << NK << ") * 8 + (c & 7);\n}\n"
           << "static __device__ __forceinline__ long long tc_vstride(long long, long long) { return 2048; }\n"
           << "static __device__ __forceinline__ long long tc_ustride(long long, long long) { return " << NK * 16
           << "; }\n";
    } else {
        os << "static __device__ __forceinline__ long long tc_voff(long long t, long long c, long long Cp) {\n"
              "  return tc_off(t, c, Cp);\n}\n"
              "static __device__ __forceinline__ long long tc_uoff(long long k, long long c, long long Cp) {\n"
              "  return tc_off(k, c, Cp);\n}\n"
              "static __device__ __forceinline__ long long tc_vstride(long long Cp, long long Tp) { return Cp * Tp; }\n"
              "static __device__ __forceinline__ long long tc_ustride(long long Cp, long long Kp) { return Cp * Kp; }\n";
    }
    const std::string cv = ty.compute_double ? "to16(__double2float_rn(" : "to16((";
    int ctr = 0;
    // filter: one thread per (k, c)
    {
        os << "static __device__ __forceinline__ void filter_tc(const in_t* __restrict__ w, unsigned short* __restrict__ U,\n"
              "    int K, int C, long long Kp, long long Cp, int k, int c) {\n"
              "  if (k >= Kp || c >= Cp) return;\n"
              "  const long long plane = Cp * Kp;\n"
              "  unsigned short* o = U + tc_off(k, c, Cp);\n"
              "  if (k >= K || c >= C) {\n"
              "#pragma unroll 1\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * plane] = 0;\n"
              "    return;\n  }\n"
           << "  const in_t* src = w + ((long long)k * C + c) * " << r * r << ";\n";
        std::vector<std::vector<std::string>> h(r, std::vector<std::string>(r));
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) {
                h[a][b] = "h" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << h[a][b] << " = (ct_t)__ldg(src + " << a * r + b << ");\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply2d(G, h);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "  o[" << (i * n + j) << " * plane] = " << cv << u[i][j] << "));\n";
        os << "}\n\n";
    }
    // input: block = 64 tiles x 8 channels, P x 64 x 8 16-bit values staged in smem
    {
        os << "static __device__ __forceinline__ void input_tc(const in_t* __restrict__ x, unsigned short* __restrict__ V,\n"
              "    unsigned short* sv, int C, int H, int W, int pad, int th, int tw, long long T, long long Tp,\n"
              "    long long Cp, int t0, int c0) {\n"
              "  const int t = t0 + threadIdx.x;\n"
              "  const long long plane = Cp * Tp;\n"
              "  const int per = th * tw;\n"
              "  const int img = t / per;\n"
              "  const int rem = t - img * per;\n"
              "  const int ti = rem / tw, tj = rem - ti * tw;\n"
           << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
           << "  const bool inner = h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W;\n"
           << "#pragma unroll 1\n"
              "  for (int cc = 0; cc < 8; ++cc) {\n"
              "    const int c = c0 + cc;\n"
              "    unsigned short* so = sv + threadIdx.x * 8 + cc;\n"
              "    if (c >= C || t >= T) {\n"
              "#pragma unroll 1\n"
           << "      for (int p = 0; p < " << P << "; ++p) so[p * 512] = 0;\n"
              "      continue;\n    }\n"
              "    const in_t* src = x + ((long long)img * C + c) * ((long long)H * W);\n";
        std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "    ct_t " << d[a][b] << ";\n";
            }
        os << "    if (inner) {\n      const in_t* rp = src + h0 * W + w0;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "      " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * W + " << b << ");\n";
        os << "    } else {\n";
        for (int a = 0; a < n; ++a)
            os << "      const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
        for (int b = 0; b < n; ++b)
            os << "      const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "      " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + (h0 + " << a
                   << ") * W + (w0 + " << b << ")) : (ct_t)0;\n";
        os << "    }\n";
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "    so[" << (i * n + j) * 512 << "] = " << cv << v[i][j] << "));\n";
        os << "  }\n"
              "  __syncthreads();\n"
           << "  // 16-byte rows (8 channels of one tile): consecutive threads -> consecutive rows\n"
           << "#pragma unroll 4\n"
           << "  for (int i = threadIdx.x; i < " << P << " * 64; i += 64) {\n"
           << "    const int p = i >> 6, tl = i & 63;\n"
           << "    const long long row = (long long)t0 + tl;\n"
           << "    *reinterpret_cast<uint4*>(V + p * plane + tc_off(row, c0, Cp)) =\n"
           << "        *reinterpret_cast<const uint4*>(sv + (long long)i * 8);\n"
           << "  }\n}\n\n";
    }
    os << "extern \"C\" __global__ void __launch_bounds__(64) wino_filter_xform(\n"
          "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, int C, long long Kp, long long Cp) {\n"
          "  filter_tc(w, U, K, C, Kp, Cp, blockIdx.x * 64 + threadIdx.x, blockIdx.y);\n"
          "}\n\n"
          "extern \"C\" __global__ void __launch_bounds__(64) wino_input_xform(\n"
          "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp) {\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  input_tc(x, V, reinterpret_cast<unsigned short*>(smem_raw), C, H, W, pad, th, tw, T, Tp, Cp,\n"
          "           blockIdx.x * 64, blockIdx.y * 8);\n"
          "}\n\n"
          "extern \"C\" __global__ void __launch_bounds__(64) wino_transforms(\n"
          "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
          "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, long long Kp, int n_kb, int cfast) {\n"
          "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
          "  const int b = blockIdx.x;\n"
          "  const int ncg = (int)(Cp / 8);\n"
          "  const int n_in = n_tb * ncg;\n"
          "  if (b < n_in) {\n"
          "    const int tb = cfast ? b / ncg : b % n_tb, cg = cfast ? b % ncg : b / n_tb;\n"
          "    input_tc(x, V, reinterpret_cast<unsigned short*>(smem_raw), C, H, W, pad, th, tw, T, Tp, Cp,\n"
          "             tb * 64, cg * 8);\n"
          "  } else {\n"
          "    const int f = b - n_in;\n"
          "    filter_tc(w, U, K, C, Kp, Cp, (f % n_kb) * 64 + threadIdx.x, f / n_kb);\n"
          "  }\n}\n\n";
    // gather forms (default): warp = 4 tiles (or filters) x 8 channels, lane
    // (c & 7) of row t -> a warp's 16-bit store of one p fills 4 consecutive
    // 16-byte rows of the canonical layout (64 contiguous bytes, whole
    // sectors) straight from registers, no smem park.  Block = 32 rows x 8
    // channels; grid (row chunks [input, then filter], Cp / 8).
    {
        os << "static __device__ __forceinline__ void filter_tcg(const in_t* __restrict__ w, unsigned short* __restrict__ U,\n"
              "    int K, int C, long long Kp, long long Cp, int k, int c) {\n"
              "  const long long plane = tc_ustride(Cp, Kp);\n"
              "  unsigned short* o = U + tc_uoff(k, c, Cp);\n"
              "  if (k >= K || c >= C) {\n"
              "#pragma unroll\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * plane] = 0;\n"
              "    return;\n  }\n"
           << "  const in_t* src = w + ((long long)k * C + c) * " << r * r << ";\n";
        std::vector<std::vector<std::string>> h(r, std::vector<std::string>(r));
        for (int a = 0; a < r; ++a)
            for (int b = 0; b < r; ++b) {
                h[a][b] = "h" + std::to_string(a) + "_" + std::to_string(b);
                os << "  const ct_t " << h[a][b] << " = (ct_t)__ldg(src + " << a * r + b << ");\n";
            }
        Emitter em(os, ty.compute_double, ctr);
        auto u = em.apply2d(G, h);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "  o[" << (i * n + j) << " * plane] = " << cv << u[i][j] << "));\n";
        os << "}\n\n";
    }
    {
        os << "static __device__ __forceinline__ void input_tcg(const in_t* __restrict__ x, unsigned short* __restrict__ V,\n"
              "    int C, int H, int W, int pad, int th, int tw, long long T, long long Tp, long long Cp,\n"
              "    float rtw, float rth, int t0, int c) {\n"
              "  const long long plane = tc_vstride(Cp, Tp);\n"
              "  const int tl = ((threadIdx.x >> 5) << 2) + ((threadIdx.x >> 3) & 3);\n"
              "  const int t = t0 + tl;\n"
              "  unsigned short* o = V + tc_voff(t, c, Cp);\n"
              "  if (c >= C || t >= T) {\n"
              "#pragma unroll\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * plane] = 0;\n"
              "    return;\n"
              "  }\n"
              "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
              "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
              "  const int off = off0 + tl;\n"
              "  const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
              "  const int di = idiv_small(ti0 + kk, th, rth);\n"
              "  const int ti = ti0 + kk - di * th;\n"
           << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
           << "  const in_t* src = x + ((long long)(img0 + di) * C + c) * ((long long)H * W);\n";
        std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "  ct_t " << d[a][b] << ";\n";
            }
        os << "  if (h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W) {\n"
           << "    const in_t* rp = src + h0 * W + w0;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * W + " << b << ");\n";
        os << "  } else {\n";
        for (int a = 0; a < n; ++a)
            os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
        for (int b = 0; b < n; ++b)
            os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + (h0 + " << a
                   << ") * W + (w0 + " << b << ")) : (ct_t)0;\n";
        os << "  }\n";
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "  o[" << (i * n + j) << " * plane] = " << cv << v[i][j] << "));\n";
        os << "}\n\n";
    }
    // 16 < P <= 96 (alpha = 5..9): thread = one tile x one channel with a WARP = 32 consecutive
    // tiles of one channel, so the window loads coalesce like the fp32 gather kernel's (the
    // 4-tiles x 8-channels map of input_tcg touches 8 image planes per load instruction).  The
    // 16-bit results are parked in shared memory as [p][channel pair 0..3][tile 0..31][channel & 1]
    // (a warp's store of one p: one 16-bit half per bank, conflict-free; the write-out reads whole
    // 32-bit channel pairs, lanes on consecutive banks) and the block then writes every p's 32 rows
    // of the canonical layout -- 16 bytes (8 channels) per row, 512 contiguous bytes per warp
    // store.  Block = 256 threads = 32 tiles x 8 channels, P x 512 bytes of shared memory.
    const bool staged_k1 = P > 16 && P <= 96 && tuning("k1tc_staged") != "0";
    if (staged_k1) {
        os << "static __device__ __forceinline__ void input_tcs(const in_t* __restrict__ x, unsigned short* __restrict__ V,\n"
              "    int C, int H, int W, int pad, int th, int tw, long long T, long long Tp, long long Cp,\n"
              "    float rtw, float rth, int t0, int c0) {\n"
           << "  __shared__ __align__(16) unsigned short park[" << P << " * 256];\n"
              "  const long long plane = tc_vstride(Cp, Tp);\n"
              "  const int tl = threadIdx.x & 31, cl = threadIdx.x >> 5;\n"
              "  const int t = t0 + tl, c = c0 + cl;\n"
              "  unsigned short* pk = park + ((cl >> 1) * 32 + tl) * 2 + (cl & 1);\n"
              "  if (c >= C || t >= T) {\n"
              "#pragma unroll\n"
           << "    for (int p = 0; p < " << P << "; ++p) pk[p * 256] = 0;\n"
              "  } else {\n"
              "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
              "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
              "  const int off = off0 + tl;\n"
              "  const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
              "  const int di = idiv_small(ti0 + kk, th, rth);\n"
              "  const int ti = ti0 + kk - di * th;\n"
           << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
           << "  const in_t* src = x + ((long long)(img0 + di) * C + c) * ((long long)H * W);\n";
        std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "  ct_t " << d[a][b] << ";\n";
            }
        os << "  const bool interior = h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W;\n";
        if (m % 2 == 0 && !ty.in_double) {
            // even m: 8-byte row loads from the even column at or below w0 (as in input_gather_body)
            for (int sh = 0; sh < 2; ++sh) {
                const int nl = (n + sh + 1) / 2;
                os << "  " << (sh == 0 ? "if" : "else if") << " (interior && (W & 1) == 0 && (pad & 1) == " << sh
                   << " && (reinterpret_cast<size_t>(src) & 7) == 0) {\n"
                   << "    const float2* rp = reinterpret_cast<const float2*>(src + h0 * W + w0 - " << sh << ");\n"
                   << "    const int W2 = W >> 1;\n";
                for (int a = 0; a < n; ++a) {
                    for (int q = 0; q < nl; ++q)
                        os << "    const float2 f" << a << "_" << q << " = __ldg(rp + " << a << " * W2 + " << q << ");\n";
                    for (int b = 0; b < n; ++b) {
                        const int e = b + sh;
                        os << "    " << d[a][b] << " = (ct_t)f" << a << "_" << e / 2 << (e % 2 ? ".y" : ".x") << ";\n";
                    }
                }
                os << "  }\n";
            }
            os << "  else if (interior) {\n";
        } else {
            os << "  if (interior) {\n";
        }
        os << "    const in_t* rp = src + h0 * W + w0;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * W + " << b << ");\n";
        os << "  } else {\n";
        for (int a = 0; a < n; ++a)
            os << "    const bool r" << a << " = (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
        for (int b = 0; b < n; ++b)
            os << "    const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "    " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + (h0 + " << a
                   << ") * W + (w0 + " << b << ")) : (ct_t)0;\n";
        os << "  }\n";
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) os << "  pk[" << (i * n + j) << " * 256] = " << cv << v[i][j] << "));\n";
        os << "  }\n"
              "  __syncthreads();\n"
              "  // write-out: item = (p, tile): 8 channels gathered from the park, one 16-byte row\n"
              "  uint4* o = reinterpret_cast<uint4*>(V + tc_voff(t0 + tl, c0, Cp));\n"
              "#pragma unroll 4\n"
           << "  for (int p = cl; p < " << P << "; p += 8) {\n"
              "    const unsigned* q = reinterpret_cast<const unsigned*>(park + p * 256) + tl;\n"
              "    o[p * (plane >> 3)] = make_uint4(q[0], q[32], q[64], q[96]);\n"
              "  }\n"
              "}\n\n";
    }
    // P <= 16: thread = one tile x 8 channels, the 8 transformed values of
    // each p packed in registers and written as one 16-byte row of the
    // canonical layout (a warp of 32 consecutive tiles stores 512 contiguous
    // bytes); the window loads keep the one-channel-per-warp coalescing of
    // the fp32 gather kernel.  Block = 128 tiles; grid (row chunks, Cp / 8).
    if (P <= 16) {
        os << "static __device__ __forceinline__ void input_tcg8(const in_t* __restrict__ x, unsigned short* __restrict__ V,\n"
              "    int C, int H, int W, int pad, int th, int tw, long long T, long long Tp, long long Cp,\n"
              "    float rtw, float rth, int t0, int c0) {\n"
              "  const long long plane = tc_vstride(Cp, Tp);\n"
              "  const int t = t0 + threadIdx.x;\n"
              "  uint4* o = reinterpret_cast<uint4*>(V + tc_voff(t, c0, Cp));\n"
           << "  unsigned pk[" << P << "][4];\n"
           << "  if (t >= T) {\n"
              "#pragma unroll\n"
           << "    for (int p = 0; p < " << P << "; ++p) o[p * (plane >> 3)] = make_uint4(0u, 0u, 0u, 0u);\n"
              "    return;\n"
              "  }\n"
              "  const int g0 = t0 / tw, off0 = t0 - g0 * tw;\n"
              "  const int img0 = g0 / th, ti0 = g0 - img0 * th;\n"
              "  const int off = off0 + threadIdx.x;\n"
              "  const int kk = idiv_small(off, tw, rtw), tj = off - kk * tw;\n"
              "  const int di = idiv_small(ti0 + kk, th, rth);\n"
              "  const int ti = ti0 + kk - di * th;\n"
           << "  const int h0 = ti * " << m << " - pad, w0 = tj * " << m << " - pad;\n"
           << "  const bool inner = h0 >= 0 && w0 >= 0 && h0 + " << n << " <= H && w0 + " << n << " <= W;\n"
           << "  const in_t* base = x + ((long long)(img0 + di) * C + c0) * ((long long)H * W);\n"
              "#pragma unroll\n"
              "  for (int cc = 0; cc < 8; ++cc) {\n"
              "    const in_t* src = base + (long long)cc * H * W;\n"
              "    const bool live = c0 + cc < C;\n";
        std::vector<std::vector<std::string>> d(n, std::vector<std::string>(n));
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                d[a][b] = "x" + std::to_string(a) + "_" + std::to_string(b);
                os << "    ct_t " << d[a][b] << ";\n";
            }
        os << "    if (live && inner) {\n      const in_t* rp = src + h0 * W + w0;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "      " << d[a][b] << " = (ct_t)__ldg(rp + " << a << " * W + " << b << ");\n";
        os << "    } else {\n";
        for (int a = 0; a < n; ++a)
            os << "      const bool r" << a << " = live && (unsigned)(h0 + " << a << ") < (unsigned)H;\n";
        for (int b = 0; b < n; ++b)
            os << "      const bool c" << b << " = (unsigned)(w0 + " << b << ") < (unsigned)W;\n";
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b)
                os << "      " << d[a][b] << " = (r" << a << " && c" << b << ") ? (ct_t)__ldg(src + (h0 + " << a
                   << ") * W + (w0 + " << b << ")) : (ct_t)0;\n";
        os << "    }\n";
        Emitter em(os, ty.compute_double, ctr);
        auto v = em.apply2d(BT, d);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const int p = i * n + j;
                os << "    {\n      const unsigned hv = live ? (unsigned)" << cv << v[i][j] << ")) : 0u;\n"
                   << "      if (cc & 1) pk[" << p << "][cc >> 1] |= hv << 16; else pk[" << p << "][cc >> 1] = hv;\n"
                   << "    }\n";
            }
        os << "  }\n"
              "#pragma unroll\n"
           << "  for (int p = 0; p < " << P << "; ++p) o[p * (plane >> 3)] = make_uint4(pk[p][0], pk[p][1], pk[p][2], pk[p][3]);\n"
              "}\n\n";
        os << "extern \"C\" __global__ void __launch_bounds__(128) wino_input_tcg8(\n"
              "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, float rtw, float rth) {\n"
              "  input_tcg8(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 128, blockIdx.y * 8);\n"
              "}\n\n"
              "extern \"C\" __global__ void __launch_bounds__(128) wino_transforms_tcg8(\n"
              "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
              "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, long long Kp, float rtw, float rth) {\n"
              "  if ((int)blockIdx.x < n_tb) {\n"
              "    input_tcg8(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 128, blockIdx.y * 8);\n"
              "  } else {\n"
              "    // filters: 4 per warp x 8 channels, as in wino_transforms_tcg (128 threads = 16 filters)\n"
              "    const int k = ((int)blockIdx.x - n_tb) * 16 + ((threadIdx.x >> 5) << 2) + ((threadIdx.x >> 3) & 3);\n"
              "    if (k < Kp) filter_tcg(w, U, K, C, Kp, Cp, k, blockIdx.y * 8 + (threadIdx.x & 7));\n"
              "  }\n"
              "}\n\n";
    }
    os << "extern \"C\" __global__ void __launch_bounds__(256) wino_input_tcg(\n"
          "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp, float rtw, float rth) {\n"
          "  input_tcg(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 32, blockIdx.y * 8 + (threadIdx.x & 7));\n"
          "}\n\n"
          "extern \"C\" __global__ void __launch_bounds__(256) wino_transforms_tcg(\n"
          "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
          "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
          "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, long long Kp, float rtw, float rth) {\n"
          "  const int c = blockIdx.y * 8 + (threadIdx.x & 7);\n"
          "  if ((int)blockIdx.x < n_tb) {\n"
          "    input_tcg(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 32, c);\n"
          "  } else {\n"
          "    const int k = ((int)blockIdx.x - n_tb) * 32 + ((threadIdx.x >> 5) << 2) + ((threadIdx.x >> 3) & 3);\n"
          "    if (k < Kp) filter_tcg(w, U, K, C, Kp, Cp, k, c);\n"
          "  }\n"
          "}\n\n"
          "extern \"C\" __global__ void __launch_bounds__(256) wino_filter_tcg(\n"
          "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, int C, long long Kp, long long Cp) {\n"
          "  const int k = (int)blockIdx.x * 32 + ((threadIdx.x >> 5) << 2) + ((threadIdx.x >> 3) & 3);\n"
          "  if (k < Kp) filter_tcg(w, U, K, C, Kp, Cp, k, blockIdx.y * 8 + (threadIdx.x & 7));\n"
          "}\n\n";
    // minimum blocks per SM of the staged K1 (register cap; tuning key k1tc_blocks)
    // (f64 transforms -- mixed precision -- hold the window in twice the registers: no cap there)
    const int tcs_blocks = std::atoi(tuning("k1tc_blocks").c_str()) > 0 ? std::atoi(tuning("k1tc_blocks").c_str())
                           : ty.compute_double ? 1 : 3;
    if (staged_k1)  // same grids and arguments as the *_tcg kernels; the host picks by image size
        os << "extern \"C\" __global__ void __launch_bounds__(256, " << tcs_blocks << ") wino_input_tcs(\n"
              "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, float rtw, float rth) {\n"
              "  input_tcs(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 32, blockIdx.y * 8);\n"
              "}\n\n"
           << "extern \"C\" __global__ void __launch_bounds__(256, " << tcs_blocks << ") wino_transforms_tcs(\n"
              "    const in_t* __restrict__ x, unsigned short* __restrict__ V, int C, int H, int W, int pad, int th,\n"
              "    int tw, long long T, long long Tp, long long Cp, int n_tb,\n"
              "    const in_t* __restrict__ w, unsigned short* __restrict__ U, int K, long long Kp, float rtw, float rth) {\n"
              "  if ((int)blockIdx.x < n_tb) {\n"
              "    input_tcs(x, V, C, H, W, pad, th, tw, T, Tp, Cp, rtw, rth, blockIdx.x * 32, blockIdx.y * 8);\n"
              "  } else {\n"
              "    const int k = ((int)blockIdx.x - n_tb) * 32 + ((threadIdx.x >> 5) << 2) + ((threadIdx.x >> 3) & 3);\n"
              "    if (k < Kp) filter_tcg(w, U, K, C, Kp, Cp, k, blockIdx.y * 8 + (threadIdx.x & 7));\n"
              "  }\n"
              "}\n\n";
    int TB = 128;
    while (TB > 32 && (long long)P * TB * 4 > 64 * 1024) TB /= 2;
    emit_output_kernel(os, r, m, AT, ty, TB, ctr, "float", 4);
    emit_output_flat(os, r, m, AT, ty, TB, ctr, "float", 4);
    emit_output_gather(os, r, m, AT, ty, 128, ctr, "float");
    // conv stacks in the tensor-core modes: K4 + ReLU (+ max-pool) in one kernel, as in the exact path
    if (!ty.y_double) emit_output_gather_act(os, r, m, AT, ty, 128, ctr, "float");
    if (fused_nk) emit_tcf_kernel(os, r, m, AT, ty, fp16, fused_nk, ctr);
    return os.str();
}

}  // namespace wino
