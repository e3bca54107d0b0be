// csrc_bench — benchmark and verification harness for the B200 CSRC products,
// the GPU counterpart of the reference's `bench` tool (tools/bench_main.cpp:
// run / verify / info subcommands, the same flags and the same CSV / JSON
// report fields, BenchReport bench.hpp:24-55).
//
// Matrix sources (bench_main.cpp:16-89):
//   --matrix PATH         Matrix Market coordinate file (matrix_market.hpp:15-85)
//   --gen KIND:k=v,...    dense:n= | band:n=,h=,valsym= | random_sym:n=,density=,seed=,valsym=
//                         (generate.hpp:12-65: same std::mt19937_64 / uniform_real_distribution
//                         draws, so the matrices equal the reference's)
//   --config c1..c5       the BASELINE FE fixtures (extension)
//   --symmetrize          pad missing transposes / diagonals with explicit zeros
// Triplets -> CSR -> CSRC run on the GPU (csrc_gpu_build_csr / csrc_gpu_csr_to_csrc);
// the symmetry analysis (symmetry.hpp:17-45) walks the host CSR.
//
// Strategies: the reference's seq / buffers / colorful, plus the GPU kinds
// gather / windowed / atomic. Timing: `reps` products per run on the device
// (x, y resident, CUDA events; --host-vectors times the host API with the
// copies), `runs` runs, median run reported; speedup_vs_seq_csrc is relative
// to the seq strategy on the same device (bench.hpp:160-275).
//
// verify (bench_main.cpp:173-266) checks every strategy against the harness's
// own product of the full CSR on the host (dense two-loop for n <= 2000,
// sequential CSR otherwise), at the reference's 1e-12 inf-norm bound
// (relative_error, bench.hpp:93-100). That host product is the checker, never
// a result path: every reported y comes from the GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/csrc_gpu.h"

namespace {

using index_t = int32_t;
using count_t = int64_t;

struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct UsageError : std::runtime_error {
    explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};

void ck(int rc) {
    if (rc != 0) throw Error(csrc_gpu_last_error());
}

struct Triplets {
    index_t n_rows = 0, n_cols = 0;
    std::vector<index_t> r, c;
    std::vector<double> v;
    void add(index_t i, index_t j, double x) {
        r.push_back(i);
        c.push_back(j);
        v.push_back(x);
    }
};

struct Csr {
    index_t n_rows = 0, n_cols = 0;
    std::vector<index_t> rp, ci;
    std::vector<double> va;
    bool has(index_t i, index_t j) const {
        auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
        return std::binary_search(b, e, j);
    }
    double at(index_t i, index_t j) const {
        auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
        auto it = std::lower_bound(b, e, j);
        return (it == e || *it != j) ? 0.0 : va[static_cast<size_t>(it - ci.begin())];
    }
};

struct Csrc {
    index_t n = 0;
    std::vector<double> ad, al, au;
    std::vector<index_t> ia, ja;
    bool value_symmetric = false;
    csrc_host_matrix view() const {
        csrc_host_matrix m{};
        m.n = n;
        m.k = static_cast<int64_t>(ja.size());
        m.ad = ad.data();
        m.ia = ia.data();
        m.ja = ja.data();
        m.al = al.data();
        m.au = value_symmetric ? nullptr : au.data();
        m.value_symmetric = value_symmetric ? 1 : 0;
        return m;
    }
    count_t k() const { return static_cast<count_t>(ja.size()); }
    count_t nnz_full() const { return n + 2 * k(); }
    count_t nnz_stored() const { return n + (value_symmetric ? 1 : 2) * k(); }
};

// ------------------------------------------------------------ Matrix Market
// Coordinate reader with the reference's rules and messages
// (matrix_market.hpp:15-85): real / integer / pattern fields; general,
// symmetric, skew-symmetric (expanded; skew stores no diagonal); 1-based.
Triplets read_matrix_market(std::istream& in) {
    std::string line;
    long ln = 0;
    auto fail = [&](const std::string& what) {
        return Error("matrix market, line " + std::to_string(ln) + ": " + what);
    };
    if (!std::getline(in, line)) throw Error("matrix market: empty stream");
    ++ln;
    std::istringstream head(line);
    std::string magic, object, format, field, sym;
    head >> magic >> object >> format >> field >> sym;
    if (magic != "%%MatrixMarket") throw fail("missing %%MatrixMarket banner");
    if (object != "matrix") throw fail("unsupported object '" + object + "'");
    if (format != "coordinate") throw fail("only coordinate format is supported");
    if (field != "real" && field != "integer" && field != "pattern")
        throw fail("unsupported field '" + field + "'");
    if (sym != "general" && sym != "symmetric" && sym != "skew-symmetric")
        throw fail("unsupported symmetry '" + sym + "'");
    const bool pattern = field == "pattern", mirror = sym != "general", skew = sym == "skew-symmetric";
    long nr = 0, nc = 0, nnz = 0;
    for (;;) {
        if (!std::getline(in, line)) throw fail("missing size line");
        ++ln;
        if (!line.empty() && line[0] == '%') continue;
        std::istringstream ss(line);
        if (ss >> nr >> nc >> nnz) break;
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        throw fail("malformed size line '" + line + "'");
    }
    if (nr < 0 || nc < 0 || nnz < 0) throw fail("negative size");
    Triplets t;
    t.n_rows = static_cast<index_t>(nr);
    t.n_cols = static_cast<index_t>(nc);
    for (long seen = 0; seen < nnz;) {
        if (!std::getline(in, line))
            throw fail("expected " + std::to_string(nnz) + " entries, got " + std::to_string(seen));
        ++ln;
        if (line.empty() || line[0] == '%' || line.find_first_not_of(" \t\r") == std::string::npos) continue;
        std::istringstream ss(line);
        long i = 0, j = 0;
        double x = 1.0;
        if (!(ss >> i >> j)) throw fail("malformed entry '" + line + "'");
        if (!pattern && !(ss >> x)) throw fail("missing value in '" + line + "'");
        if (i < 1 || i > nr || j < 1 || j > nc)
            throw fail("index (" + std::to_string(i) + ", " + std::to_string(j) + ") outside declared bounds");
        ++seen;
        const index_t a = static_cast<index_t>(i - 1), b = static_cast<index_t>(j - 1);
        if (skew && a == b) throw fail("skew-symmetric file stores a diagonal entry");
        t.add(a, b, x);
        if (mirror && a != b) t.add(b, a, skew ? -x : x);
    }
    return t;
}

// ---------------------------------------------------------------- generators
// generate.hpp:12-65; the random family draws from the same standard-library
// engine and distributions in the same order, so with libstdc++ the triplets
// are identical to the reference's.
Triplets gen_dense(index_t n) {
    if (n < 1) throw Error("generate_dense: n must be >= 1");
    Triplets t;
    t.n_rows = t.n_cols = n;
    for (index_t i = 0; i < n; ++i)
        for (index_t j = 0; j < n; ++j) t.add(i, j, 1.0 + ((31 * i + 17 * j) % 13) * 0.25);
    return t;
}

Triplets gen_band(index_t n, index_t h, bool vs) {
    if (n < 1) throw Error("generate_band: n must be >= 1");
    if (h < 0 || h >= n) throw Error("generate_band: need 0 <= half-width < n");
    Triplets t;
    t.n_rows = t.n_cols = n;
    for (index_t i = 0; i < n; ++i) {
        t.add(i, i, 4.0 + (i % 5) * 0.5);
        for (index_t j = std::max<index_t>(0, i - h); j < i; ++j) {
            const double lo = -1.0 + ((7 * i + 3 * j) % 11) * 0.1;
            t.add(i, j, lo);
            t.add(j, i, vs ? lo : -1.0 + ((7 * j + 3 * i) % 11) * 0.1);
        }
    }
    return t;
}

Triplets gen_random_sym(index_t n, double density, uint64_t seed, bool vs) {
    if (n < 1) throw Error("generate_random_sym: n must be >= 1");
    if (density < 0.0 || density > 1.0) throw Error("generate_random_sym: density in [0, 1]");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0), val(-1.0, 1.0);
    Triplets t;
    t.n_rows = t.n_cols = n;
    for (index_t i = 0; i < n; ++i) {
        t.add(i, i, 2.0 + coin(rng));
        for (index_t j = 0; j < i; ++j) {
            if (coin(rng) >= density) continue;
            const double lo = val(rng);
            const double up = vs ? lo : val(rng);
            t.add(i, j, lo);
            t.add(j, i, up);
        }
    }
    return t;
}

// ------------------------------------------------------------ GPU builders
int g_device = 0;

Csr build_csr(const Triplets& t) {
    csrc_built_t h = nullptr;
    ck(csrc_gpu_build_csr(t.n_rows, t.n_cols, static_cast<int64_t>(t.v.size()), t.r.data(), t.c.data(),
                          t.v.data(), g_device, &h));
    Csr a;
    int32_t nr = 0, nc = 0;
    int64_t nnz = 0;
    const int32_t *rp = nullptr, *ci = nullptr;
    const double* va = nullptr;
    const int rc = csrc_built_csr(h, &nr, &nc, &nnz, &rp, &ci, &va);
    if (rc == 0) {
        a.n_rows = nr;
        a.n_cols = nc;
        a.rp.assign(rp, rp + nr + 1);
        a.ci.assign(ci, ci + nnz);
        a.va.assign(va, va + nnz);
    }
    csrc_built_free(h);
    ck(rc);
    return a;
}

Csrc csr_to_csrc(const Csr& a) {
    csrc_built_t h = nullptr;
    ck(csrc_gpu_csr_to_csrc(a.n_rows, a.n_cols, a.rp.data(), a.ci.data(), a.va.data(), g_device, &h));
    csrc_host_matrix m{};
    const int rc = csrc_built_matrix(h, &m);
    Csrc c;
    if (rc == 0) {
        c.n = m.n;
        c.ad.assign(m.ad, m.ad + m.n);
        c.ia.assign(m.ia, m.ia + m.n + 1);
        c.ja.assign(m.ja, m.ja + m.k);
        c.al.assign(m.al, m.al + m.k);
        if (!m.value_symmetric) c.au.assign(m.au, m.au + m.k);
        c.value_symmetric = m.value_symmetric != 0;
    }
    csrc_built_free(h);
    ck(rc);
    return c;
}

// symmetry.hpp:17-45 (analysis) and :50-61 (zero padding), host CSR walk
struct Symmetry {
    bool structural = false;
    count_t missing_transposes = 0, missing_diagonal = 0;
};

Symmetry analyze_symmetry(const Csr& a) {
    Symmetry s;
    for (index_t i = 0; i < a.n_rows; ++i) {
        bool diag = false;
        for (index_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const index_t j = a.ci[k];
            if (j == i) diag = true;
            else if (!a.has(j, i)) ++s.missing_transposes;
        }
        if (!diag) ++s.missing_diagonal;
    }
    s.structural = s.missing_transposes == 0 && s.missing_diagonal == 0;
    return s;
}

Csr symmetrize_pattern(const Csr& a) {
    Triplets t;
    t.n_rows = a.n_rows;
    t.n_cols = a.n_cols;
    for (index_t i = 0; i < a.n_rows; ++i)
        for (index_t k = a.rp[i]; k < a.rp[i + 1]; ++k) t.add(i, a.ci[k], a.va[k]);
    for (index_t i = 0; i < a.n_rows; ++i) {
        if (!a.has(i, i)) t.add(i, i, 0.0);
        for (index_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const index_t j = a.ci[k];
            if (j != i && !a.has(j, i)) t.add(j, i, 0.0);
        }
    }
    return build_csr(t);
}

// ------------------------------------------------------------- the source
struct Source {
    std::string path, gen, config;
    bool symmetrize = false;

    std::string param_or(const std::string& key, const std::string& dflt) const {
        const auto colon = gen.find(':');
        if (colon == std::string::npos) return dflt;
        std::istringstream ss(gen.substr(colon + 1));
        std::string kv;
        while (std::getline(ss, kv, ',')) {
            const auto eq = kv.find('=');
            if (eq != std::string::npos && kv.substr(0, eq) == key) return kv.substr(eq + 1);
        }
        return dflt;
    }
    std::string kind() const { return gen.substr(0, gen.find(':')); }

    std::string name() const {
        if (!config.empty()) return config;
        if (!gen.empty()) return kind() == "dense" ? "dense_" + param_or("n", "0") : kind();
        const auto slash = path.find_last_of('/');
        std::string base = slash == std::string::npos ? path : path.substr(slash + 1);
        const auto dot = base.rfind('.');
        return dot == std::string::npos ? base : base.substr(0, dot);
    }

    Triplets triplets() const {
        if (!gen.empty()) {
            auto gi = [&](const char* k, long d) { return std::stol(param_or(k, std::to_string(d))); };
            auto gd = [&](const char* k, double d) { return std::stod(param_or(k, std::to_string(d))); };
            const std::string k = kind();
            if (k == "dense") return gen_dense(static_cast<index_t>(gi("n", 1000)));
            if (k == "band") return gen_band(static_cast<index_t>(gi("n", 1000)), static_cast<index_t>(gi("h", 1)),
                                             gi("valsym", 0) != 0);
            if (k == "random_sym")
                return gen_random_sym(static_cast<index_t>(gi("n", 100)), gd("density", 0.05),
                                      static_cast<uint64_t>(gi("seed", 1)), gi("valsym", 0) != 0);
            throw Error("unknown generator kind '" + k + "'");
        }
        std::ifstream in(path);
        if (!in) throw Error("cannot open '" + path + "'");
        return read_matrix_market(in);
    }

    Csr csr() const {
        if (!config.empty()) {
            // BASELINE fixture -> its CSR (csrc_to_csr triplets)
            static const std::map<std::string, csrc_fixture_spec> specs = {
                {"c1", {CSRC_MESH_GRID2D_Q1, 256, 256, 1, 42, 10.0, 0}},
                {"c2", {CSRC_MESH_GRID3D_27, 64, 64, 64, 7, 30.0, 0}},
                {"c3", {CSRC_MESH_GRID3D_27_RCM, 160, 160, 160, 11, 30.0, 0}},
                {"c4", {CSRC_MESH_ELASTICITY, 96, 96, 96, 3, 100.0, 0}},
                {"c5", {CSRC_MESH_GRID3D_27, 256, 256, 256, 99, 30.0, 0}}};
            auto it = specs.find(config);
            if (it == specs.end()) throw UsageError("--config must be one of c1..c5");
            csrc_fixture_t fx = nullptr;
            ck(csrc_fixture_generate(&it->second, &fx));
            csrc_host_matrix m{};
            ck(csrc_fixture_matrix(fx, &m));
            Triplets t;
            t.n_rows = t.n_cols = m.n;
            const size_t cnt = static_cast<size_t>(m.n) + 2 * static_cast<size_t>(m.k);
            t.r.reserve(cnt);
            t.c.reserve(cnt);
            t.v.reserve(cnt);
            for (index_t i = 0; i < m.n; ++i) {
                t.add(i, i, m.ad[i]);
                for (index_t q = m.ia[i]; q < m.ia[i + 1]; ++q) {
                    t.add(i, m.ja[q], m.al[q]);
                    t.add(m.ja[q], i, m.au ? m.au[q] : m.al[q]);
                }
            }
            csrc_fixture_free(fx);
            return build_csr(t);
        }
        Csr a = build_csr(triplets());
        if (a.n_rows == a.n_cols) {
            const Symmetry s = analyze_symmetry(a);
            if (!s.structural) {
                if (!symmetrize)
                    throw Error("matrix '" + name() + "' is structurally asymmetric (" +
                                std::to_string(s.missing_transposes) + " missing transposes, " +
                                std::to_string(s.missing_diagonal) +
                                " missing diagonals); pass --symmetrize to pad with zeros");
                a = symmetrize_pattern(a);
            }
        }
        return a;
    }
};

// ------------------------------------------------------------- reporting
std::vector<double> source_vector(count_t n) {  // bench_source_vector (bench.hpp:87-91)
    std::vector<double> x(static_cast<size_t>(n));
    for (count_t i = 0; i < n; ++i) x[i] = 1.0 + static_cast<double>(i % 7) / 7.0;
    return x;
}

double relative_error(const std::vector<double>& y, const std::vector<double>& ref) {  // bench.hpp:93-100
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < ref.size(); ++i) {
        num = std::max(num, std::abs(y[i] - ref[i]));
        den = std::max(den, std::abs(ref[i]));
    }
    return den == 0.0 ? num : num / den;
}

struct Report {  // BenchReport (bench.hpp:24-55), same fields in the same order
    std::string matrix;
    count_t n = 0, nnz_stored = 0, nnz_full = 0, nnz_per_row = 0, ws_kb = 0;
    std::string format, strategy, accum;
    int p = 1, reps = 0, runs = 0;
    double median_total_seconds = 0, mflops_effective = 0, mflops_true = 0, speedup_vs_seq_csrc = 0;
    double init_max = 0, compute_max = 0, accumulate_max = 0;
    int n_colors = 0;
};

const char* kFields[] = {"matrix", "n", "nnz_stored", "nnz_full", "nnz_per_row", "ws_kb", "format",
                         "strategy", "accum", "p", "reps", "runs", "median_total_seconds",
                         "mflops_effective", "mflops_true", "speedup_vs_seq_csrc", "init_max",
                         "compute_max", "accumulate_max", "n_colors"};

std::string csv_escape(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string o = "\"";
    for (char ch : s) {
        if (ch == '"') o += '"';
        o += ch;
    }
    return o + "\"";
}

std::string csv_header() {
    std::string h;
    for (const char* f : kFields) h += (h.empty() ? "" : ",") + std::string(f);
    return h;
}

std::string csv_row(const Report& r) {
    std::ostringstream os;
    os.precision(12);
    os << csv_escape(r.matrix) << ',' << r.n << ',' << r.nnz_stored << ',' << r.nnz_full << ',' << r.nnz_per_row
       << ',' << r.ws_kb << ',' << r.format << ',' << r.strategy << ',' << r.accum << ',' << r.p << ',' << r.reps
       << ',' << r.runs << ',' << r.median_total_seconds << ',' << r.mflops_effective << ',' << r.mflops_true << ','
       << r.speedup_vs_seq_csrc << ',' << r.init_max << ',' << r.compute_max << ',' << r.accumulate_max << ','
       << r.n_colors;
    return os.str();
}

std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char ch : s) {
        if (ch == '"' || ch == '\\') o += '\\';
        o += ch;
    }
    return o + "\"";
}

std::string json_num(double v) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
}

std::string report_json(const Report& r) {
    std::ostringstream os;
    os << "{\n"
       << "  \"matrix\": " << json_str(r.matrix) << ",\n  \"n\": " << r.n << ",\n  \"nnz_stored\": " << r.nnz_stored
       << ",\n  \"nnz_full\": " << r.nnz_full << ",\n  \"nnz_per_row\": " << r.nnz_per_row << ",\n  \"ws_kb\": "
       << r.ws_kb << ",\n  \"format\": " << json_str(r.format) << ",\n  \"strategy\": " << json_str(r.strategy)
       << ",\n  \"accum\": " << json_str(r.accum) << ",\n  \"p\": " << r.p << ",\n  \"reps\": " << r.reps
       << ",\n  \"runs\": " << r.runs << ",\n  \"median_total_seconds\": " << json_num(r.median_total_seconds)
       << ",\n  \"mflops_effective\": " << json_num(r.mflops_effective) << ",\n  \"mflops_true\": "
       << json_num(r.mflops_true) << ",\n  \"speedup_vs_seq_csrc\": " << json_num(r.speedup_vs_seq_csrc)
       << ",\n  \"init_max\": " << json_num(r.init_max) << ",\n  \"compute_max\": " << json_num(r.compute_max)
       << ",\n  \"accumulate_max\": " << json_num(r.accumulate_max) << ",\n  \"n_colors\": " << r.n_colors
       << "\n}\n";
    return os.str();
}

// ------------------------------------------------------------ strategies
int kind_of(const std::string& s) {
    if (s == "seq") return CSRC_KIND_SEQUENTIAL;
    if (s == "buffers") return CSRC_KIND_LOCAL_BUFFERS;
    if (s == "colorful") return CSRC_KIND_COLORFUL;
    if (s == "gather") return CSRC_KIND_GATHER;
    if (s == "windowed") return CSRC_KIND_WINDOWED;
    if (s == "atomic") return CSRC_KIND_ATOMIC;
    throw UsageError("--strategy: unknown strategy '" + s + "'");
}

int accum_of(const std::string& s) {
    if (s == "all-in-one") return CSRC_ACCUM_ALL_IN_ONE;
    if (s == "per-buffer") return CSRC_ACCUM_PER_BUFFER;
    if (s == "effective") return CSRC_ACCUM_EFFECTIVE;
    if (s == "interval") return CSRC_ACCUM_INTERVAL;
    throw UsageError("--accum: unknown accumulation method '" + s + "'");
}

const char* accum_name(int a) {
    static const char* n[] = {"all-in-one", "per-buffer", "effective", "interval"};
    return n[a];
}

struct Plan {
    csrc_gpu_plan_t h = nullptr;
    Plan(const Csrc& a, const csrc_gpu_strategy& s, const std::vector<int32_t>* color = nullptr, int nc = 0) {
        csrc_host_matrix m = a.view();
        if (color)
            ck(csrc_gpu_plan_create_colored(&m, &s, color->data(), nc, &h));
        else
            ck(csrc_gpu_plan_create(&m, &s, &h));
    }
    Plan(const Csr& a, const csrc_gpu_strategy& s) {  // spmv_csr plan
        ck(csrc_gpu_plan_create_csr(a.n_rows, a.n_cols, a.rp.data(), a.ci.data(), a.va.data(), &s, &h));
    }
    Plan(Plan&& o) noexcept : h(o.h) { o.h = nullptr; }
    ~Plan() { csrc_gpu_plan_destroy(h); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    csrc_gpu_plan_info info() const {
        csrc_gpu_plan_info i{};
        ck(csrc_gpu_plan_get_info(h, &i));
        return i;
    }
    std::vector<double> apply(const std::vector<double>& x) const {
        std::vector<double> y(x.size());
        ck(csrc_gpu_spmv(h, x.data(), static_cast<int64_t>(x.size()), y.data()));
        return y;
    }
};

csrc_gpu_strategy strategy(int kind, int accum, int p, int mode, int dtype) {
    csrc_gpu_strategy s{};
    s.kind = kind;
    s.accum = accum;
    s.p = p;
    s.dtype = dtype;
    s.conflict_mode = mode;
    s.color_order = CSRC_ORDER_NATURAL;
    s.device = g_device;
    s.bands = 0;
    return s;
}

// reps products per run, `runs` runs: total seconds per run + per-run phase
// sums. Device-resident vectors (CUDA events on the plan's stream) unless
// host_vectors, which times the drop-in host call with its copies.
struct RunTimes {
    std::vector<double> total;
    std::vector<double> init, compute, accum;
};

RunTimes time_plan(const Plan& P, const std::vector<double>& x, int reps, int runs, bool host_vectors, int dtype) {
    RunTimes rt;
    if (host_vectors) {
        std::vector<double> y(x.size());
        ck(csrc_gpu_set_timing(P.h, 1));
        for (int r = 0; r < runs; ++r) {
            double tot = 0, pi = 0, pc = 0, pa = 0;
            for (int i = 0; i < reps; ++i) {
                const auto t0 = std::chrono::steady_clock::now();
                ck(csrc_gpu_spmv(P.h, x.data(), static_cast<int64_t>(x.size()), y.data()));
                tot += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                csrc_gpu_timings t{};
                ck(csrc_gpu_last_timings(P.h, &t));
                pi += t.init_ms / 1e3;
                pc += t.compute_ms / 1e3;
                pa += t.accumulate_ms / 1e3;
            }
            rt.total.push_back(tot);
            rt.init.push_back(pi);
            rt.compute.push_back(pc);
            rt.accum.push_back(pa);
        }
        ck(csrc_gpu_set_timing(P.h, 0));
        return rt;
    }
    // device-resident: x uploaded once into the plan's vectors, CUDA events per product
    (void)dtype;
    std::vector<double> tot(static_cast<size_t>(reps)), ker(static_cast<size_t>(reps));
    for (int r = 0; r < runs; ++r) {
        ck(csrc_gpu_time_products_host(P.h, x.data(), static_cast<int64_t>(x.size()), reps, 0, tot.data(),
                                       ker.data()));
        double s = 0, k = 0;
        for (int i = 0; i < reps; ++i) {
            s += tot[i] / 1e3;
            k += ker[i] / 1e3;
        }
        rt.total.push_back(s);
        rt.init.push_back(0.0);
        rt.compute.push_back(k);
        rt.accum.push_back(std::max(0.0, s - k));
    }
    return rt;
}

size_t median_index(const std::vector<double>& t) {
    std::vector<size_t> o(t.size());
    for (size_t i = 0; i < o.size(); ++i) o[i] = i;
    std::sort(o.begin(), o.end(), [&](size_t a, size_t b) { return t[a] < t[b]; });
    return o[o.size() / 2];
}

// ---------------------------------------------------------------- args
struct Args {
    std::string cmd;
    Source src;
    std::string format = "csrc", strategy = "seq", accum = "effective", mode = "neighborhood", dtype = "f64";
    int threads = 1, reps = 1000, runs = 3;
    std::string threads_list = "1,2,4", only;
    std::vector<std::string> out;
    bool corrupt = false, host_vectors = false;
};

const char* kUsage =
    "usage: csrc_bench {run,verify,info} (--matrix PATH | --gen KIND:k=v,... | --config cN) [--symmetrize]\n"
    "  run    [--format csr|csrc] [--strategy seq|buffers|colorful|gather|windowed|atomic]\n"
    "         [--accum all-in-one|per-buffer|effective|interval] [--threads P] [--reps R] [--runs N]\n"
    "         [--conflict-mode neighborhood|exact] [--dtype f64|f32] [--host-vectors] [--device D]\n"
    "         [--out csv|json PATH]\n"
    "  verify [--threads 1,2,4] [--strategy seq|csr|buffers|colorful|gather|windowed|atomic]\n"
    "         [--conflict-mode neighborhood|exact]\n"
    "  info\n";

int to_pos_int(const std::string& flag, const std::string& v) {
    size_t used = 0;
    long x = 0;
    try {
        x = std::stol(v, &used);
    } catch (...) {
        throw UsageError(flag + ": value '" + v + "' is not a number");
    }
    if (used != v.size() || x < 1) throw UsageError(flag + ": value " + v + " not in range [1, inf)");
    return static_cast<int>(x);
}

Args parse(int argc, char** argv) {
    if (argc < 2) throw UsageError("a subcommand is required");
    Args a;
    a.cmd = argv[1];
    if (a.cmd != "run" && a.cmd != "verify" && a.cmd != "info")
        throw UsageError("unknown subcommand '" + a.cmd + "'");
    auto member = [](const std::string& flag, const std::string& v, std::initializer_list<const char*> ok) {
        for (const char* o : ok)
            if (v == o) return;
        throw UsageError(flag + ": '" + v + "' not in the allowed set");
    };
    for (int i = 2; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw UsageError(f + " requires a value");
            return argv[++i];
        };
        if (f == "--matrix") a.src.path = val();
        else if (f == "--gen") a.src.gen = val();
        else if (f == "--config") a.src.config = val();
        else if (f == "--symmetrize") a.src.symmetrize = true;
        else if (f == "--device") g_device = std::stoi(val());
        else if (a.cmd == "run" && f == "--format") member(f, a.format = val(), {"csr", "csrc"});
        else if (a.cmd == "run" && f == "--strategy")
            member(f, a.strategy = val(), {"seq", "buffers", "colorful", "gather", "windowed", "atomic"});
        else if (a.cmd == "run" && f == "--accum")
            member(f, a.accum = val(), {"all-in-one", "per-buffer", "effective", "interval"});
        else if (a.cmd == "run" && f == "--threads") a.threads = to_pos_int(f, val());
        else if (a.cmd == "run" && f == "--reps") a.reps = to_pos_int(f, val());
        else if (a.cmd == "run" && f == "--runs") a.runs = to_pos_int(f, val());
        else if (a.cmd == "run" && f == "--dtype") member(f, a.dtype = val(), {"f64", "f32"});
        else if (a.cmd == "run" && f == "--host-vectors") a.host_vectors = true;
        else if (a.cmd == "run" && f == "--out") {
            a.out.push_back(val());
            a.out.push_back(val());
            member("--out", a.out[0], {"csv", "json"});
        } else if (a.cmd != "info" && f == "--conflict-mode") member(f, a.mode = val(), {"neighborhood", "exact"});
        else if (a.cmd == "verify" && f == "--threads") a.threads_list = val();
        else if (a.cmd == "verify" && f == "--strategy")
            member(f, a.only = val(), {"seq", "csr", "buffers", "colorful", "gather", "windowed", "atomic"});
        else if (a.cmd == "verify" && f == "--corrupt-coloring") a.corrupt = true;
        else throw UsageError("unknown option '" + f + "' for " + a.cmd);
    }
    const int sources = !a.src.path.empty() + !a.src.gen.empty() + !a.src.config.empty();
    if (sources > 1) throw UsageError("--matrix, --gen and --config exclude each other");
    return a;
}

// ------------------------------------------------------------ subcommands
int do_run(const Args& A) {
    const Csr full = A.src.csr();
    const Csrc m = csr_to_csrc(full);
    const int dtype = A.dtype == "f32" ? CSRC_DTYPE_F32 : CSRC_DTYPE_F64;
    const int mode = A.mode == "exact" ? CSRC_CONFLICT_EXACT : CSRC_CONFLICT_NEIGHBORHOOD;
    Report r;
    r.matrix = A.src.name();
    r.n = m.n;
    r.nnz_stored = m.value_symmetric ? m.nnz_stored() : m.nnz_full();  // matrix_info (bench.hpp:113-122)
    r.nnz_full = m.nnz_full();
    r.nnz_per_row = m.n ? r.nnz_stored / m.n : 0;
    r.ws_kb = csrc_model_bytes(m.n, r.nnz_stored, m.value_symmetric ? 1 : 0, CSRC_DTYPE_F64) / 1024;
    r.p = A.threads;
    r.reps = A.reps;
    r.runs = A.runs;
    int kind = kind_of(A.strategy);
    const int accum = accum_of(A.accum);
    r.strategy = A.strategy;
    r.accum = kind == CSRC_KIND_LOCAL_BUFFERS ? accum_name(accum) : "-";
    // csr format: a CSR plan over the full matrix (spmv_csr, kernels.hpp:7-22)
    const bool csr = A.format == "csr";
    r.format = csr ? "csr" : (m.value_symmetric ? "csrc_sym" : "csrc");
    if (csr) kind = CSRC_KIND_GATHER;
    const std::vector<double> x = source_vector(m.n);

    Plan seq(m, strategy(CSRC_KIND_SEQUENTIAL, CSRC_ACCUM_EFFECTIVE, 1, mode, dtype));
    const std::vector<double> y_ref = seq.apply(x);
    const RunTimes base = time_plan(seq, x, A.reps, A.runs, A.host_vectors, dtype);
    const double base_med = base.total[median_index(base.total)];

    const bool sequential = kind == CSRC_KIND_SEQUENTIAL;
    Plan exec = csr ? Plan(full, strategy(CSRC_KIND_GATHER, accum, 1, mode, dtype))
                    : Plan(m, strategy(kind, accum, sequential ? 1 : A.threads, mode, dtype));
    if (kind == CSRC_KIND_COLORFUL) r.n_colors = exec.info().n_colors;
    if (!sequential || csr) {  // verify before timing (bench.hpp:221-228)
        const double err = relative_error(exec.apply(x), y_ref);
        const double bound = dtype == CSRC_DTYPE_F32 ? 1e-5 : 1e-12;
        if (err > bound)
            throw Error("benchmark verification failed: relative error " + std::to_string(err) +
                        " vs sequential CSRC");
    }
    const RunTimes rt = sequential && !csr ? base : time_plan(exec, x, A.reps, A.runs, A.host_vectors, dtype);
    const size_t med = median_index(rt.total);
    r.median_total_seconds = rt.total[med];
    r.init_max = rt.init[med];
    r.compute_max = rt.compute[med];
    r.accumulate_max = rt.accum[med];
    const double per = r.median_total_seconds / A.reps;
    r.mflops_effective = 2.0 * static_cast<double>(r.nnz_full) / per / 1e6;
    const double flops_true = csr ? 2.0 * r.nnz_full : static_cast<double>(csrc_model_flops(m.n, r.nnz_full));
    r.mflops_true = flops_true / per / 1e6;
    r.speedup_vs_seq_csrc = base_med / r.median_total_seconds;
    std::cout << csv_header() << "\n" << csv_row(r) << "\n";
    if (!A.out.empty()) {
        std::ofstream out(A.out[1]);
        if (!out) throw Error("cannot write '" + A.out[1] + "'");
        if (A.out[0] == "json") out << report_json(r);
        else out << csv_header() << "\n" << csv_row(r) << "\n";
    }
    return 0;
}

std::vector<int> int_list(const std::string& s) {
    std::vector<int> v;
    std::istringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) v.push_back(std::stoi(tok));
    return v;
}

int do_verify(const Args& A) {
    const Csr full = A.src.csr();
    const Csrc m = csr_to_csrc(full);
    const std::vector<double> x = source_vector(m.n);
    const int mode = A.mode == "exact" ? CSRC_CONFLICT_EXACT : CSRC_CONFLICT_NEIGHBORHOOD;
    // the harness's checker (bench_main.cpp:179-198): dense two-loop product for
    // small orders, sequential CSR otherwise -- on the host, compared against
    // every GPU result
    std::vector<double> ref(static_cast<size_t>(m.n), 0.0);
    if (m.n <= 2000) {
        std::vector<double> dense(static_cast<size_t>(m.n) * m.n, 0.0);
        for (index_t i = 0; i < full.n_rows; ++i)
            for (index_t k = full.rp[i]; k < full.rp[i + 1]; ++k)
                dense[static_cast<size_t>(i) * m.n + full.ci[k]] = full.va[k];
        for (index_t i = 0; i < m.n; ++i) {
            double s = 0.0;
            for (index_t j = 0; j < m.n; ++j) s += dense[static_cast<size_t>(i) * m.n + j] * x[j];
            ref[i] = s;
        }
    } else {
        for (index_t i = 0; i < full.n_rows; ++i) {
            double s = 0.0;
            for (index_t k = full.rp[i]; k < full.rp[i + 1]; ++k) s += full.va[k] * x[full.ci[k]];
            ref[i] = s;
        }
    }
    bool all = true;
    auto check = [&](const std::string& label, const std::vector<double>& y, bool ok, const std::string& note) {
        const double err = relative_error(y, ref);
        const bool pass = err <= 1e-12 && ok;
        all = all && pass;
        std::cout << (pass ? "pass" : "FAIL") << "  " << label << "  max_rel_err=" << err;
        if (!note.empty()) std::cout << "  " << note;
        std::cout << "\n";
    };
    auto want = [&](const std::string& s) { return A.only.empty() || A.only == s; };
    auto run = [&](int kind, int accum, int p) {
        Plan P(m, strategy(kind, accum, p, mode, CSRC_DTYPE_F64));
        return P.apply(x);
    };
    if (want("seq")) check("seq csrc p=1", run(CSRC_KIND_SEQUENTIAL, CSRC_ACCUM_EFFECTIVE, 1), true, "");
    if (want("csr")) {
        Plan pc(full, strategy(CSRC_KIND_GATHER, CSRC_ACCUM_EFFECTIVE, 1, mode, CSRC_DTYPE_F64));
        check("seq csr", pc.apply(x), true, "");
    }
    for (const char* g : {"gather", "windowed", "atomic"})
        if (!A.only.empty() && A.only == g) check(std::string(g) + " p=1", run(kind_of(g), CSRC_ACCUM_EFFECTIVE, 1), true, "");
    for (int p : int_list(A.threads_list)) {
        if (p > m.n) continue;
        if (want("buffers"))
            for (int acc = CSRC_ACCUM_ALL_IN_ONE; acc <= CSRC_ACCUM_INTERVAL; ++acc)
                check(std::string("buffers/") + accum_name(acc) + " p=" + std::to_string(p),
                      run(CSRC_KIND_LOCAL_BUFFERS, acc, p), true, "");
        if (want("colorful")) {
            csrc_host_matrix hm = m.view();
            std::vector<int32_t> color(static_cast<size_t>(std::max(m.n, 1)));
            int32_t nc = 0;
            ck(csrc_color_rows(&hm, mode, CSRC_ORDER_NATURAL, color.data(), &nc));
            if (A.corrupt && nc >= 2) {  // test hook: merge the first two classes (bench_main.cpp:232-243)
                for (auto& c : color) c = c <= 1 ? 0 : c - 1;
                --nc;
            }
            int32_t valid = 0, ra = -1, rb = -1, pos = -1;
            ck(csrc_validate_coloring(&hm, color.data(), nc, &valid, &ra, &rb, &pos));
            std::string note;
            if (!valid)
                note = "coloring violation: rows " + std::to_string(ra) + " and " + std::to_string(rb) + " share y[" +
                       std::to_string(pos) + "]";
            const std::string label = "colorful p=" + std::to_string(p);
            if (!valid) {
                // the GPU plan refuses an invalid coloring; report the violation
                check(label, std::vector<double>(static_cast<size_t>(m.n), NAN), false, note);
                continue;
            }
            Plan P(m, strategy(CSRC_KIND_COLORFUL, CSRC_ACCUM_EFFECTIVE, std::max(p, 1), mode, CSRC_DTYPE_F64), &color,
                   nc);
            check(label, P.apply(x), true, note);
        }
    }
    std::cout << (all ? "VERIFY PASS" : "VERIFY FAIL") << "\n";
    return all ? 0 : 1;
}

int do_info(const Args& A) {
    const Csrc m = csr_to_csrc(A.src.csr());
    const count_t nnz = m.value_symmetric ? m.nnz_stored() : m.nnz_full();  // matrix_info (bench.hpp:113-122)
    const count_t ws = csrc_model_bytes(m.n, nnz, m.value_symmetric ? 1 : 0, CSRC_DTYPE_F64) / 1024;
    std::cout << A.src.name() << " " << (m.value_symmetric ? "yes" : "no") << " " << m.n << " " << nnz << " "
              << (m.n ? nnz / m.n : 0) << " " << ws << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args A;
    try {
        A = parse(argc, argv);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return 2;
    }
    if (A.src.path.empty() && A.src.gen.empty() && A.src.config.empty()) {
        std::cerr << "error: one of --matrix or --gen is required\n";
        return 2;
    }
    try {
        if (A.cmd == "run") return do_run(A);
        if (A.cmd == "verify") return do_verify(A);
        return do_info(A);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
