// Deterministic synthetic FE matrices for the BASELINE.json configs,
// assembled directly in CSRC form (no triplet sort), multithreaded.
// Test / bench INPUT definitions: compiled into the
// product library (csrc_bench --config, P.config_matrix) and, standalone, into
// oracle/_build/libcsrc_fixtures.so for the reference arm.
//
// The reference can only generate dense / band / random patterns
// (generate.hpp:12-65); these meshes are the fixture definitions of
// DESIGN.md "Fixtures". Direct assembly produces exactly what the reference
// pipeline build_csr (csr.hpp:55-92) -> csr_to_csrc (csrc_matrix.hpp:44-91)
// produces from the same entries: rows ascending, ja strictly increasing
// within a row, al = a_ij, au = a_ji (tests/test_fixtures.py pins this
// against the reference itself).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <thread>

#ifdef CSRC_FIXTURES_STANDALONE
// Standalone build (oracle/Makefile -> oracle/_build/libcsrc_fixtures.so): the
// reference arm of bench.py and the oracle-side tests generate their inputs
// without mapping the product library. Same source, same matrices.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/csrc_gpu.h"

namespace csrcgpu {
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
thread_local std::string g_fixture_error;
template <class F>
int guarded(const char*, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_fixture_error = e.what();
        return 1;
    } catch (...) {
        g_fixture_error = "unknown error";
        return 1;
    }
}
}  // namespace csrcgpu
extern "C" const char* csrc_fixture_last_error(void) { return csrcgpu::g_fixture_error.c_str(); }
#else
#include "../paper_1003_0952_b200/csrc/internal.hpp"
#endif

namespace csrcgpu {
namespace {

// ---- counter-based RNG ------------------------------
inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull);
    h = mix64(h ^ (a * 0xD6E8FEB86659FD93ull));
    h = mix64(h ^ (b * 0xCA5A826395121157ull));
    return h;
}
inline double u01(uint64_t seed, uint64_t a, uint64_t b) {
    return static_cast<double>(hash3(seed, a, b) >> 11) * 0x1.0p-53;
}
constexpr uint64_t kXStream = 1ull << 32;     // b for x_i
constexpr uint64_t kPermStream = 1ull << 33;  // b for the Fisher-Yates draws

template <class F>
void parallel_for(int64_t n, int threads, F&& f) {
    if (threads <= 1 || n < 4096) {
        f(int64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        int64_t b = n * t / threads, e = n * (t + 1) / threads;
        pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}

// 27-point (or 9-point in 2D) node neighbourhood in natural order.
struct Grid {
    int64_t nx, ny, nz;
    int64_t nodes() const { return nx * ny * nz; }
    // neighbours of u (including u itself), ascending natural id
    int neighbours(int64_t u, int64_t* out) const {
        int64_t x = u % nx, y = (u / nx) % ny, z = u / (nx * ny);
        int c = 0;
        for (int dz = -1; dz <= 1; ++dz) {
            int64_t zz = z + dz;
            if (zz < 0 || zz >= nz) continue;
            for (int dy = -1; dy <= 1; ++dy) {
                int64_t yy = y + dy;
                if (yy < 0 || yy >= ny) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t xx = x + dx;
                    if (xx < 0 || xx >= nx) continue;
                    out[c++] = (zz * ny + yy) * nx + xx;
                }
            }
        }
        return c;
    }
};

}  // namespace
}  // namespace csrcgpu

struct csrc_fixture_s {
    int32_t n = 0;
    std::vector<double> ad, al, au, x;
    std::vector<int32_t> ia, ja, order;
};

namespace csrcgpu {
namespace {

// Reverse Cuthill-McKee over a node graph given as CSR (adjacency excludes
// self), deterministic: George-Liu pseudo-peripheral start from the
// (degree, label)-minimal vertex; neighbours visited by (degree, label).
std::vector<int64_t> rcm_order(int64_t n, const std::vector<int64_t>& ptr,
                               const std::vector<int32_t>& adj) {
    std::vector<int32_t> deg(n);
    for (int64_t v = 0; v < n; ++v) deg[v] = static_cast<int32_t>(ptr[v + 1] - ptr[v]);
    std::vector<int64_t> cm;
    cm.reserve(n);
    std::vector<char> placed(n, 0);
    std::vector<int32_t> level(n, -1);
    auto less_dl = [&](int64_t a, int64_t b) {
        return deg[a] != deg[b] ? deg[a] < deg[b] : a < b;
    };
    // BFS returning (eccentricity, last level vertices) within unplaced graph
    std::vector<int64_t> queue;
    queue.reserve(n);
    auto bfs = [&](int64_t r, std::vector<int64_t>& last) {
        queue.clear();
        queue.push_back(r);
        std::vector<int64_t> touched;
        level[r] = 0;
        size_t head = 0;
        int ecc = 0;
        while (head < queue.size()) {
            int64_t v = queue[head++];
            ecc = std::max(ecc, level[v]);
            for (int64_t q = ptr[v]; q < ptr[v + 1]; ++q) {
                int32_t w = adj[q];
                if (placed[w] || level[w] >= 0) continue;
                level[w] = level[v] + 1;
                queue.push_back(w);
            }
        }
        last.clear();
        for (int64_t v : queue)
            if (level[v] == ecc) last.push_back(v);
        for (int64_t v : queue) level[v] = -1;
        return ecc;
    };
    int64_t scan = 0;
    std::vector<int64_t> last;
    std::vector<int64_t> nb;
    while (static_cast<int64_t>(cm.size()) < n) {
        // minimal (degree, label) unplaced vertex
        int64_t r = -1;
        for (int64_t v = scan; v < n; ++v)
            if (!placed[v] && (r < 0 || less_dl(v, r))) r = v;
        while (scan < n && placed[scan]) ++scan;
        // pseudo-peripheral node (George-Liu)
        int ecc = bfs(r, last);
        for (;;) {
            int64_t c = last[0];
            for (int64_t v : last)
                if (less_dl(v, c)) c = v;
            int ecc_c = bfs(c, last);
            if (ecc_c <= ecc) break;
            r = c;  // `last` now holds c's deepest level
            ecc = ecc_c;
        }
        // Cuthill-McKee from r
        size_t head = cm.size();
        cm.push_back(r);
        placed[r] = 1;
        while (head < cm.size()) {
            int64_t v = cm[head++];
            nb.clear();
            for (int64_t q = ptr[v]; q < ptr[v + 1]; ++q)
                if (!placed[adj[q]]) nb.push_back(adj[q]);
            std::sort(nb.begin(), nb.end(), less_dl);
            for (int64_t w : nb) {
                placed[w] = 1;
                cm.push_back(w);
            }
        }
    }
    std::reverse(cm.begin(), cm.end());
    return cm;  // cm[new] = old label
}

void generate(const csrc_fixture_spec& s, csrc_fixture_s& fx) {
    const int threads = s.threads > 0 ? s.threads
                                      : std::max(1u, std::thread::hardware_concurrency());
    if (s.nx < 1 || s.ny < 1 || s.nz < 1) throw Error("fixture: mesh dimensions must be >= 1");
    Grid g{s.nx, s.ny, s.nz};
    if (s.mesh == CSRC_MESH_GRID2D_Q1 && s.nz != 1) throw Error("fixture: 2D mesh needs nz = 1");
    const int dof = s.mesh == CSRC_MESH_ELASTICITY ? 3 : 1;
    const int64_t nodes = g.nodes();
    const int64_t n64 = nodes * dof;
    if (n64 >= (1ll << 31)) throw Error("fixture: n exceeds int32 index range");
    const int32_t n = static_cast<int32_t>(n64);
    fx.n = n;
    const uint64_t seed = s.seed;

    // node ordering: final index f(u) of natural node u, and its inverse
    std::vector<int64_t> f, finv;
    if (s.mesh == CSRC_MESH_GRID3D_27_RCM) {
        // permutation p from seed (Fisher-Yates, descending i)
        std::vector<int64_t> p(nodes);
        std::iota(p.begin(), p.end(), int64_t{0});
        for (int64_t i = nodes - 1; i >= 1; --i) {
            int64_t j = static_cast<int64_t>(u01(seed, static_cast<uint64_t>(i), kPermStream) *
                                             static_cast<double>(i + 1));
            if (j > i) j = i;
            std::swap(p[i], p[j]);
        }
        // graph in permuted labels: label p[u] for natural u
        std::vector<int64_t> pinv(nodes);
        for (int64_t u = 0; u < nodes; ++u) pinv[p[u]] = u;
        std::vector<int64_t> ptr(nodes + 1, 0);
        {
            int64_t nb[27];
            for (int64_t l = 0; l < nodes; ++l) ptr[l + 1] = g.neighbours(pinv[l], nb) - 1;
        }
        for (int64_t l = 0; l < nodes; ++l) ptr[l + 1] += ptr[l];
        std::vector<int32_t> adj(ptr[nodes]);
        parallel_for(nodes, threads, [&](int64_t b, int64_t e) {
            int64_t nb[27];
            for (int64_t l = b; l < e; ++l) {
                int64_t u = pinv[l];
                int c = g.neighbours(u, nb);
                int64_t q = ptr[l];
                for (int i = 0; i < c; ++i)
                    if (nb[i] != u) adj[q++] = static_cast<int32_t>(p[nb[i]]);
                std::sort(adj.begin() + ptr[l], adj.begin() + ptr[l + 1]);
            }
        });
        std::vector<int64_t> cm = rcm_order(nodes, ptr, adj);  // cm[new] = label
        f.resize(nodes);
        finv.resize(nodes);
        for (int64_t nw = 0; nw < nodes; ++nw) {
            int64_t u = pinv[cm[nw]];
            finv[nw] = u;
            f[u] = nw;
        }
    }
    const bool permuted = !f.empty();
    fx.order.resize(n);
    for (int64_t i = 0; i < n64; ++i) fx.order[i] = static_cast<int32_t>(permuted ? f[i] : i);

    // row lengths: row i (final) -> lower columns j < i
    fx.ia.assign(static_cast<size_t>(n) + 1, 0);
    auto row_cols = [&](int64_t i, int64_t* nodebuf, std::vector<int64_t>& cols) {
        // final dof i -> natural node u, component a
        int64_t node_final = i / dof, a = i % dof;
        int64_t u = permuted ? finv[node_final] : node_final;
        int c = g.neighbours(u, nodebuf);
        cols.clear();
        for (int q = 0; q < c; ++q) {
            int64_t vf = permuted ? f[nodebuf[q]] : nodebuf[q];
            for (int b = 0; b < dof; ++b) {
                int64_t j = vf * dof + b;
                if (j < i) cols.push_back(j);
            }
        }
        if (permuted) std::sort(cols.begin(), cols.end());
        (void)a;
    };
    parallel_for(n64, threads, [&](int64_t b, int64_t e) {
        int64_t nodebuf[27];
        std::vector<int64_t> cols;
        for (int64_t i = b; i < e; ++i) {
            row_cols(i, nodebuf, cols);
            fx.ia[i + 1] = static_cast<int32_t>(cols.size());
        }
    });
    int64_t total = 0;
    for (int64_t i = 0; i < n64; ++i) {
        total += fx.ia[i + 1];
        if (total >= (1ll << 31)) throw Error("fixture: nnz exceeds int32 index range");
        fx.ia[i + 1] = static_cast<int32_t>(total);
    }
    fx.ja.resize(total);
    fx.al.resize(total);
    fx.au.resize(total);
    fx.ad.resize(n);
    fx.x.resize(n);
    // natural dof id of final dof i
    auto natural = [&](int64_t i) -> int64_t {
        if (!permuted) return i;
        return finv[i / dof] * dof + i % dof;
    };
    parallel_for(n64, threads, [&](int64_t b, int64_t e) {
        int64_t nodebuf[27];
        std::vector<int64_t> cols;
        for (int64_t i = b; i < e; ++i) {
            const int64_t ni = natural(i);
            fx.ad[i] = s.diag_base + u01(seed, ni, ni);
            fx.x[i] = 2.0 * u01(seed, static_cast<uint64_t>(i), kXStream) - 1.0;
            row_cols(i, nodebuf, cols);
            int64_t t = fx.ia[i];
            for (int64_t j : cols) {
                const int64_t nj = natural(j);
                fx.ja[t] = static_cast<int32_t>(j);
                fx.al[t] = 2.0 * u01(seed, ni, nj) - 1.0;  // a_ij
                fx.au[t] = 2.0 * u01(seed, nj, ni) - 1.0;  // a_ji
                ++t;
            }
        }
    });
}

}  // namespace
}  // namespace csrcgpu

using namespace csrcgpu;

extern "C" {

int csrc_fixture_generate(const csrc_fixture_spec* spec, csrc_fixture_t* out) {
    return guarded(__func__, [&] {
        if (!spec || !out) throw Error("csrc_fixture_generate: null argument");
        *out = nullptr;
        auto fx = std::make_unique<csrc_fixture_s>();
        generate(*spec, *fx);
        *out = fx.release();
    });
}

int csrc_fixture_matrix(csrc_fixture_t fx, csrc_host_matrix* m) {
    return guarded(__func__, [&] {
        if (!fx || !m) throw Error("csrc_fixture_matrix: null argument");
        m->n = fx->n;
        m->k = static_cast<int64_t>(fx->ja.size());
        m->ad = fx->ad.data();
        m->ia = fx->ia.data();
        m->ja = fx->ja.data();
        m->al = fx->al.data();
        m->au = fx->au.data();
        m->value_symmetric = 0;
    });
}

const double* csrc_fixture_x(csrc_fixture_t fx) { return fx ? fx->x.data() : nullptr; }
const int32_t* csrc_fixture_order(csrc_fixture_t fx) { return fx ? fx->order.data() : nullptr; }
void csrc_fixture_free(csrc_fixture_t fx) { delete fx; }
double csrc_fixture_u01(uint64_t seed, uint64_t a, uint64_t b) { return u01(seed, a, b); }

}  // extern "C"
