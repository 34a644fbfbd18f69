// Runtime specialisation of pass kernels (see qsv_jit.h).
#include "qsv_jit.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cctype>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <sys/stat.h>
#include <unistd.h>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <vector>

namespace qsv {

// File-scope declarations gathered while a kernel body is generated (per-thread
// factor tables, StageGen::materialize); jit_source inserts them before the
// kernel.  One generation at a time per thread.
thread_local std::ostringstream *g_decls = nullptr;
thread_local int g_decl_id = 0;


namespace {

// ---------------------------------------------------------------------------
// dynamically loaded NVRTC + driver API (the library itself must load on
// machines without a GPU driver, so nothing here is linked at build time)
// ---------------------------------------------------------------------------

struct Nvrtc {
    bool ok = false;
    std::string why;
    nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                                 const char *const *) = nullptr;
    nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
    nvrtcResult (*Version)(int *, int *) = nullptr;
};

struct Driver {
    bool ok = false;
    std::string why;
    CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **) = nullptr;
    CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
    CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int *, CUfunction, int, size_t) = nullptr;
    CUresult (*LaunchCooperativeKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                        unsigned, CUstream, void **) = nullptr;
};

template <typename F>
bool sym(void *h, const char *name, F &fn) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    return fn != nullptr;
}

Nvrtc &nvrtc() {
    static Nvrtc api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = nullptr;
        for (const char *p : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
            if ((h = dlopen(p, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            api.why = "libnvrtc not found";
            return;
        }
        api.ok = sym(h, "nvrtcCreateProgram", api.CreateProgram) && sym(h, "nvrtcCompileProgram", api.CompileProgram) &&
                 sym(h, "nvrtcGetProgramLogSize", api.GetProgramLogSize) &&
                 sym(h, "nvrtcGetProgramLog", api.GetProgramLog) && sym(h, "nvrtcGetCUBINSize", api.GetCUBINSize) &&
                 sym(h, "nvrtcGetCUBIN", api.GetCUBIN) && sym(h, "nvrtcDestroyProgram", api.DestroyProgram);
        if (!api.ok) api.why = "libnvrtc lacks a required symbol";
        sym(h, "nvrtcVersion", api.Version);
    });
    return api;
}

Driver &driver() {
    static Driver api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libcuda.so.1 not found";
            return;
        }
        api.ok = sym(h, "cuModuleLoadData", api.ModuleLoadData) && sym(h, "cuModuleGetFunction", api.ModuleGetFunction) &&
                 sym(h, "cuFuncSetAttribute", api.FuncSetAttribute) && sym(h, "cuLaunchKernel", api.LaunchKernel) &&
                 sym(h, "cuGetErrorString", api.GetErrorString) &&
                 sym(h, "cuOccupancyMaxActiveBlocksPerMultiprocessor", api.OccupancyMaxActiveBlocksPerMultiprocessor) &&
                 sym(h, "cuLaunchCooperativeKernel", api.LaunchCooperativeKernel);
        if (!api.ok) api.why = "libcuda lacks a required symbol";
    });
    return api;
}

// ---------------------------------------------------------------------------
// source generation
// ---------------------------------------------------------------------------

const char *kPrelude = R"(
typedef unsigned long long u64;
__device__ __forceinline__ double2 ldcs2(const double2 *p) {
    double2 r;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcs2(double2 *p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 ldwb2(const double2 *p) {
    double2 r;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stwb2(double2 *p, double2 v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// one 128-byte line into L2 (a plain per-thread prefetch: the bulk form needs a
// uniform address, so per-lane bulk prefetches were serialised into ~10-instruction
// loops - 21-30 % of all issued instructions of the C2 passes, ncu r02)
__device__ __forceinline__ void prefetch_line(const void *g) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(g));
}
__device__ __forceinline__ void prefetch_l2(const void *g, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(unsigned saddr, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try(bar, parity))
        if (++spins > (1u << 26)) __trap();  // never hang the GPU: fail loudly
}
// TMA bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// sign flip of a double by an XOR mask on its sign bit: an integer op, keeps
// the FP64 pipe free (a negation would otherwise issue a DADD)
__device__ __forceinline__ double xsg(double x, u64 m) {
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)m);
}
)";

std::string lit(double x) {
    if (x == 0.0) return "0.0";
    if (x == 1.0) return "1.0";
    if (x == -1.0) return "-1.0";
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%a", x);
    return std::string("(") + buf + ")";
}

inline uint64_t deposit(uint64_t v, const std::vector<int> &pos) {
    uint64_t out = 0;
    for (size_t j = 0; j < pos.size(); ++j)
        if ((v >> j) & 1) out |= 1ull << pos[j];
    return out;
}

// expression depositing bits [0, pos.size()) of `src` at positions pos[] (ascending)
std::string deposit_expr(const std::string &src, const std::vector<int> &pos, bool wide) {
    std::ostringstream e;
    const char *one = wide ? "1ull" : "1u";
    const std::string s = wide ? "((u64)" + src + ")" : src;
    bool first = true;
    size_t j = 0;
    while (j < pos.size()) {
        size_t k = j;
        while (k + 1 < pos.size() && pos[k + 1] == pos[k] + 1) ++k;
        const int len = (int)(k - j + 1);
        if (!first) e << " | ";
        first = false;
        // bits [j, k] of src land at positions [pos[j], pos[k]]
        e << "(((" << s << " >> " << j << ") & ((" << one << " << " << len << ") - " << one << "))";
        if (pos[j] > 0) e << " << " << pos[j];
        e << ")";
        j = k + 1;
    }
    if (first) return wide ? "0ull" : "0u";
    return e.str();
}

inline int popc64(uint64_t x) { return __builtin_popcountll(x); }

}  // namespace

// Tile double buffering (cp.async prefetch of the next tile into a second smem
// buffer) was measured and dropped: the first stage now loads straight into
// registers and occupancy (2 CTAs/SM) hides the load latency.
bool jit_double_buffer() { return false; }

// One CTA per tile (default) or the persistent grid (QSV_JIT_GRID_TILES=0)
bool jit_per_tile_grid() {
    static const bool v = !std::getenv("QSV_JIT_GRID_TILES") || std::atoi(std::getenv("QSV_JIT_GRID_TILES")) != 0;
    return v;
}

// L2 prefetch distance in tiles under one-CTA-per-tile grids (QSV_JIT_PREFETCH_DIST,
// default 2 x 148: about one wave of resident CTAs ahead); 0 with persistent grids
long gridDim_prefetch_distance() {
    if (!jit_per_tile_grid()) return 0;
    static const long d = std::getenv("QSV_JIT_PREFETCH_DIST") ? std::atol(std::getenv("QSV_JIT_PREFETCH_DIST")) : 296;
    return d;
}

namespace {

// Shared-memory slot map of one pass: slot(e) = e ^ G(e), G linear from the
// local bits >= 3 into the low 3 bits (16-byte slots, 8 per 128-byte bank
// row).  A stage's 128-bit accesses are conflict-free when the three local
// bits carried by lanes 0-2 of a warp map to independent bank bits; the map
// is chosen per pass so that this holds for every stage's lane layout (the
// fixed XOR fold i ^ (i>>3) ^ (i>>6) ^ (i>>9) fails whenever two of those
// bits are congruent mod 3: 2-way conflicts, measured 271M on one C2 pass).
struct SmemMap {
    uint32_t g[32];
    SmemMap() {
        for (int j = 0; j < 32; ++j) g[j] = 1u << ((j + 3) % 3);
    }
    uint32_t vec(int p) const { return p < 3 ? (1u << p) : g[p - 3]; }
    uint32_t map(uint32_t e) const {
        uint32_t x = e;
        for (int p = 3; p < 32; ++p)
            if ((e >> p) & 1) x ^= g[p - 3];
        return x;
    }
    // slot of the local index deposit(tid, bits) as a runtime expression
    std::string tid_expr(const std::vector<int> &bits) const;
};

bool independent3(uint32_t a, uint32_t b, uint32_t c) {
    return a && b && c && a != b && (a ^ b) != c && a != c && b != c;
}

// lane_sets: for each stage, the local bits carried by lanes 0, 1, 2
SmemMap choose_smem_map(const std::vector<std::vector<int>> &lane_sets) {
    SmemMap M;
    std::vector<int> vars;  // high positions that appear in some lane set
    for (const auto &ls : lane_sets)
        for (int p : ls)
            if (p >= 3 && std::find(vars.begin(), vars.end(), p) == vars.end()) vars.push_back(p);
    auto ok_all = [&](size_t assigned) {
        for (const auto &ls : lane_sets) {
            if (ls.size() < 3) continue;
            bool ready = true;
            for (int p : ls)
                if (p >= 3) ready &= std::find(vars.begin(), vars.begin() + (long)assigned, p) != vars.begin() + (long)assigned;
            if (ready && !independent3(M.vec(ls[0]), M.vec(ls[1]), M.vec(ls[2]))) return false;
        }
        return true;
    };
    std::function<bool(size_t)> solve = [&](size_t k) -> bool {
        if (k == vars.size()) return true;
        const int j = vars[k] - 3;
        const uint32_t def = 1u << (vars[k] % 3);
        for (uint32_t t = 0; t < 8; ++t) {
            M.g[j] = t == 0 ? def : (t == def ? 0 : t);  // the default first
            if (M.g[j] && ok_all(k + 1) && solve(k + 1)) return true;
        }
        M.g[j] = def;
        return false;
    };
    if (!solve(0)) return SmemMap();  // not found: default map (correct, may conflict)
    return M;
}

std::string SmemMap::tid_expr(const std::vector<int> &bits) const {
    std::string e = "(" + deposit_expr("tid", bits, false) + ")";
    for (size_t k = 0; k < bits.size(); ++k) {
        const uint32_t v = bits[k] >= 3 ? g[bits[k] - 3] : 0u;
        if (v) e += " ^ (((tid >> " + std::to_string(k) + ") & 1u) * " + std::to_string(v) + "u)";
    }
    return e;
}


struct StageGen {
    std::ostringstream &o;
    int R;
    const std::vector<int> &tq;     // tile qubits by local bit
    std::vector<int> regq;          // register position k -> global qubit
    std::map<int, int> thread_bit;  // global qubit -> thread id bit (stage thread bits)
    std::vector<cd> pend;           // pending constant phase per register amplitude
    double fp64 = 0;                // FP64 instructions emitted per thread (cost model)
    // runtime diagonal accumulators: qG (thread-wide) and qA<k>_<b> (factor
    // for amplitudes whose register bit k is b); they collect every diagonal
    // factor that depends on thread/tile bits, applied once per stage
    std::vector<int> acc;           // acc[2k+b]: accumulator in use
    bool accG = false;
    // factors not yet multiplied into their accumulator: per accumulator
    // (k, b; k = -1: qG) a list of (scalar qubits, control condition, value
    // table over the scalar bits).  Factors with the same scalar qubits and
    // condition multiply at compile time (QFT: all CR phases controlled by one
    // thread/tile qubit become one complex multiply per accumulator)
    struct PendFactor {
        std::vector<int> sq;
        std::string ccond;
        std::vector<cd> val;
    };
    std::map<std::pair<int, int>, std::vector<PendFactor>> pacc;
    // runtime sign flips (CZ-like diagonals on thread/tile qubits): each
    // register amplitude carries a pending set of runtime sign variables
    // (bit i <-> variable sg<id[i]>), applied to the sign bits with integer
    // XORs only when the amplitude meets a differently signed partner in a
    // gate, and at stage end
    std::vector<uint64_t> psign;
    std::vector<std::string> svar;  // condition of each live variable
    std::vector<int> svar_id;       // its emitted name
    std::map<uint64_t, std::string> smask;
    int next_id = 0;

    int T = 0;                  // threads per tile (per-thread factor tables)
    bool host_render = false;

    StageGen(std::ostringstream &out, int r, const std::vector<int> &t)
        : o(out), R(r), tq(t), pend(1u << r, cd(1, 0)), acc(2 * r, 0), psign(1u << r, 0) {}

    void apply_sign(int rho) {
        apply_sign_set(rho, psign[rho]);
        psign[rho] = 0;
    }
    void apply_sign_set(int rho, uint64_t set) {
        if (!set) return;
        auto it = smask.find(set);
        if (it == smask.end()) {
            std::string e;
            for (int i = 0; i < 64; ++i)
                if ((set >> i) & 1) e += (e.empty() ? "" : " ^ ") + std::string("sg") + std::to_string(svar_id[i]);
            const std::string name = "sm" + std::to_string(next_id++);
            o << "    const u64 " << name << " = " << e << ";\n";
            it = smask.emplace(set, name).first;
        }
        const std::string v = "v" + std::to_string(rho);
        o << "    " << v << " = make_double2(xsg(" << v << ".x, " << it->second << "), xsg(" << v << ".y, "
          << it->second << "));\n";
    }
    void apply_signs() {
        for (int r = 0; r < (1 << R); ++r) apply_sign(r);
        svar.clear();
        svar_id.clear();
        smask.clear();
    }
    // a group of amplitudes entering one gate: a common sign commutes with it.
    // Otherwise every member's sign is applied (keeping the most frequent set
    // pending instead was measured to cost more flips later in the stage).
    void signs_for_group(const std::vector<int> &grp) {
        bool same = true;
        for (int r : grp) same &= psign[r] == psign[grp[0]];
        if (!same)
            for (int r : grp) apply_sign(r);
    }
    int sign_var(const std::string &cond) {
        for (size_t i = 0; i < svar.size(); ++i)
            if (svar[i] == cond) return (int)i;
        if (svar.size() == 64) apply_signs();
        const int id = next_id++;
        o << "    const u64 sg" << id << " = (u64)(" << cond << ") << 63;\n";
        svar.push_back(cond);
        svar_id.push_back(id);
        return (int)svar.size() - 1;
    }

    static std::string c2(cd c) { return "make_double2(" + lit(c.real()) + ", " + lit(c.imag()) + ")"; }

    void declare_accumulators() {
        o << "    double2 qG = make_double2(1.0, 0.0);";
        for (int k = 0; k < R; ++k)
            o << " double2 qA" << k << "_0 = qG, qA" << k << "_1 = qG;";
        o << "\n";
    }

    // emits the folded pending factors of accumulator (k, b) (k = -1: qG)
    void materialize(int k, int b) {
        auto it = pacc.find({k, b});
        if (it == pacc.end()) return;
        const std::string name = k < 0 ? std::string("qG") : "qA" + std::to_string(k) + "_" + std::to_string(b);
        const std::string one = "make_double2(1.0, 0.0)";
        // factors over thread bits only (no control condition) fold into one
        // per-thread table, indexed by tid: one load and one complex multiply
        // instead of a select chain + multiply per factor (QFT: the CR phases
        // of every thread-bit control of a register target)
        std::vector<const PendFactor *> thr;
        for (const PendFactor &f : it->second) {
            bool only = f.ccond.empty() && !f.sq.empty();
            for (int q : f.sq) only &= thread_bit.count(q) > 0;
            if (only) thr.push_back(&f);
        }
        if (g_decls && thr.size() >= 2 && T > 0) {
            std::vector<cd> tab((size_t)T, cd(1, 0));
            for (int tid = 0; tid < T; ++tid)
                for (const PendFactor *f : thr) {
                    int combo = 0;
                    for (size_t si = 0; si < f->sq.size(); ++si)
                        combo |= ((tid >> thread_bit.at(f->sq[si])) & 1) << si;
                    tab[tid] *= f->val[combo];
                }
            const std::string tname = "qtab" + std::to_string(g_decl_id++);
            *g_decls << (host_render ? "static const double2 " : "__device__ const double2 ") << tname << "[" << T
                     << "] = {";
            for (int tid = 0; tid < T; ++tid) {
                const cd c = snap(tab[tid]);
                *g_decls << (tid ? ", " : "") << "{" << lit(c.real()) << ", " << lit(c.imag()) << "}";
            }
            *g_decls << "};\n";
            o << "    " << name << " = cmulc(" << name << ", " << tname << "[tid]);\n";
            fp64 += 4;
        } else {
            thr.clear();
        }
        // factors over tile-external bits only are uniform over the CTA: groups of up to six
        // external qubits fold into one table indexed by those bits of the tile's base index,
        // one load and one complex multiply per group instead of a select + multiply per
        // control qubit (QFT: the CR phases of the 18 external controls of a register target
        // were 216 of the middle pass's 468 complex multiplies per thread and every FSEL)
        std::vector<const PendFactor *> ext;
        for (const PendFactor &f : it->second) {
            bool only = f.ccond.empty() && !f.sq.empty() && f.sq.size() <= 6;
            for (int q : f.sq) only &= thread_bit.count(q) == 0;
            if (only) ext.push_back(&f);
        }
        if (g_decls && ext.size() >= 2) {
            std::vector<const PendFactor *> order = ext;
            std::stable_sort(order.begin(), order.end(), [](const PendFactor *a, const PendFactor *b) {
                return *std::min_element(a->sq.begin(), a->sq.end()) < *std::min_element(b->sq.begin(), b->sq.end());
            });
            std::vector<std::pair<std::vector<int>, std::vector<const PendFactor *>>> chunks;
            for (const PendFactor *f : order) {
                bool placed = false;
                if (!chunks.empty()) {
                    std::vector<int> u = chunks.back().first;
                    for (int q : f->sq)
                        if (std::find(u.begin(), u.end(), q) == u.end()) u.push_back(q);
                    if (u.size() <= 6) {
                        chunks.back().first = u;
                        chunks.back().second.push_back(f);
                        placed = true;
                    }
                }
                if (!placed) chunks.push_back({f->sq, {f}});
            }
            for (auto &ch : chunks) {
                std::vector<int> &cq = ch.first;
                std::sort(cq.begin(), cq.end());
                const int nq = (int)cq.size();
                std::vector<cd> tab((size_t)1 << nq, cd(1, 0));
                for (int x = 0; x < (1 << nq); ++x)
                    for (const PendFactor *f : ch.second) {
                        int combo = 0;
                        for (size_t si = 0; si < f->sq.size(); ++si) {
                            const int pos = (int)(std::find(cq.begin(), cq.end(), f->sq[si]) - cq.begin());
                            combo |= ((x >> pos) & 1) << si;
                        }
                        tab[x] *= f->val[combo];
                    }
                bool trivial = true;
                for (const cd &c : tab) trivial &= snap(c) == cd(1, 0);
                if (trivial) continue;
                const std::string tname = "qtab" + std::to_string(g_decl_id++);
                *g_decls << (host_render ? "static const double2 " : "__device__ const double2 ") << tname << "["
                         << (1 << nq) << "] = {";
                for (int x = 0; x < (1 << nq); ++x) {
                    const cd c = snap(tab[x]);
                    *g_decls << (x ? ", " : "") << "{" << lit(c.real()) << ", " << lit(c.imag()) << "}";
                }
                *g_decls << "};\n";
                // index: bit i <-> external qubit cq[i]; contiguous qubits are one shift + mask
                std::string idx;
                if (cq.back() - cq.front() == nq - 1) {
                    idx = "((unsigned)(base >> " + std::to_string(cq.front()) + ") & " + std::to_string((1 << nq) - 1) + "u)";
                } else {
                    for (int i = 0; i < nq; ++i)
                        idx += (i ? " | " : "") + std::string("(((unsigned)(base >> ") + std::to_string(cq[i]) +
                               ") & 1u) << " + std::to_string(i) + ")";
                    idx = "(" + idx + ")";
                }
                o << "    " << name << " = cmulc(" << name << ", " << tname << "[" << idx << "]);\n";
                fp64 += 4;
            }
        } else {
            ext.clear();
        }
        for (const PendFactor &f : it->second) {
            if (std::find(thr.begin(), thr.end(), &f) != thr.end()) continue;
            if (std::find(ext.begin(), ext.end(), &f) != ext.end()) continue;
            const std::string e = select_from(f.sq, f.val);
            if (e == c2(cd(1, 0))) continue;
            const std::string g = f.ccond.empty() ? e : "((" + f.ccond + ") ? " + e + " : " + one + ")";
            o << "    " << name << " = cmulc(" << name << ", " << g << ");\n";
            fp64 += 4;
        }
        pacc.erase(it);
    }
    void materialize_all() {
        materialize(-1, 0);
        for (int k = 0; k < R; ++k)
            for (int b = 0; b < 2; ++b) materialize(k, b);
    }

    // apply + reset the accumulators of register position k
    void flush_acc(int k) {
        materialize(k, 0);
        materialize(k, 1);
        for (int b = 0; b < 2; ++b) {
            if (!acc[2 * k + b]) continue;
            for (int rho = 0; rho < (1 << R); ++rho)
                if (((rho >> k) & 1) == b) o << "    v" << rho << " = cmulc(v" << rho << ", qA" << k << "_" << b << ");\n";
            o << "    qA" << k << "_" << b << " = make_double2(1.0, 0.0);\n";
            acc[2 * k + b] = 0;
            fp64 += 4.0 * (1 << (R - 1));
        }
    }

    // stage end: one product table over the active accumulators, then one
    // complex multiply per amplitude (plus its compile-time pending factor)
    void flush_runtime() {
        materialize_all();
        std::vector<int> used;
        for (int k = 0; k < R; ++k)
            if (acc[2 * k] || acc[2 * k + 1]) used.push_back(k);
        if (used.empty() && !accG) return;
        // product tables over groups of the active register bits: one table
        // over all of them costs 2^|used| live temporaries (spills at r = 5:
        // QFT); with four or more bits two tables (~2 and ~3 bits) take fewer
        // multiplies in total and a quarter of the registers
        std::vector<std::vector<int>> groups;
        if (used.size() >= 4) {
            const size_t a = used.size() / 2;
            groups.push_back(std::vector<int>(used.begin(), used.begin() + (long)a));
            groups.push_back(std::vector<int>(used.begin() + (long)a, used.end()));
        } else {
            groups.push_back(used);
        }
        int id = 0;
        std::vector<std::vector<std::string>> tabs;
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            std::vector<std::string> tab = {gi == 0 && accG ? "qG" : ""};
            const std::vector<int> &grp = groups[gi];
            for (size_t u = 0; u < grp.size(); ++u) {
                const int k = grp[u];
                // entry index: bit u <-> register bit of position grp[u]
                std::vector<std::string> next(2 * tab.size());
                for (size_t j = 0; j < tab.size(); ++j)
                    for (int b = 0; b < 2; ++b) {
                        const std::string &t = tab[j];
                        const std::string a = "qA" + std::to_string(k) + "_" + std::to_string(b);
                        std::string &dst = next[j | ((size_t)b << u)];
                        if (!acc[2 * k + b]) {
                            dst = t;
                        } else if (t.empty()) {
                            dst = a;
                        } else {
                            dst = "qT" + std::to_string(id++);
                            o << "    const double2 " << dst << " = cmulc(" << t << ", " << a << ");\n";
                            fp64 += 4;
                        }
                    }
                tab.swap(next);
            }
            tabs.push_back(tab);
        }
        for (int rho = 0; rho < (1 << R); ++rho)
            for (size_t gi = 0; gi < groups.size(); ++gi) {
                int idx = 0;
                for (size_t u = 0; u < groups[gi].size(); ++u) idx |= ((rho >> groups[gi][u]) & 1) << u;
                const std::string &t = tabs[gi][idx];
                if (t.empty()) continue;
                o << "    v" << rho << " = cmulc(v" << rho << ", " << t << ");\n";
                fp64 += 4;
            }
        for (int k = 0; k < 2 * R; ++k) acc[k] = 0;
        accG = false;
    }

    int regpos(int q) const {
        for (int k = 0; k < R; ++k)
            if (regq[k] == q) return k;
        return -1;
    }
    // runtime expression of a non-register qubit's bit value
    std::string scalar_expr(int q) const {
        auto it = thread_bit.find(q);
        if (it != thread_bit.end()) return "((tid >> " + std::to_string(it->second) + ") & 1u)";
        return "((unsigned)(base >> " + std::to_string(q) + ") & 1u)";
    }

    void mul_const(int rho, cd c) {
        const std::string v = "v" + std::to_string(rho);
        c = snap(c);
        const double cr = c.real(), ci = c.imag();
        if (cr == 1.0 && ci == 0.0) return;
        fp64 += flush_cost(c);
        const char *neg = "0x8000000000000000ull";
        if (std::fabs(cr) == 1.0 && std::fabs(ci) == 1.0) {
            // (a + ib)(x + iy), a, b = +-1: two adds
            auto sg = [](double k) { return k > 0 ? " + " : " - "; };
            o << "    { const double2 t = " << v << "; " << v << " = make_double2(" << (cr > 0 ? "" : "-") << "t.x"
              << sg(-ci) << "t.y, " << (cr > 0 ? "" : "-") << "t.y" << sg(ci) << "t.x); }\n";
        } else if (cr == -1.0 && ci == 0.0) {
            o << "    " << v << " = make_double2(xsg(" << v << ".x, " << neg << "), xsg(" << v << ".y, " << neg << "));\n";
        } else if (ci == 0.0) {
            o << "    " << v << " = make_double2(" << v << ".x * " << lit(cr) << ", " << v << ".y * " << lit(cr) << ");\n";
        } else if (cr == 0.0) {
            if (ci == 1.0) o << "    " << v << " = make_double2(xsg(" << v << ".y, " << neg << "), " << v << ".x);\n";
            else if (ci == -1.0) o << "    " << v << " = make_double2(" << v << ".y, xsg(" << v << ".x, " << neg << "));\n";
            else
                o << "    " << v << " = make_double2(-" << v << ".y * " << lit(ci) << ", " << v << ".x * " << lit(ci)
                  << ");\n";
        } else {
            o << "    { const double2 t = " << v << "; " << v << " = make_double2(t.x * " << lit(cr) << " - t.y * "
              << lit(ci) << ", t.x * " << lit(ci) << " + t.y * " << lit(cr) << "); }\n";
        }
    }

    void flush(int rho) {
        if (pend[rho] != cd(1, 0)) {
            mul_const(rho, pend[rho]);
            pend[rho] = cd(1, 0);
        }
    }
    // FP64 cost of the stage-end multiply by c (after snap)
    static int flush_cost(cd c) {
        const double a = c.real(), b = c.imag();
        if ((b == 0.0 && std::fabs(a) == 1.0) || (a == 0.0 && std::fabs(b) == 1.0)) return 0;  // sign bits only
        if (a == 0.0 || b == 0.0 || (std::fabs(a) == 1.0 && std::fabs(b) == 1.0)) return 2;
        return 4;
    }
    // Stage end.  Amplitudes stored between stages/passes are the true ones
    // divided by a uniform real scale `sigma` that is carried forward, so
    // when every pending factor of the stage has the same magnitude (H,
    // RX/RY(pi/2), sqrt(X), T, CZ... all do) only its phase is multiplied in:
    // +-1 / +-i then cost no FP64 at all and (+-1 +-i) two adds.  The final
    // stage of the plan multiplies the scale back in.
    void flush_all(double &sigma, bool final) {
        flush_runtime();
        const int A = 1 << R;
        double mu = 0;
        if (!final) {
            const double m0 = std::abs(pend[0]);
            bool uniform = m0 > 0;
            for (int r = 1; r < A && uniform; ++r) uniform = std::fabs(std::abs(pend[r]) - m0) <= kSnap * m0;
            // keep the carried scale within +-2^200
            const double next = std::fabs(std::log2(sigma * m0));
            if (uniform && next < 200) {
                int best = 1 << 30;
                for (double cand : {m0, m0 * std::sqrt(0.5)}) {
                    int c = 0;
                    for (int r = 0; r < A; ++r) c += flush_cost(snap(pend[r] / cand));
                    if (c < best) {
                        best = c;
                        mu = cand;
                    }
                }
            }
        }
        if (final) {
            for (int r = 0; r < A; ++r) pend[r] *= sigma;
            sigma = 1.0;
        } else if (mu > 0) {
            for (int r = 0; r < A; ++r) pend[r] /= mu;
            sigma *= mu;
        }
        for (int r = 0; r < A; ++r) flush(r);
        apply_signs();
    }

    // complex linear map on register amplitudes idx[0..d) : out_r = sum_c M[r*d+c] in_c
    void linear(const std::vector<int> &idx, const cd *M) {
        const int d = (int)idx.size();
        o << "    {";
        for (int c = 0; c < d; ++c) o << " const double2 i" << c << " = v" << idx[c] << ";";
        o << "\n";
        for (int r = 0; r < d; ++r) {
            auto comp = [&](bool im) {
                std::ostringstream e;
                bool any = false;
                for (int c = 0; c < d; ++c) {
                    const double mr = M[r * d + c].real(), mi = M[r * d + c].imag();
                    // re: mr*x - mi*y ; im: mr*y + mi*x
                    const std::string x = "i" + std::to_string(c) + ".x", y = "i" + std::to_string(c) + ".y";
                    const double c1 = mr, c2 = im ? mi : -mi;
                    const std::string t1 = im ? y : x, t2 = im ? x : y;
                    for (int part = 0; part < 2; ++part) {
                        const double k = part == 0 ? c1 : c2;
                        const std::string &t = part == 0 ? t1 : t2;
                        if (k == 0.0) continue;
                        if (k == 1.0) e << (any ? " + " : "") << t;
                        else if (k == -1.0) e << (any ? " - " : "-") << t;
                        else e << (any ? " + " : "") << t << " * " << lit(k);
                        any = true;
                    }
                }
                if (any) {
                    int terms = 0, muls = 0;
                    for (int c = 0; c < d; ++c) {
                        const double mr = M[r * d + c].real(), mi = M[r * d + c].imag();
                        for (double k : {mr, mi})
                            if (k != 0.0) {
                                ++terms;
                                if (k != 1.0 && k != -1.0) ++muls;
                            }
                    }
                    // fma chains: one op per term after the first, plus a multiply
                    // when every term carries a coefficient
                    fp64 += (terms - 1) + (muls == terms ? 1 : 0);
                }
                return any ? e.str() : std::string("0.0");
            };
            o << "      v" << idx[r] << " = make_double2(" << comp(false) << ", " << comp(true) << ");\n";
        }
        o << "    }\n";
    }

    // FP64 cost class of multiplying by a constant coefficient in a linear row
    static int coeff_cost(cd z) {
        const double a = z.real(), b = z.imag();
        if ((b == 0.0 && (a == 1.0 || a == -1.0)) || (a == 0.0 && (b == 1.0 || b == -1.0))) return 1;
        if (a == 0.0 || b == 0.0) return 2;
        return 4;
    }
    // Canonicalise a coefficient that products of gate matrices left a few
    // ulps off an exact form: a zero component, a unit, or equal |re| = |im|
    // (the pi/4 phases of T-type gates).  kSnap (relative) is far below the
    // 1e-10 parity tolerance and far above accumulated rounding.
    static constexpr double kSnap = 1e-13;
    static cd snap(cd z) {
        const double eps = kSnap * std::abs(z);
        double a = z.real(), b = z.imag();
        if (std::fabs(a) <= eps) a = 0.0;
        if (std::fabs(b) <= eps) b = 0.0;
        for (double u : {1.0, -1.0}) {
            if (std::fabs(a - u) <= kSnap && b == 0.0) a = u;
            if (std::fabs(b - u) <= kSnap && a == 0.0) b = u;
        }
        if (a != 0.0 && b != 0.0 && std::fabs(std::fabs(a) - std::fabs(b)) <= eps) {
            const double h = 0.5 * (std::fabs(a) + std::fabs(b));
            a = std::copysign(h, a);
            b = std::copysign(h, b);
        }
        return cd(a, b);
    }
    static bool diag_phase(cd z) { return z.real() != 0.0 && std::fabs(z.real()) == std::fabs(z.imag()); }

    // linear map that first absorbs the inputs' pending factors into the
    // compile-time coefficients, then factors one coefficient out of every
    // output row (chosen to make the rest cheapest) and leaves it pending on
    // that output.  H, sqrt(X), sqrt(Y) and phase-preceded gates become
    // add/subtract rows; the pending factors are absorbed by the next gate or
    // multiplied in once at the end of the stage.
    void linear_absorb(const std::vector<int> &idx, const cd *M) {
        const int d = (int)idx.size();
        std::vector<cd> Mp(d * d), Mn(d * d);
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) Mp[r * d + c] = M[r * d + c] * pend[idx[c]];
        if (d == 2 && pair_rotated(idx, Mp)) return;
        std::vector<cd> newp(d, cd(1, 0));
        for (int r = 0; r < d; ++r) {
            double mx = 0;
            for (int c = 0; c < d; ++c) mx = std::max(mx, std::abs(Mp[r * d + c]));
            if (mx == 0.0) {
                for (int c = 0; c < d; ++c) Mn[r * d + c] = 0;
                continue;
            }
            int best = -1, best_cost = 1 << 30;
            for (int k = 0; k < d; ++k) {
                const cd ck = Mp[r * d + k];
                if (std::abs(ck) < 0.5 * mx) continue;
                int cost = 0;
                for (int c = 0; c < d; ++c)
                    if (c != k && Mp[r * d + c] != cd(0, 0)) cost += coeff_cost(snap(Mp[r * d + c] / ck));
                if (cost < best_cost) {
                    best_cost = cost;
                    best = k;
                }
            }
            const cd ck = Mp[r * d + best];
            for (int c = 0; c < d; ++c)
                Mn[r * d + c] = c == best ? cd(1, 0) : (Mp[r * d + c] == cd(0, 0) ? cd(0, 0) : snap(Mp[r * d + c] / ck));
            newp[r] = ck;
        }
        linear(idx, Mn.data());
        for (int r = 0; r < d; ++r) pend[idx[r]] = newp[r];
    }

    // A 2x2 block whose rows, each normalised on the same column k, read
    // (1, c0) and (1, c1) with c0, c1 on one pi/4 diagonal (c_r = a_r (+-1 +-i),
    // a_r real - always the case for a unitary block whose off-column phase is
    // an odd multiple of pi/4): rotate the other input once, w = (+-1 +-i) x_o
    // (two adds), then each row is x_k + a_r w (two FMAs): 6 FP64 per pair
    // instead of 8.
    bool pair_rotated(const std::vector<int> &idx, const std::vector<cd> &Mp) {
        for (int k = 0; k < 2; ++k) {
            const int oc = 1 - k;
            if (std::abs(Mp[k]) == 0.0 || std::abs(Mp[2 + k]) == 0.0) continue;
            if (std::abs(Mp[k]) < 0.5 * std::abs(Mp[oc]) || std::abs(Mp[2 + k]) < 0.5 * std::abs(Mp[2 + oc])) continue;
            const cd c0 = snap(Mp[oc] / Mp[k]), c1 = snap(Mp[2 + oc] / Mp[2 + k]);
            if (!diag_phase(c0) || !diag_phase(c1)) continue;
            const cd u(c0.real() > 0 ? 1.0 : -1.0, c0.imag() > 0 ? 1.0 : -1.0);  // c0 = a0 u, a0 > 0
            const double a0 = (c0 * std::conj(u)).real() / 2.0, a1 = (c1 * std::conj(u)).real() / 2.0;
            if (std::fabs((c1 * std::conj(u)).imag()) > kSnap * std::abs(c1)) continue;  // c1 not along u
            const std::string xo = "i" + std::to_string(oc), xk = "i" + std::to_string(k);
            // w = u * x_o with u = (ur + i ui), ur, ui = +-1
            auto sgn = [](double v) { return v > 0 ? " + " : " - "; };
            o << "    { const double2 i0 = v" << idx[0] << "; const double2 i1 = v" << idx[1] << ";\n";
            o << "      const double2 w = make_double2(" << (u.real() > 0 ? "" : "-") << xo << ".x" << sgn(-u.imag()) << xo
              << ".y, " << (u.real() > 0 ? "" : "-") << xo << ".y" << sgn(u.imag()) << xo << ".x);\n";
            for (int r = 0; r < 2; ++r) {
                const double a = r == 0 ? a0 : a1;
                auto term = [&](const char *comp) {
                    const std::string wc = std::string("w.") + comp;
                    if (a == 1.0) return xk + "." + comp + " + " + wc;
                    if (a == -1.0) return xk + "." + comp + " - " + wc;
                    return xk + "." + comp + " + " + wc + " * " + lit(a);
                };
                o << "      v" << idx[r] << " = make_double2(" << term("x") << ", " << term("y") << ");\n";
            }
            o << "    }\n";
            fp64 += 6;
            pend[idx[0]] = Mp[k];
            pend[idx[1]] = Mp[2 + k];
            return true;
        }
        return false;
    }

    std::string scalar_cond(uint64_t smask) const {
        std::string c;
        for (int q = 0; q < 64; ++q)
            if ((smask >> q) & 1) c += (c.empty() ? "" : " && ") + scalar_expr(q);
        return c;
    }

    // factor expression over the scalar target bits (nested selects of constants)
    std::string select_expr(const std::vector<int> &dq, const std::vector<cd> &d, const std::vector<int> &sq,
                            int reg_t, int reg_bit) const {
        // enumerate scalar assignments; build a chain of ternaries
        const int ns = (int)sq.size();
        std::vector<cd> val(1u << ns);
        for (int combo = 0; combo < (1 << ns); ++combo) {
            int idx = 0;
            for (size_t t = 0; t < dq.size(); ++t) {
                int bit;
                if ((int)t == reg_t) bit = reg_bit;
                else {
                    int si = 0;
                    while (sq[si] != dq[t]) ++si;
                    bit = (combo >> si) & 1;
                }
                idx = 2 * idx + bit;
            }
            val[combo] = d[idx];
        }
        std::function<std::string(int, int)> build = [&](int si, int prefix) -> std::string {
            if (si == ns) return c2(val[prefix]);
            const std::string a = build(si + 1, prefix), b = build(si + 1, prefix | (1 << si));
            if (a == b) return a;
            return "(" + scalar_expr(sq[si]) + " ? " + b + " : " + a + ")";
        };
        return build(0, 0);
    }

    // nested selects of constants over the scalar bits sq (val indexed by combo)
    std::string select_from(const std::vector<int> &sq, const std::vector<cd> &val) const {
        const int ns = (int)sq.size();
        std::function<std::string(int, int)> build = [&](int si, int prefix) -> std::string {
            if (si == ns) return c2(val[prefix]);
            const std::string a = build(si + 1, prefix), b = build(si + 1, prefix | (1 << si));
            if (a == b) return a;
            return "(" + scalar_expr(sq[si]) + " ? " + b + " : " + a + ")";
        };
        return build(0, 0);
    }

    // value table of the factor over the scalar bits for register bit reg_bit
    std::vector<cd> factor_table(const std::vector<int> &dq, const std::vector<cd> &d, const std::vector<int> &sq,
                                 int reg_t, int reg_bit) const {
        const int ns = (int)sq.size();
        std::vector<cd> val(1u << ns);
        for (int combo = 0; combo < (1 << ns); ++combo) {
            int idx = 0;
            for (size_t t = 0; t < dq.size(); ++t) {
                int bit;
                if ((int)t == reg_t) bit = reg_bit;
                else {
                    int si = 0;
                    while (sq[si] != dq[t]) ++si;
                    bit = (combo >> si) & 1;
                }
                idx = 2 * idx + bit;
            }
            val[combo] = d[idx];
        }
        return val;
    }

    void defer(int k, int b, const std::vector<int> &sq, const std::string &ccond, const std::vector<cd> &val) {
        bool trivial = true;
        for (const cd &x : val) trivial &= x == cd(1, 0);
        if (trivial) return;
        std::vector<PendFactor> &lst = pacc[{k, b}];
        for (PendFactor &f : lst)
            if (f.sq == sq && f.ccond == ccond) {
                for (size_t i = 0; i < val.size(); ++i) f.val[i] *= val[i];
                return;
            }
        lst.push_back(PendFactor{sq, ccond, val});
    }

    void accumulate(const std::vector<int> &dq, const std::vector<cd> &d, const std::vector<int> &sq,
                    const std::string &ccond) {
        int reg_t = -1;
        for (size_t t = 0; t < dq.size(); ++t)
            if (regpos(dq[t]) >= 0) reg_t = (int)t;
        if (reg_t < 0) {
            defer(-1, 0, sq, ccond, factor_table(dq, d, sq, -1, 0));
            accG = true;
            return;
        }
        const int k = regpos(dq[reg_t]);
        for (int b = 0; b < 2; ++b) {
            const std::vector<cd> val = factor_table(dq, d, sq, reg_t, b);
            bool trivial = true;
            for (const cd &x : val) trivial &= x == cd(1, 0);
            if (trivial) continue;
            defer(k, b, sq, ccond, val);
            acc[2 * k + b] = 1;
        }
    }

    void op(const GlobalOp &g) {
        uint32_t rcm = 0;
        uint64_t smask = 0;
        for (int q = 0; q < 64; ++q) {
            if (!((g.cmask >> q) & 1)) continue;
            const int k = regpos(q);
            if (k >= 0) rcm |= 1u << k;
            else smask |= 1ull << q;
        }
        if (g.kind == QSV_OP_MAT1 || g.kind == QSV_OP_MAT2) {
            const int A = regpos(g.qa);
            const int B = g.kind == QSV_OP_MAT2 ? regpos(g.qb) : -1;
            const uint32_t tb = (1u << A) | (B >= 0 ? 1u << B : 0u);
            std::vector<std::vector<int>> groups;
            for (int rho = 0; rho < (1 << R); ++rho) {
                if ((rho & tb) || (rho & rcm) != rcm) continue;
                if (B < 0) groups.push_back({rho, rho | (1 << A)});
                else groups.push_back({rho, rho | (1 << B), rho | (1 << A), rho | (1 << A) | (1 << B)});
            }
            flush_acc(A);
            if (B >= 0) flush_acc(B);
            for (auto &grp : groups) signs_for_group(grp);
            const std::string cond = scalar_cond(smask);
            if (cond.empty()) {
                for (auto &grp : groups) linear_absorb(grp, g.m);
                return;
            }
            // a thread/tile-dependent control: pending factors must be applied
            // on both sides of the branch, so materialise them first
            for (auto &grp : groups)
                for (int r : grp) flush(r);
            o << "    if (" << cond << ") {\n";
            for (auto &grp : groups) linear(grp, g.m);
            o << "    }\n";
            return;
        }
        // diagonal: factor(rho, scalars) = controls ? d[bits] : 1
        std::vector<int> dq = {g.qa};
        std::vector<cd> d = {g.m[0], g.m[1]};
        if (g.kind == QSV_OP_DIAG2) {
            dq = {g.qa, g.qb};
            d = {g.m[0], g.m[1], g.m[2], g.m[3]};
        }
        // fold the controls into the diagonal itself (a controlled diagonal is a
        // diagonal over controls + targets that is 1 unless every control is
        // set), so a register control costs nothing and a thread/tile control
        // becomes one more select bit of a runtime accumulator
        {
            std::vector<int> cq;
            for (int q = 0; q < 64; ++q)
                if ((g.cmask >> q) & 1) cq.push_back(q);
            if (!cq.empty() && cq.size() + dq.size() <= 8) {
                const int nc = (int)cq.size(), nt = (int)dq.size();
                std::vector<cd> full(1u << (nc + nt), cd(1, 0));
                for (int t = 0; t < (1 << nt); ++t) full[(((1 << nc) - 1) << nt) | t] = d[t];
                std::vector<int> all = cq;
                all.insert(all.end(), dq.begin(), dq.end());
                dq.swap(all);
                d.swap(full);
                rcm = 0;
                smask = 0;
            }
        }
        std::vector<int> sq;  // scalar target qubits
        for (int q : dq)
            if (regpos(q) < 0) sq.push_back(q);
        const std::string ccond = scalar_cond(smask);
        const int ns = (int)sq.size();
        const int nreg = (int)dq.size() - ns;
        bool signs_only = true;  // +-1 factors: sign flips in a branch are cheaper than accumulating
        for (const cd &x : d) signs_only &= x.imag() == 0.0 && (x.real() == 1.0 || x.real() == -1.0);
        if ((ns > 0 || !ccond.empty()) && rcm == 0 && nreg <= 1 && !signs_only) {
            accumulate(dq, d, sq, ccond);
            return;
        }
        for (int combo = 0; combo < (1 << ns); ++combo) {
            std::vector<cd> f(1u << R, cd(1, 0));
            bool any = false;
            for (int rho = 0; rho < (1 << R); ++rho) {
                if ((rho & rcm) != rcm) continue;
                int idx = 0;
                for (size_t t = 0; t < dq.size(); ++t) {
                    const int k = regpos(dq[t]);
                    int bit;
                    if (k >= 0) bit = (rho >> k) & 1;
                    else {
                        int si = 0;
                        while (sq[si] != dq[t]) ++si;
                        bit = (combo >> si) & 1;
                    }
                    idx = 2 * idx + bit;
                }
                f[rho] = d[idx];
                if (f[rho] != cd(1, 0)) any = true;
            }
            if (!any) continue;
            if (ns == 0 && ccond.empty()) {
                for (int rho = 0; rho < (1 << R); ++rho) pend[rho] *= f[rho];
                continue;
            }
            std::string cond = ccond;
            for (int si = 0; si < ns; ++si)
                cond += (cond.empty() ? "" : " && ") + std::string((combo >> si) & 1 ? "" : "!") + scalar_expr(sq[si]);
            if (signs_only) {
                // runtime sign: one more pending sign variable, no FP64
                const int var = sign_var(cond);
                for (int rho = 0; rho < (1 << R); ++rho)
                    if (f[rho] == cd(-1, 0)) psign[rho] ^= 1ull << var;
                continue;
            }
            o << "    if (" << cond << ") {\n";
            for (int rho = 0; rho < (1 << R); ++rho) mul_const(rho, f[rho]);
            o << "    }\n";
        }
    }
};

}  // namespace

bool jit_available(std::string &why) {
    if (!nvrtc().ok) {
        why = nvrtc().why;
        return false;
    }
    if (!driver().ok) {
        why = driver().why;
        return false;
    }
    return true;
}

// Host rendering of the same kernels (test infrastructure: tests compile it
// with gcc and run it on CPU to check the generator against the oracle
// without a GPU).  Identical op emission; the CTA becomes explicit loops over
// threads between barriers and the grid becomes a sequential tile loop.
const char *kHostPrelude = R"(
#include <stdint.h>
typedef unsigned long long u64;
struct double2 { double x, y; };
static inline double2 make_double2(double x, double y) { double2 r; r.x = x; r.y = y; return r; }
static inline double2 ldcs2(const double2 *p) { return *p; }
static inline void stcs2(double2 *p, double2 v) { *p = v; }
static inline void stwb2(double2 *p, double2 v) { *p = v; }
static inline double2 ldwb2(const double2 *p) { return *p; }
static inline void prefetch_l2(const void *, unsigned) {}
static inline void prefetch_line(const void *) {}
static inline double2 cmulc(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
static inline double xsg(double x, u64 m) {
    u64 b;
    __builtin_memcpy(&b, &x, 8);
    b ^= m;
    __builtin_memcpy(&x, &b, 8);
    return x;
}
)";

// grid-wide barrier of the persistent super-pass kernel (all CTAs are
// co-resident: cooperative launch).  Monotonic counter, reset per launch.
const char *kGridSync = R"(
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &gen) {
    __syncthreads();
    gen += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned spins = 0;
        while (ld_acquire(bar) < gen) {
            __nanosleep(64);
            if (++spins > (1u << 27)) __trap();  // never hang the GPU: fail loudly
        }
        __threadfence();
    }
    __syncthreads();
}
)";

namespace {

// Emits the processing of tiles for one pass: a (persistent, double-buffered
// on the device) loop over `ntiles` tiles whose global base offset is
// `base_of(t)`; the tile body is the pass's register stages.
// Emits the processing of all tiles of one pass: a persistent loop over
// `ntiles` tiles whose global base offset is `base_of(t)`.  The FIRST stage
// loads its 2^R amplitudes straight from global memory into registers and the
// LAST stage stores them straight back (a single-stage pass never touches
// shared memory); only the re-layouts between stages go through the swizzled
// shared-memory tile.  Returns the FP64 instructions emitted per thread per
// tile (cost model).
double emit_tile_loop(std::ostringstream &o, const Plan &P, int pi, bool host, const std::string &ntiles,
                      const std::function<std::string(const std::string &)> &base_of, bool stream_out = true,
                      bool basis_param = false, bool prefetch = true, double scale_in = 1.0,
                      bool final_pass = true, double *scale_out = nullptr, int gang = 1, uint64_t xmask = 0,
                      bool tma = false, const std::vector<int> *probe = nullptr) {
    double fp64 = 0;
    double sigma = scale_in;  // stored amplitudes = true amplitudes / sigma (see StageGen::flush_all)
    const DevPass &dp = P.passes[pi];
    const int m = dp.m, R = pass_r(P, pi);
    std::vector<int> tq(dp.tq, dp.tq + m);
    const std::string thread_loop = host ? "    for (unsigned tid = 0; tid < " + std::to_string(1 << (m - R)) + "u; ++tid) {\n" : "";
    const std::string thread_end = host ? "    }\n" : "";
    const std::string barrier = host ? "" : "    __syncthreads();\n";
    const int S = dp.stage_end - dp.stage_begin;
    // product-start plan: pass 0 synthesises its input (no read, no TMA, no prefetch)
    const bool product = P.product && pi == 0 && !xmask;
    o << "  { // pass " << pi << ": " << S << " stage(s)" << (product ? ", product-state input" : "") << "\n";
    o << "  const u64 ntiles = " << ntiles << ";\n";
    // gang > 1: the CTA holds `gang` tiles side by side (sub-tile `sub`), its
    // warps run every stage in lock step (one code region in flight per SM);
    // a sub-tile past the end recomputes the last tile without storing it
    const std::string guard = (!host && gang > 1) ? "if (act) " : "";
    tma = tma && !host && !product;
    // TMA-fed tiles (QSV_JIT_TMA): the next tile (group) is brought into the
    // shared tile by bulk copies (one 2^lr-amplitude run per copy, completion
    // on an mbarrier) as soon as this tile's last shared-memory read is done,
    // so the load overlaps the last stage's math and no LDG is issued
    int tma_lr = 0;
    while (tma_lr < m && dp.tq[tma_lr] == tma_lr) ++tma_lr;
    std::vector<int> tma_runq(dp.tq + tma_lr, dp.tq + m);
    const std::string step = gang > 1 ? "(u64)gridDim.x * " + std::to_string(gang) + "u" : "(u64)gridDim.x";
    auto tma_issue = [&](const std::string &tgx) {
        // tgx: first tile of the group to load; every thread issues its runs
        o << "    if (tma_on && " << tgx << " < ntiles) {\n";
        o << "      const u64 tn = " << (gang > 1 ? "min(" + tgx + " + sub, ntiles - 1)" : tgx) << ";\n";
        o << "      const u64 bn = " << base_of("tn") << ";\n";
        o << "      if (threadIdx.x == 0) mbar_expect_tx(mbar, " << gang * (16u << m) << "u);\n";
        o << "      for (unsigned j = tid; j < " << (1u << (m - tma_lr)) << "u; j += " << (1 << (m - R)) << "u)\n";
        o << "        bulk_g2s(smem_u32(tile) + (j << " << (tma_lr + 4) << "), psi + bn + ("
          << deposit_expr("j", tma_runq, true) << "), " << (16u << tma_lr) << "u, mbar);\n";
        o << "    }\n";
    };
    if (tma) {
        o << "  __shared__ __align__(8) unsigned long long qsv_mbar;\n";
        o << "  const unsigned mbar = smem_u32(&qsv_mbar);\n  unsigned ph = 0;\n";
        o << "  const bool tma_on = " << (basis_param ? "basis == ~0ull" : "true") << ";\n";
        o << "  if (threadIdx.x == 0) mbar_init(mbar, 1);\n  __syncthreads();\n";
        tma_issue(gang > 1 ? "((u64)blockIdx.x * " + std::to_string(gang) + "u)" : "(u64)blockIdx.x");
    }
    if (host) o << "  for (u64 t = 0; t < ntiles; ++t) {\n";
    else if (gang == 1) o << "  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {\n";
    else
        o << "  for (u64 tg = (u64)blockIdx.x * " << gang << "u; tg < ntiles; tg += (u64)gridDim.x * " << gang
          << "u) {\n    const bool act = tg + sub < ntiles;\n    const u64 t = act ? tg + sub : ntiles - 1;\n";
    // QSV_JIT_DIAG_L2=1 (diagnostic only, wrong results): every CTA re-processes its
    // first tile, so the kernel runs out of L2 and its time is compute + smem + barriers
    static const bool diag_l2 = std::getenv("QSV_JIT_DIAG_L2") != nullptr;
    o << "    const u64 base = " << (diag_l2 && !host ? base_of("(u64)blockIdx.x") : base_of("t")) << ";\n";
    // exchange-out pass (sharded layout): every output amplitude goes to the
    // rank selected by its index bits at the exchanged positions `xmask`, at
    // its index with those bits replaced by this rank's own global bits
    // (QSV_XDST) - the global<->local qubit swap fused into the pass's stores
    // (remote stores over NVLink into the peer's receive buffer)
    SmemMap smap;
    {
        std::vector<std::vector<int>> lane_sets;
        for (int s = dp.stage_begin; s < dp.stage_end; ++s) {
            std::vector<int> ls;
            for (int j = 0; j < m && ls.size() < 3; ++j)
                if (!((P.stages[s].reg_local_mask >> j) & 1)) ls.push_back(j);
            lane_sets.push_back(ls);
        }
        smap = choose_smem_map(lane_sets);
    }
    std::vector<int> natural(m - R);
    for (int j = 0; j < m - R; ++j) natural[j] = j;
    for (int s = dp.stage_begin; s < dp.stage_end; ++s) {
        const DevStage &st = P.stages[s];
        const bool first = s == dp.stage_begin, last = s + 1 == dp.stage_end;
        StageGen g(o, R, tq);
        g.T = 1 << (m - R);
        g.host_render = host;
        g.regq.resize(R);
        for (int k = 0; k < R; ++k) g.regq[k] = tq[st.rb[k]];
        std::vector<int> nonreg, nonreg_q;
        for (int j = 0; j < m; ++j)
            if (!((st.reg_local_mask >> j) & 1)) {
                nonreg.push_back(j);
                nonreg_q.push_back(tq[j]);
            }
        for (size_t j = 0; j < nonreg.size(); ++j) g.thread_bit[tq[nonreg[j]]] = (int)j;
        // per register amplitude: smem slot (swizzled local index) and global offset
        std::vector<uint32_t> c(1u << R);
        std::vector<uint64_t> goff(1u << R);
        for (int rho = 0; rho < (1 << R); ++rho) {
            uint32_t off = 0;
            uint64_t go = 0;
            for (int k = 0; k < R; ++k)
                if ((rho >> k) & 1) {
                    off |= 1u << st.rb[k];
                    go |= 1ull << tq[st.rb[k]];
                }
            c[rho] = smap.map(off);
            goff[rho] = go;
        }
        // Global memory is accessed straight from the registers of the first /
        // last stage unless the stage holds qubit 0 in registers: a warp's lanes
        // would then stride through memory in 16-byte pieces (measured: C2 pass
        // with q0 q2 q4 in registers 8.5 -> 7.4 ms when staged; a stage holding
        // only q1 loses from staging), so the tile goes through shared memory
        // in the natural layout (thread tid <-> local indices tid + k*T).
        int run = 0;
        while (run < (int)nonreg.size() && nonreg[run] == run && tq[run] == run) ++run;
        static const int stage_min = std::getenv("QSV_JIT_STAGE_MIN") ? std::atoi(std::getenv("QSV_JIT_STAGE_MIN")) : 1;
        const bool synth = product && first;  // registers synthesised from the product tables
        const bool staged_in = !synth && !tma && first && run < stage_min, staged_out = last && run < stage_min;
        const int T = 1 << (m - R);
        std::vector<int> lowq(tq.begin(), tq.begin() + (m - R));
        std::vector<uint64_t> goffc(1u << R);
        std::vector<uint32_t> cc(1u << R);
        for (int k = 0; k < (1 << R); ++k) {
            uint64_t go = 0;
            for (int j = 0; j < R; ++j)
                if ((k >> j) & 1) go |= 1ull << tq[m - R + j];
            goffc[k] = go;
            cc[k] = smap.map((uint32_t)k << (m - R));
        }
        o << "    { // stage " << (s - dp.stage_begin) << " registers:";
        for (int k = 0; k < R; ++k) o << " q" << g.regq[k];
        o << (staged_in || staged_out ? " (staged through shared memory)" : "") << "\n";
        const bool staged_basis = staged_in && basis_param;  // device code only (host rendering has no basis)
        if (staged_basis) {
            // |basis>: synthesise the registers directly; otherwise stage the load
            // (the branch is uniform: basis is a kernel argument)
            o << "    const unsigned tsw = " << smap.tid_expr(nonreg) << ";\n    double2";
            for (int rho = 0; rho < (1 << R); ++rho) o << (rho ? ", v" : " v") << rho;
            o << ";\n    if (basis != ~0ull) {\n";
            o << "    const u64 gb = base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
            for (int rho = 0; rho < (1 << R); ++rho)
                o << "    v" << rho << " = make_double2(gb + " << goff[rho] << "ull == basis ? 1.0 : 0.0, 0.0);\n";
            o << "    } else {\n" << barrier << "    {\n";
            o << "    const unsigned tsc = " << smap.tid_expr(natural) << ";\n";
            o << "    double2 *gpc = psi + base + (" << deposit_expr("tid", lowq, true) << ");\n";
            for (int k = 0; k < (1 << R); ++k)
                o << "    tile[tsc ^ " << cc[k] << "u] = " << (stream_out ? "ldcs2" : "ldwb2") << "(gpc + " << goffc[k]
                  << "ull);\n";
            o << "    }\n" << barrier;
            for (int rho = 0; rho < (1 << R); ++rho) o << "    v" << rho << " = tile[tsw ^ " << c[rho] << "u];\n";
            o << "    }\n";
            if (last && !staged_out) o << "    double2 *gp = psi + base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
        } else if (staged_in) {
            // the previous tile's last stage may still read the shared tile
            o << barrier << thread_loop << "    {\n";
            o << "    const unsigned tsc = " << smap.tid_expr(natural) << ";\n";
            o << "    double2 *gpc = psi + base + (" << deposit_expr("tid", lowq, true) << ");\n";
            if (basis_param) o << "    const u64 gb = (u64)(gpc - psi);\n";
            for (int k = 0; k < (1 << R); ++k) {
                o << "    tile[tsc ^ " << cc[k] << "u] = ";
                if (basis_param)
                    o << "basis != ~0ull ? make_double2(gb + " << goffc[k] << "ull == basis ? 1.0 : 0.0, 0.0) : ";
                o << (stream_out ? "ldcs2" : "ldwb2") << "(gpc + " << goffc[k] << "ull);\n";
            }
            o << "    }\n" << thread_end << barrier;
        }
        if (synth) {
            // product-state input: amplitude(i) = prod_q v_q[bit q of i]; the thread's
            // factor over its non-register qubits from the 5-bit group tables (the
            // register bits of gb are zero), then a tree over the register qubits
            o << thread_loop;
            if (!last || staged_out) o << "    const unsigned tsw = " << smap.tid_expr(nonreg) << ";\n";
            o << "    const u64 gb = base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
            if (last && !staged_out) o << "    double2 *gp = psi + gb;\n";
            const int G = (P.n + 4) / 5;
            o << "    double2 v0 = ptab[(unsigned)(gb & 31ull)]";
            for (int rho = 1; rho < (1 << R); ++rho) o << ", v" << rho;
            o << ";\n";
            for (int gi = 1; gi < G; ++gi)
                o << "    v0 = cmulc(v0, ptab[" << 32 * gi << "u + (unsigned)((gb >> " << 5 * gi << ") & 31ull)]);\n";
            for (int k = 0; k < R; ++k) {
                o << "    { const double2 w0 = ptab[" << 32 * G + 2 * k << "u], w1 = ptab[" << 32 * G + 2 * k + 1
                  << "u];\n";
                for (int j = 0; j < (1 << k); ++j)
                    o << "      v" << (j + (1 << k)) << " = cmulc(v" << j << ", w1); v" << j << " = cmulc(v" << j
                      << ", w0);\n";
                o << "    }\n";
            }
            fp64 += 4.0 * (double)((G - 1) + (2 << R) - 2);
        } else if (!staged_basis) {
        o << thread_loop;
        if (!first || !last || staged_in || staged_out)
            o << "    const unsigned tsw = " << smap.tid_expr(nonreg) << ";\n";
        if ((first && !staged_in) || (last && !staged_out))
            o << "    double2 *gp = psi + base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
        }
        if (synth) {
        } else if (staged_basis) {
        } else if (staged_in) {
            for (int rho = 0; rho < (1 << R); ++rho) o << "    double2 v" << rho << " = tile[tsw ^ " << c[rho] << "u];\n";
        } else if (first && tma) {
            // the tile arrived by TMA in the raw layout (slot = local index)
            std::vector<uint32_t> raw(1u << R);
            for (int rho = 0; rho < (1 << R); ++rho) {
                uint32_t off = 0;
                for (int k = 0; k < R; ++k)
                    if ((rho >> k) & 1) off |= 1u << st.rb[k];
                raw[rho] = off;
            }
            o << "    if (tma_on) { mbar_wait(mbar, ph); ph ^= 1u; }\n";
            o << "    const unsigned tr = (unsigned)(" << deposit_expr("tid", nonreg, true) << ");\n";
            if (basis_param) o << "    const u64 gb = (u64)(gp - psi);\n";
            for (int rho = 0; rho < (1 << R); ++rho) {
                o << "    double2 v" << rho << " = ";
                if (basis_param)
                    o << "!tma_on ? make_double2(gb + " << goff[rho] << "ull == basis ? 1.0 : 0.0, 0.0) : ";
                o << "tile[tr + " << raw[rho] << "u];\n";
            }
        } else if (first) {
            if (basis_param) {
                // the state is |basis>: synthesise the registers instead of
                // reading 2^n amplitudes that are known
                o << "    const u64 gb = (u64)(gp - psi);\n";
                for (int rho = 0; rho < (1 << R); ++rho)
                    o << "    double2 v" << rho << " = basis != ~0ull ? make_double2(gb + " << goff[rho]
                      << "ull == basis ? 1.0 : 0.0, 0.0) : ldcs2(gp + " << goff[rho] << "ull);\n";
            } else {
                for (int rho = 0; rho < (1 << R); ++rho)
                    o << "    double2 v" << rho << " = " << (stream_out ? "ldcs2" : "ldwb2") << "(gp + " << goff[rho]
                      << "ull);\n";
            }
        } else {
            for (int rho = 0; rho < (1 << R); ++rho) o << "    double2 v" << rho << " = tile[tsw ^ " << c[rho] << "u];\n";
        }
        if (first && stream_out && !host && prefetch && !synth) {
            // TMA bulk prefetch of this CTA's NEXT tile into L2 (contiguous runs
            // of 2^lr amplitudes), so HBM streaming overlaps this tile's math
            int lr = 0;
            while (lr < m && tq[lr] == lr) ++lr;
            std::vector<int> runq(tq.begin() + lr, tq.end());
            // (fewer than 5 forced low qubits: more runs than threads, each
            // thread prefetches several)
            // persistent grid: this CTA's next tile; one CTA per tile: the tile a
            // CTA launched about one residency wave later will take
            if (gridDim_prefetch_distance() > 0 && gang == 1)
                o << "    { const u64 nt = t + " << gridDim_prefetch_distance() << "ull;\n";
            else
                o << "    { const u64 nt = t + (u64)gridDim.x * " << gang << "u;\n";
            o << "      if (nt < ntiles" << (basis_param ? " && basis == ~0ull" : "") << ")\n";
            // one prefetch per 128-byte line of the next tile (runs of 2^lb amplitudes,
            // lb = min(lr, 3): 8 amplitudes = one line when the 3 lowest qubits are resident)
            const int lb = std::min(lr, 3);
            std::vector<int> lineq(tq.begin() + lb, tq.end());
            o << "      for (unsigned j = tid; j < " << (1u << (m - lb)) << "u; j += " << T
              << "u) prefetch_line(psi + (" << base_of("nt") << ") + (" << deposit_expr("j", lineq, true)
              << ")); }\n";
        }
        const std::string next_group = gang > 1 ? "(tg + " + step + ")" : "(t + " + step + ")";
        if (tma && last && !staged_out) {
            // every thread has read this tile's registers: the shared tile is
            // free for the next tile (group) while this stage computes
            o << barrier;
            o << "    fence_proxy_async();\n";
            tma_issue(next_group);
        }
        g.declare_accumulators();
        // QSV_JIT_DIAG_NOOPS=1 (diagnostic only, wrong results): no gate math, so the kernel's
        // time is its memory traffic, shared-memory re-layouts and barriers
        static const bool diag_noops = std::getenv("QSV_JIT_DIAG_NOOPS") != nullptr;
        for (int oi = st.op_begin; oi < st.op_end && !(diag_noops && !host); ++oi) g.op(P.gops[oi]);
        g.flush_all(sigma, final_pass && last);
        fp64 += g.fp64;
        if (probe && last && !host) {
            // probe-out pass: |amp|^2 of the final amplitudes accumulated per
            // probe key (first probe qubit = MSB) while they are stored; the
            // register-qubit part of the key is compile-time per amplitude
            const int M = (int)probe->size(), B = 1 << M;
            std::vector<std::pair<int, int>> regbits;  // (probe index, register position)
            for (int i = 0; i < M; ++i)
                for (int k = 0; k < R; ++k)
                    if (g.regq[k] == (*probe)[i]) regbits.push_back({i, k});
            const int K = 1 << regbits.size();
            unsigned regmask = 0;
            for (auto &e : regbits) regmask |= 1u << (M - 1 - e.first);
            o << "    " << guard << "{\n    double pk0 = 0.0";
            for (int kr = 1; kr < K; ++kr) o << ", pk" << kr << " = 0.0";
            o << ";\n";
            for (int rho = 0; rho < (1 << R); ++rho) {
                int kr = 0;
                for (size_t e = 0; e < regbits.size(); ++e) kr |= ((rho >> regbits[e].second) & 1) << e;
                o << "    pk" << kr << " = fma(v" << rho << ".x, v" << rho << ".x, fma(v" << rho << ".y, v" << rho
                  << ".y, pk" << kr << "));\n";
            }
            o << "    const u64 pib = base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
            o << "    const unsigned kt = 0u";
            for (int i = 0; i < M; ++i)
                if (!((regmask >> (M - 1 - i)) & 1))
                    o << " | ((unsigned)((pib >> " << (*probe)[i] << ") & 1ull) << " << (M - 1 - i) << ")";
            o << ";\n";
            for (int kr = 0; kr < K; ++kr) {
                unsigned KR = 0;
                for (size_t e = 0; e < regbits.size(); ++e)
                    if ((kr >> e) & 1) KR |= 1u << (M - 1 - regbits[e].first);
                for (int b = 0; b < B; ++b)
                    if (((unsigned)b & regmask) == KR)
                        o << "    pb" << b << " += kt == " << ((unsigned)b & ~regmask) << "u ? pk" << kr << " : 0.0;\n";
            }
            o << "    }\n";
        }
        if (last && staged_out) {
            // each thread overwrites only the slots it read this stage; a
            // first stage read global memory, and the previous tile's last
            // stage may still read the shared tile
            if (first && !staged_in) o << barrier;
            for (int rho = 0; rho < (1 << R); ++rho) o << "    tile[tsw ^ " << c[rho] << "u] = v" << rho << ";\n";
            o << thread_end << barrier << thread_loop << "    " << guard << "{\n";
            o << "    const unsigned tsc = " << smap.tid_expr(natural) << ";\n";
            if (xmask) {
                o << "    const u64 xib = base + (" << deposit_expr("tid", lowq, true) << ");\n";
                for (int k = 0; k < (1 << R); ++k)
                    o << "    " << (stream_out ? "stcs2" : "stwb2") << "(QSV_XDST(xib + " << goffc[k] << "ull), tile[tsc ^ "
                      << cc[k] << "u]);\n";
            } else {
            o << "    double2 *gpc = psi + base + (" << deposit_expr("tid", lowq, true) << ");\n";
            for (int k = 0; k < (1 << R); ++k)
                o << "    " << (stream_out ? "stcs2" : "stwb2") << "(gpc + " << goffc[k] << "ull, tile[tsc ^ " << cc[k]
                  << "u]);\n";
            }
            o << "    }\n" << thread_end;
            if (tma) {
                o << barrier << "    fence_proxy_async();\n";
                tma_issue(next_group);
            }
            o << "    }\n";
        } else if (last) {
            // evict-first stores when the data leaves for HBM; write-back (L2
            // resident) stores between the inner passes of a super-pass
            o << "    " << guard << "{\n";
            if (xmask) o << "    const u64 xib = base + (" << deposit_expr("tid", nonreg_q, true) << ");\n";
            for (int rho = 0; rho < (1 << R); ++rho)
                o << "    " << (stream_out ? "stcs2" : "stwb2") << (xmask ? "(QSV_XDST(xib + " : "(gp + ") << goff[rho]
                  << (xmask ? "ull), v" : "ull, v") << rho << ");\n";
            o << "    }\n";
            o << thread_end << "    }\n";
        } else {
            // the previous tile's last stage may still read the shared tile
            if (first && !staged_in) o << barrier;
            for (int rho = 0; rho < (1 << R); ++rho) o << "    tile[tsw ^ " << c[rho] << "u] = v" << rho << ";\n";
            o << thread_end << barrier << "    }\n";
        }
    }
    o << "  }\n  }\n";
    if (scale_out) *scale_out = sigma;
    return fp64;
}

constexpr double kThreeCtaMinFp64 = 60.0;
constexpr long kStaggerCycles = 2500;

std::string kernel_head(const Plan &P, int m, bool host, const char *name, const char *params,
                        double fp64_per_amp = 0, int gang = 1, int r = 0, long stagger = 0) {
    std::ostringstream o;
    if (r <= 0) r = P.r;
    const int T = 1 << (m - r);
    if (host) {
        o << kHostPrelude << "extern \"C\" void " << name << "_host(" << params << ") {\n";
        o << "  static double2 tile[" << (1 << m) << "];\n";
    } else {
        o << kPrelude << kGridSync;
        // Resident CTAs per SM: two by default; one when the CTA has 512
        // threads or its tile takes more than half of the 228 KB of shared
        // memory (capping registers for a CTA that cannot be resident only
        // spills); three for compute-bound passes of 128-thread CTAs with
        // tiles <= 64 KB (registers capped at 168: a few bytes of spill, 12
        // warps/SM; measured on C2: passes >= ~60 FP64/amp gain 5-7 %, lighter
        // passes lose up to 20 %).  QSV_JIT_MIN_BLOCKS overrides.
        const char *mb = std::getenv("QSV_JIT_MIN_BLOCKS");
        const bool one = T >= 512 || (16u << m) > (113u << 10);
        const bool three = !one && T <= 128 && (16u << m) <= (64u << 10) && fp64_per_amp >= kThreeCtaMinFp64;
        if (gang > 1) {
            o << "// gang=" << gang << "\n";
            o << "extern \"C\" __global__ void __launch_bounds__(" << gang * T << ", 1) " << name << "(" << params
              << ") {\n";
            o << "  extern __shared__ double2 smem[];\n";
            o << "  const unsigned tid = threadIdx.x & " << (T - 1) << "u, sub = threadIdx.x >> " << (m - r) << ";\n";
            o << "  double2 *tile = smem + ((size_t)sub << " << m << ");\n";
        } else {
        o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", "
          << (mb ? std::atoi(mb) : (one ? 1 : three ? 3 : 2)) << ") "
          << name << "(" << params << ") {\n";
        o << "  extern __shared__ double2 smem[];\n";
        o << "  double2 *tile = smem;\n";
        o << "  const unsigned tid = threadIdx.x;\n";
        // The CTAs of the first residency wave that share an SM start out of phase: slot 1
        // (blockIdx / #SMs) spins for `stagger` cycles first, and with one CTA per tile a
        // successor inherits its slot's phase.  A pass launched on an idle GPU (the first
        // pass after an upload or copy) otherwise runs its two CTAs per SM in lock step -
        // both load, both compute, both store - and overlaps nothing: QFT n = 30 first pass
        // 8.81-8.87 -> 7.66-7.92 ms (2500-14000 cycles alike); passes that follow another
        // pass start staggered by its tail and gain nothing (C2 neutral).
        // QSV_JIT_STAGGER=<cycles> forces it on every pass (0: off).
        if (stagger > 0)
            o << "  { unsigned nsm; asm volatile(\"mov.u32 %0, %%nsmid;\" : \"=r\"(nsm));\n"
              << "    if (blockIdx.x / nsm == 1u) { const long long t0 = clock64();\n"
              << "      while (clock64() - t0 < " << stagger << "ll) { } } }\n";
        }
    }
    return o.str();
}

}  // namespace

constexpr double kPrefetchMinFp64 = 55.0;

// The uniform scale each pass's kernel finds the state stored with (chained
// through dry runs of the generator: pass i's last stage decides pass i+1's).
// FP64 instructions per amplitude of every pass (the specialiser's cost model) from
// one dry emission per pass, filling the uniform-scale chain on the way (the same
// emission pass_scales runs; jit_source's own dry run gives the same numbers).
std::vector<double> pass_costs(const Plan &P) {
    const size_t np = P.passes.size();
    std::vector<double> sc(np + 1, 1.0), cost(np, 0.0);
    std::ostringstream *saved = g_decls;
    for (size_t pi = 0; pi < np; ++pi) {
        // with a declaration sink, as jit_source emits: per-thread factor tables replace
        // computed products (fewer FP64), the scale chain is unaffected
        std::ostringstream dry, decls;
        g_decls = &decls;
        g_decl_id = 0;
        const double f = emit_tile_loop(
            dry, P, (int)pi, false, "n", [](const std::string &) { return std::string("0"); }, true, false, false,
            sc[pi], pi + 1 == np, &sc[pi + 1]);
        cost[pi] = f / (double)(1 << pass_r(P, (int)pi));
    }
    g_decls = saved;
    return cost;
}

const std::vector<double> &pass_scales(const Plan &P) {
    const size_t np = P.passes.size();
    if (P.jit_scale_in.size() != np + 1) {
        std::vector<double> sc(np + 1, 1.0);
        for (size_t pi = 0; pi < np; ++pi) {
            std::ostringstream dry;
            emit_tile_loop(
                dry, P, (int)pi, false, "n", [](const std::string &) { return std::string("0"); }, true, false, false,
                sc[pi], pi + 1 == np, &sc[pi + 1]);
        }
        P.jit_scale_in = sc;
    }
    return P.jit_scale_in;
}

std::string jit_source(const Plan &P, int pi, bool host, double *fp64_per_amp, uint64_t xmask,
                       const std::vector<int> *probe) {
    if (host) probe = nullptr;
    const DevPass &dp = P.passes[pi];
    std::ostringstream o;
    o << "// libqsv specialised pass kernel: n=" << P.n << " m=" << dp.m << " R=" << pass_r(P, pi) << " pass=" << pi << "\n";
    std::vector<int> ext;
    for (int q = 0; q < P.n; ++q)
        if (!((dp.tile_mask >> q) & 1)) ext.push_back(q);
    auto base_of = [&](const std::string &t) { return deposit_expr(t, ext, true); };
    const double sc = pass_scales(P)[pi];
    const bool final_pass = pi + 1 == (int)P.passes.size();
    // per-thread factor tables land in `decls` (inserted before the kernel)
    std::ostringstream decls;
    std::ostringstream *saved_decls = g_decls;
    g_decls = &decls;
    g_decl_id = 0;
    // FP64 work per amplitude (dry run) decides the compute-bound tuning
    double cost;
    {
        std::ostringstream dry;
        cost = emit_tile_loop(dry, P, pi, host, "n_tiles", base_of, true, false, false, sc, final_pass) /
               (double)(1 << pass_r(P, pi));
    }
    decls.str("");
    g_decl_id = 0;
    // QSV_JIT_GANG=G: compute-bound passes run G tiles per CTA in lock step
    // (one CTA per SM) instead of independent CTAs; QSV_JIT_TMA=1: their
    // tiles arrive by TMA bulk copies during the previous tile's last stage
    int gang = 1;
    bool tma = false;
    if (!host) {
        static const int env_gang = std::getenv("QSV_JIT_GANG") ? std::atoi(std::getenv("QSV_JIT_GANG")) : 1;
        const int T = 1 << (dp.m - pass_r(P, pi));
        static const double gang_min =
            std::getenv("QSV_JIT_GANG_MIN") ? std::atof(std::getenv("QSV_JIT_GANG_MIN")) : kThreeCtaMinFp64;
        if (env_gang > 1 && cost >= gang_min && env_gang * T <= 1024 &&
            ((size_t)env_gang << (dp.m + 4)) <= ((size_t)227 << 10))
            gang = env_gang;
        static const bool env_tma = std::getenv("QSV_JIT_TMA") && std::atoi(std::getenv("QSV_JIT_TMA")) != 0;
        tma = env_tma && cost >= gang_min;
    }
    if (xmask) {
        gang = 1;
        o << "struct XDst { unsigned long long p[8]; unsigned long long self; };\n";
        o << "#define QSV_XDST(ix) ((double2 *)xd.p[";
        int i = 0;
        for (int q = 0; q < 64; ++q)
            if ((xmask >> q) & 1) o << (i ? " | " : "") << "((((ix) >> " << q << ") & 1ull) << " << i++ << ")";
        o << "] + (((ix) & ~" << xmask << "ull) | xd.self))\n";
    }
    std::string params = host ? "double2 *__restrict__ psi, u64 n_tiles" : "double2 *__restrict__ psi, u64 n_tiles, u64 basis";
    if (P.product && pi == 0 && !xmask) params += ", const double2 *__restrict__ ptab";
    if (xmask) params += ", XDst xd";
    if (probe) {
        gang = 1;
        params += ", double *__restrict__ probe_out";
    }
    // first pass of a large state that reads its input: see kernel_head (stagger)
    long stagger = (pi == 0 && !P.product && !xmask && !probe && P.n - dp.m >= 16) ? kStaggerCycles : 0;
    if (const char *sg = std::getenv("QSV_JIT_STAGGER")) stagger = std::atol(sg);
    o << kernel_head(P, dp.m, host, "qsv_pass", params.c_str(), cost, gang, pass_r(P, pi), stagger);
    const int PB = probe ? 1 << probe->size() : 0;
    if (probe) {
        o << "  // probe-out pass: qubits";
        for (int q : *probe) o << " " << q;
        o << "\n  double pb0 = 0.0";
        for (int b = 1; b < PB; ++b) o << ", pb" << b << " = 0.0";
        o << ";\n";
    }
    // L2 prefetch of the next tile pays only in compute-bound passes (measured
    // per pass on C2: it slows memory-bound passes by ~0.3 ms and speeds up
    // passes above ~55 FP64/amplitude); QSV_JIT_PREFETCH=0/1 forces it
    // With one CTA per tile the prefetch targets the tile a CTA launched one
    // residency wave later takes (gridDim_prefetch_distance): measured a gain
    // for the r = 4 passes (two 8-warp CTAs per SM; C2 59.0 -> 57.6 ms) and a
    // loss for the r = 5 ones (QFT 41.6 -> 45.8 ms)
    const char *e = std::getenv("QSV_JIT_PREFETCH");
    const bool prefetch = e ? std::atoi(e) != 0
                            : (jit_per_tile_grid() ? pass_r(P, pi) == 4 : cost >= kPrefetchMinFp64);
    const double f = emit_tile_loop(o, P, pi, host, "n_tiles", base_of, true, !host && !jit_double_buffer(), prefetch,
                                    sc, final_pass, nullptr, gang, xmask, tma && !xmask && !probe, probe);
    if (fp64_per_amp) *fp64_per_amp = f / (double)(1 << pass_r(P, pi));
    g_decls = saved_decls;
    if (probe) {
        // per-CTA partials in a fixed order (warp tree, then warps in order)
        o << "  {\n  __shared__ double qsv_pred[" << PB << "][32];\n";
        o << "  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;\n";
        for (int b = 0; b < PB; ++b)
            o << "  { double s = pb" << b << "; for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);"
              << " if (lane == 0) qsv_pred[" << b << "][wid] = s; }\n";
        o << "  __syncthreads();\n";
        o << "  if (threadIdx.x < " << PB << "u) { double s = 0.0;"
          << " for (unsigned w = 0; w < (blockDim.x + 31u) / 32u; ++w) s += qsv_pred[threadIdx.x][w];"
          << " probe_out[(size_t)blockIdx.x * " << PB << "u + threadIdx.x] = s; }\n  }\n";
    }
    o << "}\n";
    std::string src = o.str();
    const std::string d = decls.str();
    if (!d.empty()) {
        const size_t at = src.find("extern \"C\"");
        src.insert(at == std::string::npos ? 0 : at, d);
    }
    return src;
}

// Register qubits per pass.  32 amplitudes per thread (r = 5) needs the
// fewest stages, but its straight-line code is twice as long per thread as
// r = 4 and the three CTAs per SM then stall on instruction fetch; with one CTA
// per tile, r = 4 measured faster on every C2 pass whose FP64 work it does not
// raise (7.0-9.1 vs 7.9-9.5 ms, same FP64/amp), while QFT passes, whose extra
// stages cost FP64 at r = 4 (+27-45 %), stay faster at r = 5.  Both
// stagings of the same passes are generated and each pass takes r = 4 when its
// FP64 work per amplitude is within kR4CostRatio of the r = 5 staging.
constexpr double kR4CostRatio = 1.10;
constexpr double kR4LightFp64 = 65.0;

Plan build_plan_auto(const std::vector<GateRec> &recs, int n, int m, int r, int L, int s, bool auto_r) {
    Plan P5 = build_plan(recs, n, m, r, L, s);
    static const bool off = std::getenv("QSV_MIXED_R") && std::atoi(std::getenv("QSV_MIXED_R")) == 0;
    if (off || !auto_r || r != 5 || P5.s != P5.m || P5.passes.empty()) return P5;
    // the same tiles and gate sets re-staged with r = 4 (no second tile planning)
    Plan P4 = rebuild_with_pass_r(P5, std::vector<int>(P5.passes.size(), 4));
    const int np = (int)P5.passes.size();
    std::vector<int> rs(np, 5);
    int n4 = 0;
    // both stagings' cost models at once (one dry emission per pass each)
    std::vector<double> c4;
    std::thread t4([&] { c4 = pass_costs(P4); });
    const std::vector<double> c5 = pass_costs(P5);
    t4.join();
    for (int i = 0; i < np; ++i) {
        // light passes (memory- or latency-bound) also take r = 4 when its FP64 work stays
        // below the HBM floor: the 8-warp r = 5 CTAs hide less latency (QFT passes 1 and 3,
        // 59 vs 48 FP64/amp: 42.3 -> 41.4 ms); the last pass keeps r = 5 (measured slower at
        // r = 4: it flushes the deferred scale)
        // ... unless its tile spreads over 2^8 or more 2 MB pages (8+ tile qubits at positions
        // >= 17): such a pass is bound by the latency of its scattered lines, which 32 loads per
        // thread in flight cover better than 16 (QFT's first pass, tile 0-2 + 21-29: 8.4 ms at
        // r = 5, 9.9 ms at r = 4, though r = 4 needs no more FP64 there)
        int high = 0;
        for (int q = 17; q < n; ++q) high += (int)((P5.passes[i].tile_mask >> q) & 1);
        const bool light = c4[i] <= kR4LightFp64 && i + 1 < np && high < 8;
        if (c4[i] <= kR4CostRatio * c5[i] || light) {
            rs[i] = 4;
            ++n4;
        }
    }
    // QSV_MIXED_R_PATTERN (tests): e.g. "45" forces r = 4, 5, 4, 5, ... per pass
    if (const char *pat = std::getenv("QSV_MIXED_R_PATTERN")) {
        const std::string ps(pat);
        if (!ps.empty()) {
            n4 = 0;
            for (int i = 0; i < np; ++i) n4 += (rs[i] = ps[i % ps.size()] == '4' ? 4 : 5) == 4;
        }
    }
    if (n4 == 0) return P5;
    if (n4 == np) return P4;
    return rebuild_with_pass_r(P5, rs);
}

Plan build_plan_start(const std::vector<GateRec> &recs, int n, int m, int r, int L, int s, bool auto_r,
                      bool product) {
    if (product) {
        std::vector<GateRec> kept;
        std::vector<cd> prefix;
        if (split_product_prefix(recs, n, kept, prefix) > 0 && !kept.empty()) {
            Plan P = build_plan_auto(kept, n, m, r, L, s, auto_r);
            if (P.s == P.m && !P.passes.empty()) {  // flat plans only (no L2 super-passes)
                P.product = true;
                P.prefix = std::move(prefix);
                P.gates = (int64_t)recs.size();
                return P;
            }
        }
    }
    return build_plan_auto(recs, n, m, r, L, s, auto_r);
}

std::vector<int> product_regs(const Plan &P) {
    const DevPass &dp = P.passes[0];
    const DevStage &st = P.stages[dp.stage_begin];
    std::vector<int> regs(pass_r(P, 0));
    for (int k = 0; k < (int)regs.size(); ++k) regs[k] = dp.tq[st.rb[k]];
    return regs;
}

int super_batch(const Plan &P) {
    // super-tiles processed together: keep the batch within the L2 budget
    // (default 64 MB of the 126 MB L2; QSV_L2_BYTES overrides)
    const char *env = std::getenv("QSV_L2_BYTES");
    const size_t budget = env ? (size_t)std::atoll(env) : ((size_t)64 << 20);
    const int s = P.s, n = P.n;
    int b = 0;
    while (b < n - s && ((size_t)16 << (s + b + 1)) <= budget) ++b;
    return b;  // log2 of the batch size
}

std::string jit_super_source(const Plan &P, int si, bool host) {
    const SuperPass &sp = P.supers[si];
    const int n = P.n, s = popc64(sp.mask), m = P.m, lb = super_batch(P);
    std::ostringstream o;
    o << "// libqsv super-pass kernel: n=" << n << " s=" << s << " m=" << m << " inner passes "
      << sp.pass_begin << ".." << sp.pass_end - 1 << " batch=2^" << lb << "\n";
    std::vector<int> outside;
    for (int q = 0; q < n; ++q)
        if (!((sp.mask >> q) & 1)) outside.push_back(q);
    o << kernel_head(P, m, host, "qsv_super", "double2 *__restrict__ psi, u64 n_batches, unsigned *__restrict__ bar");
    if (!host) o << "  unsigned gen = 0;\n";
    o << "  for (u64 batch = 0; batch < n_batches; ++batch) {\n";
    for (int pi = sp.pass_begin; pi < sp.pass_end; ++pi) {
        const DevPass &dp = P.passes[pi];
        std::vector<int> inner;  // super-tile qubits outside this pass's tile
        for (int q = 0; q < n; ++q)
            if (((sp.mask >> q) & 1) && !((dp.tile_mask >> q) & 1)) inner.push_back(q);
        const int ib = (int)inner.size();  // = s - m
        const std::string ntiles = "(1ull << " + std::to_string(ib + lb) + ")";
        emit_tile_loop(
            o, P, pi, host, ntiles,
            [&, ib](const std::string &t) {
                const std::string lowpart = "(" + t + " & ((1ull << " + std::to_string(ib) + ") - 1ull))";
                const std::string stile =
                    "((batch << " + std::to_string(lb) + ") + (" + t + " >> " + std::to_string(ib) + "))";
                return "(" + deposit_expr(lowpart, inner, true) + ") | (" + deposit_expr(stile, outside, true) + ")";
            },
            pi + 1 == sp.pass_end, false, false, pass_scales(P)[pi], pi + 1 == (int)P.passes.size());
        if (!host) o << "  grid_sync(bar, gen);\n";
    }
    o << "  }\n}\n";
    return o.str();
}

// spill stores reported by ptxas -v in an NVRTC log ("N bytes spill stores")
size_t spill_bytes(const std::string &log) {
    size_t total = 0;
    for (size_t at = log.find("bytes spill stores"); at != std::string::npos; at = log.find("bytes spill stores", at + 1)) {
        size_t b = at;
        while (b > 0 && log[b - 1] == ' ') --b;
        size_t e = b;
        while (b > 0 && std::isdigit((unsigned char)log[b - 1])) --b;
        if (b < e) total += std::stoul(log.substr(b, e - b));
    }
    return total;
}
constexpr size_t kMaxSpillBytes = 128;
// QSV_JIT_MAX_SPILL (diagnostic): spill bytes a three-CTA kernel may keep before it is
// recompiled for two CTAs per SM
size_t max_spill_bytes() {
    static const size_t v = std::getenv("QSV_JIT_MAX_SPILL") ? (size_t)std::atol(std::getenv("QSV_JIT_MAX_SPILL"))
                                                             : kMaxSpillBytes;
    return v;
}

// QSV_NVRTC_FAST=min|mid (diagnostic): NVRTC --Ofast-compile level (cuts front-end time,
// slightly different code); part of the disk-cache key
const std::string &nvrtc_fast_compile() {
    static const std::string v = [] {
        const char *e = std::getenv("QSV_NVRTC_FAST");
        return (e && *e) ? std::string("--Ofast-compile=") + e : std::string();
    }();
    return v;
}

std::string jit_compile_cubin(const std::string &src, std::string &log) {
    Nvrtc &api = nvrtc();
    if (!api.ok) {
        log = api.why;
        return {};
    }
    nvrtcProgram prog;
    if (api.CreateProgram(&prog, src.c_str(), "qsv_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        log = "nvrtcCreateProgram failed";
        return {};
    }
    std::vector<const char *> opts = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                                      "--extra-device-vectorization", "--ptxas-options=-v", "-diag-suppress=177"};
    const std::string &fast = nvrtc_fast_compile();
    if (!fast.empty()) opts.push_back(fast.c_str());
    const nvrtcResult rc = api.CompileProgram(prog, (int)opts.size(), opts.data());
    size_t ls = 0;
    api.GetProgramLogSize(prog, &ls);
    log.assign(ls, '\0');
    if (ls) api.GetProgramLog(prog, log.data());
    std::string cubin;
    if (rc == NVRTC_SUCCESS) {
        size_t cs = 0;
        api.GetCUBINSize(prog, &cs);
        cubin.assign(cs, '\0');
        api.GetCUBIN(prog, cubin.data());
    }
    api.DestroyProgram(&prog);
    return cubin;
}

namespace {

// On-disk cubin cache: a fresh process (the CLI, a new job) loads the
// specialised kernels of a circuit it has seen before instead of recompiling
// them with NVRTC (C2: ~1.4 s of first-call latency).  Key: FNV-1a of the
// kernel source (which embeds the whole pass) + compile options + NVRTC
// version.  $QSV_CACHE_DIR (empty or "0": off), else $XDG_CACHE_HOME/qsv,
// else $HOME/.cache/qsv.  Files are written to a temporary name and renamed.
std::string disk_cache_path(const std::string &src) {
    static const std::string dir = [] {
        const char *e = std::getenv("QSV_CACHE_DIR");
        if (e) return (std::string(e) == "0") ? std::string() : std::string(e);
        if (const char *x = std::getenv("XDG_CACHE_HOME")) return std::string(x) + "/qsv";
        if (const char *h = std::getenv("HOME")) return std::string(h) + "/.cache/qsv";
        return std::string();
    }();
    if (dir.empty()) return {};
    static const std::string salt = [] {
        int major = 0, minor = 0;
        Nvrtc &api = nvrtc();
        if (api.ok && api.Version) api.Version(&major, &minor);
        return "sm_100a|lineinfo|xdv|nvrtc" + std::to_string(major) + "." + std::to_string(minor) + nvrtc_fast_compile();
    }();
    uint64_t h = 1469598103934665603ull;
    for (const std::string *part : {&salt, &src})
        for (unsigned char c : *part) {
            h ^= c;
            h *= 1099511628211ull;
        }
    char name[64];
    std::snprintf(name, sizeof(name), "/%016" PRIx64 "-%zu.cubin", h, src.size());
    return dir + name;
}

bool disk_cache_load(const std::string &path, std::string &cubin) {
    if (path.empty()) return false;
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    std::string data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (data.size() < 16) return false;
    cubin.swap(data);
    return true;
}

void disk_cache_store(const std::string &path, const std::string &cubin) {
    if (path.empty() || cubin.empty()) return;
    const size_t slash = path.rfind('/');
    std::string cmd_dir = path.substr(0, slash);
    // mkdir -p
    for (size_t at = 1; at <= cmd_dir.size(); ++at)
        if (at == cmd_dir.size() || cmd_dir[at] == '/') {
            const std::string d = cmd_dir.substr(0, at);
            mkdir(d.c_str(), 0755);
        }
    const std::string tmp = path + ".tmp" + std::to_string((long)getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f.write(cubin.data(), (std::streamsize)cubin.size());
        if (!f) return;
    }
    std::rename(tmp.c_str(), path.c_str());
}

}  // namespace

namespace {

struct CacheEntry {
    CUfunction fn = nullptr;
    int grid = 0;  // persistent grid: resident CTAs per SM x SMs
    int gang = 1;  // tiles per CTA
};

// tiles per CTA of a generated pass kernel (the "// gang=G" marker)
int source_gang(const std::string &src) {
    const size_t at = src.find("// gang=");
    return at == std::string::npos ? 1 : std::atoi(src.c_str() + at + 8);
}

std::mutex g_cache_mu;
std::map<std::pair<int, std::string>, CacheEntry> g_cache;  // (device, source) -> kernel

}  // namespace

// a compile unit: one generated kernel
struct Unit {
    std::string src, name, cubin, log;
    int m = 0;
    bool super = false;
    int index = 0;  // pass or super-pass index
};

bool use_supers(const Plan &P) { return P.s > P.m; }

void jit_choose_supers(Plan &P, int sms) {
    P.super_use.assign(P.supers.size(), 0);
    if (!use_supers(P)) return;
    // B200 sm_100a: 64 FP64 lanes/SM at ~1.9 GHz, ~60% sustained on this
    // kernel shape; HBM ~6.0 TB/s achieved.  The persistent super kernel adds
    // ~20% on its compute (tails + grid barriers, measured).
    const double amps = std::ldexp(1.0, P.n);
    const double fp64_rate = (double)sms * 64.0 * 1.9e9 * 0.6;
    const double t_hbm = 32.0 * amps / 6.0e12;
    for (size_t si = 0; si < P.supers.size(); ++si) {
        const SuperPass &sp = P.supers[si];
        if (sp.pass_end - sp.pass_begin < 2) continue;
        double flat = 0, comp = 0;
        for (int i = sp.pass_begin; i < sp.pass_end; ++i) {
            double f = 0;
            jit_source(P, i, false, &f);
            const double t = amps * f / fp64_rate;
            flat += std::max(t_hbm, t);
            comp += t;
        }
        P.super_use[si] = std::max(t_hbm, 1.2 * comp) < flat ? 1 : 0;
    }
}

namespace {

// One NVRTC compile (disk cache first); a three-CTA register cap that spills
// (accumulator-heavy passes, e.g. QFT: 1.2 KB of local memory, +20 % time) is
// recompiled for two CTAs per SM (the cache key stays the original source).
void compile_unit(Unit &u) {
    const std::string path = disk_cache_path(u.src);
    if (disk_cache_load(path, u.cubin)) return;
    u.cubin = jit_compile_cubin(u.src, u.log);
    const std::string three = "__launch_bounds__(128, 3)";
    const size_t at = u.src.find(three);
    if (!u.cubin.empty() && at != std::string::npos && spill_bytes(u.log) > max_spill_bytes()) {
        std::string src2 = u.src;
        src2.replace(at, three.size(), "__launch_bounds__(128, 2)");
        std::string log2;
        std::string cubin2 = jit_compile_cubin(src2, log2);
        if (!cubin2.empty()) u.cubin.swap(cubin2);
    }
    disk_cache_store(path, u.cubin);
}

// ---- asynchronous compilation (the cold call of a new circuit) ----------------
// Units submitted here compile on a small pool of host threads while the caller
// runs the passes that are not ready yet on the interpreted kernel
// (execute_plan_mixed in qsv_api.cu).  A blocking jit_prepare that meets a unit in
// flight waits for it instead of compiling it again.  The pool and its maps are
// never destroyed (threads may outlive static destruction); an atexit hook waits
// for compiles in flight so NVRTC is not torn down under a running compile.
struct AsyncUnit {
    Unit u;
    bool done = false;
};
struct AsyncPool {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::shared_ptr<AsyncUnit>> queue;
    std::map<std::string, std::shared_ptr<AsyncUnit>> by_src;  // submitted, not yet loaded
    int active = 0;
    bool started = false;
};
AsyncPool &apool() {
    static AsyncPool *p = new AsyncPool();
    return *p;
}
void async_worker() {
    AsyncPool &A = apool();
    for (;;) {
        std::shared_ptr<AsyncUnit> job;
        {
            std::unique_lock<std::mutex> lk(A.mu);
            A.cv.wait(lk, [&] { return !A.queue.empty(); });
            job = A.queue.front();
            A.queue.pop_front();
            ++A.active;
        }
        compile_unit(job->u);
        {
            std::lock_guard<std::mutex> lk(A.mu);
            job->done = true;
            --A.active;
        }
        A.cv.notify_all();
    }
}
void async_drain_at_exit() {
    AsyncPool &A = apool();
    std::unique_lock<std::mutex> lk(A.mu);
    A.queue.clear();
    A.cv.wait(lk, [&] { return A.active == 0; });
}
std::shared_ptr<AsyncUnit> async_submit(const Unit &u) {
    AsyncPool &A = apool();
    std::lock_guard<std::mutex> lk(A.mu);
    auto it = A.by_src.find(u.src);
    if (it != A.by_src.end()) return it->second;
    if (!A.started) {
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        for (unsigned t = 0; t < hw; ++t) std::thread(async_worker).detach();
        std::atexit(async_drain_at_exit);
        A.started = true;
    }
    auto job = std::make_shared<AsyncUnit>();
    job->u = u;
    A.by_src[u.src] = job;
    A.queue.push_back(job);
    A.cv.notify_all();
    return job;
}
// the finished async unit for `src` (removed from the pool), waiting for it when
// `wait`; nullptr when none was submitted (or it is still running and !wait)
std::shared_ptr<AsyncUnit> async_take(const std::string &src, bool wait) {
    AsyncPool &A = apool();
    std::unique_lock<std::mutex> lk(A.mu);
    auto it = A.by_src.find(src);
    if (it == A.by_src.end()) return nullptr;
    auto job = it->second;
    if (!job->done) {
        if (!wait) return nullptr;
        A.cv.wait(lk, [&] { return job->done; });
    }
    A.by_src.erase(src);
    return job;
}

// Loads a compiled unit for `device` (module, dynamic smem, occupancy) into the
// in-process cache.  Caller holds g_cache_mu.
int load_unit(const Plan &P, Unit &u, int device, CacheEntry &out, std::string &err) {
    Driver &drv = driver();
    if (u.cubin.empty()) {
        err = "NVRTC failed for " + u.name + " " + std::to_string(u.index) + ": " + u.log;
        return QSV_E_DEVICE;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    CUmodule mod;
    CUfunction fn;
    CUresult r = drv.ModuleLoadData(&mod, u.cubin.data());
    if (r == CUDA_SUCCESS) r = drv.ModuleGetFunction(&fn, mod, u.name.c_str());
    const int gang = u.super ? 1 : source_gang(u.src);
    const int smem = gang * (int)((size_t)(jit_double_buffer() ? 32 : 16) << u.m);  // tile buffer(s)
    if (r == CUDA_SUCCESS) r = drv.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
    int per_sm = 0;
    if (r == CUDA_SUCCESS)
        r = drv.OccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn,
                                                          gang << (u.m - (u.super ? P.r : pass_r(P, u.index))),
                                                          (size_t)smem);
    if (r != CUDA_SUCCESS || per_sm < 1) {
        const char *s = nullptr;
        if (r != CUDA_SUCCESS) drv.GetErrorString(r, &s);
        err = std::string("loading specialised kernel: ") + (s ? s : "zero occupancy");
        return QSV_E_DEVICE;
    }
    // QSV_JIT_CTAS_PER_SM (diagnostic): cap the persistent grid's CTAs per SM
    if (const char *c = std::getenv("QSV_JIT_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(c)));
    out = CacheEntry{fn, per_sm * sms, gang};
    g_cache[{device, u.src}] = out;
    return QSV_OK;
}

}  // namespace

// The pass kernels' sources, generated on up to 16 host threads (the uniform-scale
// chain is filled first; jit_source is then read-only on the plan).
std::vector<std::string> pass_sources(const Plan &P) {
    const size_t np = P.passes.size();
    std::vector<std::string> src(np);
    pass_scales(P);
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t k; (k = next.fetch_add(1)) < np;) src[k] = jit_source(P, (int)k);
    };
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < std::min<size_t>(hw, np); ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    return src;
}

int jit_prepare(Plan &P, int device, std::string &err) {
    if (P.jit_device == device && P.jit_funcs.size() == P.passes.size()) return QSV_OK;
    if (!jit_available(err)) return QSV_E_DEVICE;
    std::vector<Unit> units;
    {
        std::vector<std::string> src = P.jit_part_src.size() == P.passes.size() ? P.jit_part_src : pass_sources(P);
        for (size_t i = 0; i < P.passes.size(); ++i)
            units.push_back(Unit{std::move(src[i]), "qsv_pass", {}, {}, P.passes[i].m, false, (int)i});
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    jit_choose_supers(P, sms);
    for (size_t si = 0; si < P.supers.size(); ++si)
        if (P.super_use[si])
            units.push_back(Unit{jit_super_source(P, (int)si), "qsv_super", {}, {}, P.m, true, (int)si});
    std::vector<CacheEntry> found(units.size());
    std::vector<int> todo;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < units.size(); ++i) {
            auto it = g_cache.find({device, units[i].src});
            if (it != g_cache.end()) found[i] = it->second;
            else todo.push_back((int)i);
        }
    }
    // units compiling asynchronously (an earlier cold call) are awaited, the others are
    // compiled here concurrently (independent NVRTC programs)
    std::vector<int> local;
    for (int i : todo) {
        if (auto job = async_take(units[i].src, true)) units[i].cubin.swap(job->u.cubin), units[i].log.swap(job->u.log);
        else local.push_back(i);
    }
    {
        std::vector<std::thread> pool;
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::atomic<size_t> next{0};
        for (unsigned t = 0; t < std::min<size_t>(hw, local.size()); ++t)
            pool.emplace_back([&] {
                for (size_t k; (k = next.fetch_add(1)) < local.size();) compile_unit(units[local[k]]);
            });
        for (auto &th : pool) th.join();
    }
    cudaSetDevice(device);
    cudaFree(nullptr);  // make the primary context current for the driver API
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (int i : todo) {
        const int rc = load_unit(P, units[i], device, found[i], err);
        if (rc) return rc;
    }
    P.jit_funcs.assign(P.passes.size(), nullptr);
    P.jit_grids.assign(P.passes.size(), 0);
    P.jit_gangs.assign(P.passes.size(), 1);
    P.jit_super_funcs.assign(P.supers.size(), nullptr);
    P.jit_super_grids.assign(P.supers.size(), 0);
    for (size_t i = 0; i < units.size(); ++i) {
        if (units[i].super) {
            P.jit_super_funcs[units[i].index] = found[i].fn;
            P.jit_super_grids[units[i].index] = found[i].grid;
        } else {
            P.jit_funcs[units[i].index] = found[i].fn;
            P.jit_grids[units[i].index] = found[i].grid;
            P.jit_gangs[units[i].index] = found[i].gang;
        }
    }
    P.jit_device = device;
    return QSV_OK;
}

void jit_wait_async() {
    AsyncPool &A = apool();
    std::unique_lock<std::mutex> lk(A.mu);
    A.cv.wait(lk, [&] { return A.queue.empty() && A.active == 0; });
}

bool jit_ready(const Plan &P, int device) { return P.jit_device == device && P.jit_funcs.size() == P.passes.size(); }

int jit_start_async(Plan &P, int device, std::string &err) {
    if (jit_ready(P, device)) return QSV_OK;
    if (!jit_available(err)) return QSV_E_DEVICE;
    if (P.jit_part_src.size() != P.passes.size()) {
        P.jit_part_src = pass_sources(P);
        P.jit_part_funcs.assign(P.passes.size(), nullptr);
        P.jit_part_grids.assign(P.passes.size(), 0);
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    // last passes first: the first ones run interpreted on a cold call anyway, the
    // late (often light, quick to compile) ones may be ready when the GPU gets there
    for (size_t i = P.passes.size(); i-- > 0;) {
        if (P.jit_part_funcs[i]) continue;
        auto it = g_cache.find({device, P.jit_part_src[i]});
        if (it != g_cache.end()) {
            P.jit_part_funcs[i] = it->second.fn;
            P.jit_part_grids[i] = it->second.grid;
            continue;
        }
        async_submit(Unit{P.jit_part_src[i], "qsv_pass", {}, {}, P.passes[i].m, false, (int)i});
    }
    return QSV_OK;
}

int jit_try_pass(Plan &P, int pass, int device, bool *ready, std::string &err) {
    *ready = false;
    if (jit_ready(P, device)) {
        *ready = true;
        return QSV_OK;
    }
    if ((int)P.jit_part_funcs.size() <= pass) return QSV_OK;
    if (!P.jit_part_funcs[pass]) {
        auto job = async_take(P.jit_part_src[pass], false);
        if (!job) {
            // compiled by another caller (blocking jit_prepare) in the meantime?
            std::lock_guard<std::mutex> lk(g_cache_mu);
            auto it = g_cache.find({device, P.jit_part_src[pass]});
            if (it == g_cache.end()) return QSV_OK;
            P.jit_part_funcs[pass] = it->second.fn;
            P.jit_part_grids[pass] = it->second.grid;
        } else {
            cudaSetDevice(device);
            cudaFree(nullptr);
            std::lock_guard<std::mutex> lk(g_cache_mu);
            CacheEntry e;
            const int rc = load_unit(P, job->u, device, e, err);
            if (rc) return rc;
            P.jit_part_funcs[pass] = e.fn;
            P.jit_part_grids[pass] = e.grid;
        }
    }
    *ready = true;
    // every pass loaded: the plan becomes an ordinary prepared plan
    bool all = true;
    for (void *f : P.jit_part_funcs) all = all && f;
    if (all && !use_supers(P)) {
        P.jit_funcs = P.jit_part_funcs;
        P.jit_grids = P.jit_part_grids;
        P.jit_gangs.assign(P.passes.size(), 1);
        for (size_t i = 0; i < P.passes.size(); ++i) P.jit_gangs[i] = source_gang(P.jit_part_src[i]);
        P.jit_super_funcs.assign(P.supers.size(), nullptr);
        P.jit_super_grids.assign(P.supers.size(), 0);
        P.super_use.assign(P.supers.size(), 0);
        P.jit_device = device;
    }
    return QSV_OK;
}

// Exchange-out variant of one pass (compiled on demand, cached by source).
int jit_variant_prepare(const Plan &P, int pass, const std::string &src, int device, void **fn, int *grid,
                        std::string &err);

int jit_exchange_prepare(const Plan &P, int pass, uint64_t xmask, int device, void **fn, int *grid, std::string &err) {
    if (P.product) {
        err = "exchange-out passes of a product-start plan are not generated";
        return QSV_E_UNSUPPORTED;
    }
    return jit_variant_prepare(P, pass, jit_source(P, pass, false, nullptr, xmask), device, fn, grid, err);
}

int jit_probe_prepare(const Plan &P, int pass, const std::vector<int> &probe, int device, void **fn, int *grid,
                      std::string &err) {
    if (P.product) {
        err = "probe-out passes of a product-start plan are not generated";
        return QSV_E_UNSUPPORTED;
    }
    return jit_variant_prepare(P, pass, jit_source(P, pass, false, nullptr, 0, &probe), device, fn, grid, err);
}

int jit_launch_probe(const Plan &P, int pass, void *fn, int grid, void *psi, int n, cudaStream_t stream,
                     std::string &err, unsigned long long basis, double *probe_out) {
    const int m = P.passes[pass].m, T = 1 << (m - pass_r(P, pass));
    unsigned long long n_tiles = 1ull << (n - m);
    void *args[] = {&psi, &n_tiles, &basis, &probe_out};
    const CUresult r = driver().LaunchKernel((CUfunction)fn, (unsigned)grid, 1, 1, T, 1, 1, (unsigned)((size_t)16 << m),
                                             (CUstream)stream, args, nullptr);
    if (r != CUDA_SUCCESS) {
        const char *s2 = nullptr;
        driver().GetErrorString(r, &s2);
        err = std::string("cuLaunchKernel (probe-out): ") + (s2 ? s2 : "?");
        return QSV_E_DEVICE;
    }
    return QSV_OK;
}

// Compiles (disk cache, NVRTC) and loads a variant of one pass kernel; cached by source.
int jit_variant_prepare(const Plan &P, int pass, const std::string &src, int device, void **fn, int *grid,
                        std::string &err) {
    if (!jit_available(err)) return QSV_E_DEVICE;
    Driver &drv = driver();
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_cache.find({device, src});
        if (it != g_cache.end()) {
            *fn = it->second.fn;
            *grid = it->second.grid;
            return QSV_OK;
        }
    }
    std::string cubin;
    const std::string path = disk_cache_path(src);
    if (!disk_cache_load(path, cubin)) {
        std::string log;
        cubin = jit_compile_cubin(src, log);
        if (cubin.empty()) {
            err = "NVRTC failed for a pass-kernel variant: " + log;
            return QSV_E_DEVICE;
        }
        disk_cache_store(path, cubin);
    }
    cudaSetDevice(device);
    cudaFree(nullptr);
    const int m = P.passes[pass].m;
    CUmodule mod;
    CUfunction f;
    CUresult r = drv.ModuleLoadData(&mod, cubin.data());
    if (r == CUDA_SUCCESS) r = drv.ModuleGetFunction(&f, mod, "qsv_pass");
    const int smem = (int)((size_t)16 << m);
    if (r == CUDA_SUCCESS) r = drv.FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
    int per_sm = 0;
    if (r == CUDA_SUCCESS)
        r = drv.OccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 1 << (m - pass_r(P, pass)), (size_t)smem);
    if (r != CUDA_SUCCESS || per_sm < 1) {
        err = "loading a pass-kernel variant failed";
        return QSV_E_DEVICE;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[{device, src}] = CacheEntry{f, per_sm * sms, 1};
    *fn = f;
    *grid = per_sm * sms;
    return QSV_OK;
}

int jit_launch_exchange(const Plan &P, int pass, void *fn, int grid_cap, void *psi, int n, cudaStream_t stream,
                        std::string &err, unsigned long long basis, const unsigned long long *dst8,
                        unsigned long long self_bits) {
    const int m = P.passes[pass].m, T = 1 << (m - pass_r(P, pass));
    unsigned long long n_tiles = 1ull << (n - m);
    const unsigned grid = (unsigned)std::min<unsigned long long>(n_tiles, (unsigned long long)grid_cap);
    struct XDst {
        unsigned long long p[8];
        unsigned long long self;
    } xd;
    for (int i = 0; i < 8; ++i) xd.p[i] = dst8[i];
    xd.self = self_bits;
    void *args[] = {&psi, &n_tiles, &basis, &xd};
    const CUresult r = driver().LaunchKernel((CUfunction)fn, grid, 1, 1, T, 1, 1, (unsigned)((size_t)16 << m),
                                             (CUstream)stream, args, nullptr);
    if (r != CUDA_SUCCESS) {
        const char *s2 = nullptr;
        driver().GetErrorString(r, &s2);
        err = std::string("cuLaunchKernel (exchange-out): ") + (s2 ? s2 : "?");
        return QSV_E_DEVICE;
    }
    return QSV_OK;
}

static int cu_fail(CUresult r, const char *what, std::string &err) {
    const char *s = nullptr;
    driver().GetErrorString(r, &s);
    err = std::string(what) + ": " + (s ? s : "?");
    return QSV_E_DEVICE;
}

namespace {
int launch_fn(const Plan &P, int pass, void *fnp, int grid_cap_in, int gang, void *psi, int n, cudaStream_t stream,
              std::string &err, unsigned long long basis, const void *ptab);
}

int jit_launch(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err,
               unsigned long long basis, const void *ptab) {
    const int gang = pass < (int)P.jit_gangs.size() ? P.jit_gangs[pass] : 1;
    return launch_fn(P, pass, P.jit_funcs[pass], P.jit_grids[pass], gang, psi, n, stream, err, basis, ptab);
}

int jit_launch_partial(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err,
                       unsigned long long basis, const void *ptab) {
    return launch_fn(P, pass, P.jit_part_funcs[pass], P.jit_part_grids[pass], source_gang(P.jit_part_src[pass]), psi,
                     n, stream, err, basis, ptab);
}

namespace {
int launch_fn(const Plan &P, int pass, void *fnp, int grid_cap_in, int gang, void *psi, int n, cudaStream_t stream,
              std::string &err, unsigned long long basis, const void *ptab) {
    const DevPass &dp = P.passes[pass];
    const int m = dp.m, T = 1 << (m - pass_r(P, pass));
    unsigned long long n_tiles = 1ull << (n - m);
    // One CTA per tile (group) by default: measured faster than the persistent
    // grid (C2 70.7 -> 67.5 ms, QFT 48.5 -> 48.0, C5 1.03 -> 1.00 s) - freshly
    // scheduled CTAs keep the tiles in flight adjacent, and a kernel sharing the
    // GPU with another stream's kernels is not stuck with its early residents.
    // QSV_JIT_GRID_TILES=0 restores the persistent grid.
    const bool per_tile = jit_per_tile_grid();
    const unsigned long long cap = per_tile ? 0x7fffffffull : (unsigned long long)grid_cap_in;
    const unsigned grid = (unsigned)std::min<unsigned long long>((n_tiles + gang - 1) / gang, cap);
    if (P.product && pass == 0 && !ptab) {
        err = "product-start pass launched without its factor tables";
        return QSV_E_UNSUPPORTED;
    }
    void *args[] = {&psi, &n_tiles, &basis, &ptab};
    const CUresult r = driver().LaunchKernel((CUfunction)fnp, grid, 1, 1, gang * T, 1, 1,
                                             gang * (unsigned)((size_t)(jit_double_buffer() ? 32 : 16) << m),
                                             (CUstream)stream, args, nullptr);
    return r == CUDA_SUCCESS ? QSV_OK : cu_fail(r, "cuLaunchKernel", err);
}
}  // namespace

int jit_launch_super(const Plan &P, int si, void *psi, unsigned *bar, cudaStream_t stream, std::string &err) {
    const int m = P.m, T = 1 << (m - P.r), s = popc64(P.supers[si].mask), lb = super_batch(P);
    unsigned long long n_batches = 1ull << (P.n - s - lb);
    cudaError_t ce = cudaMemsetAsync(bar, 0, sizeof(unsigned), stream);
    if (ce != cudaSuccess) {
        err = std::string("barrier reset: ") + cudaGetErrorString(ce);
        return QSV_E_DEVICE;
    }
    const unsigned long long tiles = 1ull << (s - m + lb);
    const unsigned grid = (unsigned)std::min<unsigned long long>(tiles, (unsigned long long)P.jit_super_grids[si]);
    void *args[] = {&psi, &n_batches, &bar};
    // every CTA must be co-resident for the grid barrier: cooperative launch
    const CUresult r = driver().LaunchCooperativeKernel((CUfunction)P.jit_super_funcs[si], grid, 1, 1, T, 1, 1,
                                                        (unsigned)((size_t)(jit_double_buffer() ? 32 : 16) << m),
                                                        (CUstream)stream, args);
    return r == CUDA_SUCCESS ? QSV_OK : cu_fail(r, "cuLaunchCooperativeKernel", err);
}

}  // namespace qsv
