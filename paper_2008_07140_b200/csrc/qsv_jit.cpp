// Runtime specialisation of pass kernels (see qsv_jit.h).
#include "qsv_jit.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <vector>

namespace qsv {

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
                 sym(h, "cuGetErrorString", api.GetErrorString);
        if (!api.ok) api.why = "libcuda lacks a required symbol";
    });
    return api;
}

// ---------------------------------------------------------------------------
// source generation
// ---------------------------------------------------------------------------

const char *kPrelude = R"(
typedef unsigned long long u64;
__device__ __forceinline__ unsigned swz(unsigned i) {
    unsigned h = i >> 3;
    h ^= h >> 3;
    h ^= h >> 6;
    return i ^ (h & 7u);
}
__device__ __forceinline__ double2 ldcs2(const double2 *p) {
    double2 r;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcs2(double2 *p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
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

uint32_t swz_host(uint32_t i) {
    uint32_t h = i >> 3;
    h ^= h >> 3;
    h ^= h >> 6;
    return i ^ (h & 7u);
}

struct StageGen {
    std::ostringstream &o;
    int R;
    const std::vector<int> &tq;     // tile qubits by local bit
    std::vector<int> regq;          // register position k -> global qubit
    std::map<int, int> thread_bit;  // global qubit -> thread id bit (stage thread bits)
    std::vector<cd> pend;           // pending constant phase per register amplitude

    StageGen(std::ostringstream &out, int r, const std::vector<int> &t) : o(out), R(r), tq(t), pend(1u << r, cd(1, 0)) {}

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
        const double cr = c.real(), ci = c.imag();
        if (cr == 1.0 && ci == 0.0) return;
        if (cr == -1.0 && ci == 0.0) {
            o << "    " << v << " = make_double2(-" << v << ".x, -" << v << ".y);\n";
        } else if (ci == 0.0) {
            o << "    " << v << " = make_double2(" << v << ".x * " << lit(cr) << ", " << v << ".y * " << lit(cr) << ");\n";
        } else if (cr == 0.0) {
            if (ci == 1.0) o << "    " << v << " = make_double2(-" << v << ".y, " << v << ".x);\n";
            else if (ci == -1.0) o << "    " << v << " = make_double2(" << v << ".y, -" << v << ".x);\n";
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
    void flush_all() {
        for (int r = 0; r < (1 << R); ++r) flush(r);
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
                return any ? e.str() : std::string("0.0");
            };
            o << "      v" << idx[r] << " = make_double2(" << comp(false) << ", " << comp(true) << ");\n";
        }
        o << "    }\n";
    }

    std::string scalar_cond(uint64_t smask) const {
        std::string c;
        for (int q = 0; q < 64; ++q)
            if ((smask >> q) & 1) c += (c.empty() ? "" : " && ") + scalar_expr(q);
        return c;
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
            for (auto &grp : groups)
                for (int r : grp) flush(r);
            const std::string cond = scalar_cond(smask);
            if (!cond.empty()) o << "    if (" << cond << ") {\n";
            for (auto &grp : groups) linear(grp, g.m);
            if (!cond.empty()) o << "    }\n";
            return;
        }
        // diagonal: factor(rho, scalars) = controls ? d[bits] : 1
        std::vector<int> dq = {g.qa};
        std::vector<cd> d = {g.m[0], g.m[1]};
        if (g.kind == QSV_OP_DIAG2) {
            dq = {g.qa, g.qb};
            d = {g.m[0], g.m[1], g.m[2], g.m[3]};
        }
        std::vector<int> sq;  // scalar target qubits
        for (int q : dq)
            if (regpos(q) < 0) sq.push_back(q);
        const std::string ccond = scalar_cond(smask);
        const int ns = (int)sq.size();
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

// Host rendering of the same pass (test infrastructure: tests compile it with
// gcc and run it on CPU to check the generator against the oracle without a
// GPU).  Identical op emission; the CTA becomes explicit loops over threads
// between barriers.
const char *kHostPrelude = R"(
#include <stdint.h>
typedef unsigned long long u64;
struct double2 { double x, y; };
static inline double2 make_double2(double x, double y) { double2 r; r.x = x; r.y = y; return r; }
static inline unsigned swz(unsigned i) {
    unsigned h = i >> 3;
    h ^= h >> 3;
    h ^= h >> 6;
    return i ^ (h & 7u);
}
static inline double2 ldcs2(const double2 *p) { return *p; }
static inline void stcs2(double2 *p, double2 v) { *p = v; }
)";

std::string jit_source(const Plan &P, int pi, bool host) {
    const DevPass &dp = P.passes[pi];
    const int n = P.n, m = dp.m, R = P.r, T = 1 << (m - R);
    std::vector<int> tq(dp.tq, dp.tq + m);
    std::ostringstream o;
    o << "// libqsv specialised pass kernel: n=" << n << " m=" << m << " R=" << R << " pass=" << pi << "\n";
    // tile base: deposit tile_id into the non-tile qubits
    std::vector<int> ext;
    for (int q = 0; q < n; ++q)
        if (!((dp.tile_mask >> q) & 1)) ext.push_back(q);
    std::vector<int> low(tq.begin(), tq.begin() + (m - R)), high(tq.begin() + (m - R), tq.end());
    const std::string thread_loop = host ? "    for (unsigned tid = 0; tid < " + std::to_string(T) + "u; ++tid) {\n" : "";
    const std::string thread_end = host ? "    }\n" : "";
    const std::string barrier = host ? "" : "    __syncthreads();\n";
    if (host) {
        o << kHostPrelude;
        o << "extern \"C\" void qsv_pass_host(double2 *psi, u64 n_tiles) {\n";
        o << "  static double2 tile[" << (1 << m) << "];\n";
        o << "  for (u64 tile_id = 0; tile_id < n_tiles; ++tile_id) {\n";
    } else {
        o << kPrelude;
        o << "extern \"C\" __global__ void __launch_bounds__(" << T
          << ") qsv_pass(double2 *__restrict__ psi, u64 n_tiles) {\n";
        o << "  extern __shared__ double2 tile[];\n";
        o << "  const unsigned tid = threadIdx.x;\n";
        o << "  const u64 toff = " << deposit_expr("tid", low, true) << ";\n";
        o << "  const unsigned tsl = swz(tid);\n";
        o << "  for (u64 tile_id = blockIdx.x; tile_id < n_tiles; tile_id += gridDim.x) {\n";
    }
    o << "    const u64 base = " << deposit_expr("tile_id", ext, true) << ";\n";
    o << barrier << thread_loop;
    if (host) {
        o << "    const u64 toff = " << deposit_expr("tid", low, true) << ";\n";
        o << "    const unsigned tsl = swz(tid);\n";
    }
    o << "    double2 *p = psi + base + toff;\n";
    for (int k = 0; k < (1 << R); ++k) {
        const uint64_t off = deposit((uint64_t)k, high);
        o << "    tile[tsl ^ " << swz_host((uint32_t)k * T) << "u] = ldcs2(p + " << off << "ull);\n";
    }
    o << thread_end << barrier;
    for (int s = dp.stage_begin; s < dp.stage_end; ++s) {
        const DevStage &st = P.stages[s];
        StageGen g(o, R, tq);
        g.regq.resize(R);
        for (int k = 0; k < R; ++k) g.regq[k] = tq[st.rb[k]];
        std::vector<int> nonreg;
        for (int j = 0; j < m; ++j)
            if (!((st.reg_local_mask >> j) & 1)) nonreg.push_back(j);
        for (size_t j = 0; j < nonreg.size(); ++j) g.thread_bit[tq[nonreg[j]]] = (int)j;
        o << "    { // stage " << (s - dp.stage_begin) << " registers:";
        for (int k = 0; k < R; ++k) o << " q" << g.regq[k];
        o << "\n" << thread_loop;
        o << "    const unsigned tsw = swz(" << deposit_expr("tid", nonreg, false) << ");\n";
        std::vector<uint32_t> c(1u << R);
        for (int rho = 0; rho < (1 << R); ++rho) {
            uint32_t off = 0;
            for (int k = 0; k < R; ++k)
                if ((rho >> k) & 1) off |= 1u << st.rb[k];
            c[rho] = swz_host(off);
            o << "    double2 v" << rho << " = tile[tsw ^ " << c[rho] << "u];\n";
        }
        for (int oi = st.op_begin; oi < st.op_end; ++oi) g.op(P.gops[oi]);
        g.flush_all();
        for (int rho = 0; rho < (1 << R); ++rho) o << "    tile[tsw ^ " << c[rho] << "u] = v" << rho << ";\n";
        o << thread_end << barrier << "    }\n";
    }
    o << thread_loop;
    if (host) {
        o << "    const u64 toff = " << deposit_expr("tid", low, true) << ";\n";
        o << "    const unsigned tsl = swz(tid);\n";
        o << "    double2 *p = psi + base + toff;\n";
    }
    for (int k = 0; k < (1 << R); ++k) {
        const uint64_t off = deposit((uint64_t)k, high);
        o << "    stcs2(p + " << off << "ull, tile[tsl ^ " << swz_host((uint32_t)k * T) << "u]);\n";
    }
    o << thread_end << "  }\n}\n";
    return o.str();
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
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "--extra-device-vectorization"};
    const nvrtcResult rc = api.CompileProgram(prog, 5, opts);
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

struct CacheEntry {
    CUfunction fn = nullptr;
    int smem_set = 0;
};

std::mutex g_cache_mu;
std::map<std::pair<int, std::string>, CacheEntry> g_cache;  // (device, source) -> kernel

}  // namespace

int jit_prepare(Plan &P, int device, std::string &err) {
    if (P.jit_device == device && P.jit_funcs.size() == P.passes.size()) return QSV_OK;
    if (!jit_available(err)) return QSV_E_DEVICE;
    Driver &drv = driver();
    const size_t np = P.passes.size();
    std::vector<std::string> srcs(np), cubins(np), logs(np);
    std::vector<void *> funcs(np, nullptr);
    std::vector<int> todo;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < np; ++i) {
            srcs[i] = jit_source(P, (int)i);
            auto it = g_cache.find({device, srcs[i]});
            if (it != g_cache.end()) funcs[i] = it->second.fn;
            else todo.push_back((int)i);
        }
    }
    // compile the missing kernels concurrently (independent NVRTC programs)
    {
        std::vector<std::thread> pool;
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::atomic<size_t> next{0};
        for (unsigned t = 0; t < std::min<size_t>(hw, todo.size()); ++t)
            pool.emplace_back([&] {
                for (size_t k; (k = next.fetch_add(1)) < todo.size();) {
                    const int i = todo[k];
                    cubins[i] = jit_compile_cubin(srcs[i], logs[i]);
                }
            });
        for (auto &th : pool) th.join();
    }
    cudaSetDevice(device);
    cudaFree(nullptr);  // make the primary context current for the driver API
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (int i : todo) {
        if (cubins[i].empty()) {
            err = "NVRTC failed for pass " + std::to_string(i) + ": " + logs[i];
            return QSV_E_DEVICE;
        }
        CUmodule mod;
        CUfunction fn;
        CUresult r = drv.ModuleLoadData(&mod, cubins[i].data());
        if (r == CUDA_SUCCESS) r = drv.ModuleGetFunction(&fn, mod, "qsv_pass");
        const int smem = (int)((size_t)16 << P.passes[i].m);
        if (r == CUDA_SUCCESS) r = drv.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
        if (r != CUDA_SUCCESS) {
            const char *s = nullptr;
            drv.GetErrorString(r, &s);
            err = std::string("loading specialised kernel: ") + (s ? s : "?");
            return QSV_E_DEVICE;
        }
        g_cache[{device, srcs[i]}] = CacheEntry{fn, smem};
        funcs[i] = fn;
    }
    P.jit_funcs = funcs;
    P.jit_device = device;
    return QSV_OK;
}

int jit_launch(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err) {
    const DevPass &dp = P.passes[pass];
    const int m = dp.m, T = 1 << (m - P.r);
    unsigned long long n_tiles = 1ull << (n - m);
    const unsigned grid = (unsigned)std::min<unsigned long long>(n_tiles, 0x7fffffffull);
    void *args[] = {&psi, &n_tiles};
    const CUresult r = driver().LaunchKernel((CUfunction)P.jit_funcs[pass], grid, 1, 1, T, 1, 1,
                                             (unsigned)((size_t)16 << m), (CUstream)stream, args, nullptr);
    if (r != CUDA_SUCCESS) {
        const char *s = nullptr;
        driver().GetErrorString(r, &s);
        err = std::string("cuLaunchKernel: ") + (s ? s : "?");
        return QSV_E_DEVICE;
    }
    return QSV_OK;
}

}  // namespace qsv
