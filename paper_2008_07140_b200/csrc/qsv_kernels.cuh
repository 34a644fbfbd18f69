// sm_100a kernels of libqsv.  Included once, by qsv_api.cu.
//
// Layout in HBM: one contiguous complex128 array (double2, 16 B, 16-B aligned),
// index bit k <-> qubit k.  Every kernel moves amplitudes as 128-bit
// double2 loads/stores; consecutive threads touch consecutive amplitudes
// wherever the schedule allows (the planner forces the lowest qubits into
// every tile so a warp streams >= 512 contiguous bytes).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qsv_plan.h"

namespace qsv {

// ---------------------------------------------------------------------------
// complex helpers (FP64 on the CUDA cores; B200 has no FP64 tcgen05 kind)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// u0*x0 + u1*x1
__device__ __forceinline__ double2 cdot2(double2 u0, double2 x0, double2 u1, double2 x1) {
    double re = u0.x * x0.x;
    re = fma(-u0.y, x0.y, re);
    re = fma(u1.x, x1.x, re);
    re = fma(-u1.y, x1.y, re);
    double im = u0.x * x0.y;
    im = fma(u0.y, x0.x, im);
    im = fma(u1.x, x1.y, im);
    im = fma(u1.y, x1.x, im);
    return make_double2(re, im);
}

// op records are read through generic pointers: the pass kernel stages its
// ops in shared memory (uniform broadcast reads), or reads them from global
__device__ __forceinline__ double2 ldm(const double *m, int k) { return make_double2(m[2 * k], m[2 * k + 1]); }

// matrix entry load the compiler may not hoist out of a loop (keeps register
// pressure bounded for dense 4x4 ops; the entries stay L1-resident)
__device__ __forceinline__ double2 ldm_v(const double *m, int k) {
    double2 r;
    asm volatile("ld.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(m + 2 * k));
    return r;
}

// shared-memory swizzle: XOR the 16-B slot inside each 128-B row with a fold
// of the higher index bits, so lanes whose local indices differ only in high
// bits still spread over all bank groups (a bijection: bits >= 3 unchanged).
__device__ __forceinline__ uint32_t swz(uint32_t i) {
    uint32_t h = i >> 3;
    h ^= h >> 3;
    h ^= h >> 6;
    return i ^ (h & 7u);
}

__device__ __forceinline__ uint32_t deposit32(uint32_t v, uint32_t mask) {
    uint32_t out = 0;
    while (mask) {
        const uint32_t low = mask & (0u - mask);
        if (v & 1u) out |= low;
        v >>= 1;
        mask ^= low;
    }
    return out;
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t v, int q) {
    const uint64_t lowm = (1ull << q) - 1;
    return ((v & ~lowm) << 1) | (v & lowm);
}

// ---------------------------------------------------------------------------
// fused pass kernel
// ---------------------------------------------------------------------------

template <int R>
__device__ __forceinline__ uint32_t reg_offset(int rho, const uint32_t (&rm)[R]) {
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < R; ++k)
        if ((rho >> k) & 1) s |= rm[k];
    return s;
}

__device__ __forceinline__ double2 cneg(double2 x) {
    return make_double2(__longlong_as_double(__double_as_longlong(x.x) ^ (long long)0x8000000000000000ull),
                        __longlong_as_double(__double_as_longlong(x.y) ^ (long long)0x8000000000000000ull));
}

// multiply the amplitudes of one register class (rho & cls_mask) == cls_val by f;
// mode (from the plan): 0 f == 1 (nothing), 1 f == -1 (sign flip), 2 general
template <int R, bool CTRL>
__device__ __forceinline__ void scale_class(double2 (&v)[1 << R], int cls_mask, int cls_val, double2 f, uint32_t mode,
                                            uint32_t rc) {
    if (mode == 0) return;
    if (mode == 1) {
#pragma unroll
        for (int rho = 0; rho < (1 << R); ++rho)
            if ((rho & cls_mask) == cls_val && (!CTRL || (rho & rc) == rc)) v[rho] = cneg(v[rho]);
    } else {
#pragma unroll
        for (int rho = 0; rho < (1 << R); ++rho)
            if ((rho & cls_mask) == cls_val && (!CTRL || (rho & rc) == rc)) v[rho] = cmul(v[rho], f);
    }
}

template <int V>
__device__ __forceinline__ void mat1_pair(double2 &x0, double2 &x1, const double *m) {
    const double2 a = x0, b = x1;
    if constexpr (V == V_REAL) {
        const double u00 = m[0], u01 = m[2], u10 = m[4], u11 = m[6];
        x0 = make_double2(fma(u01, b.x, u00 * a.x), fma(u01, b.y, u00 * a.y));
        x1 = make_double2(fma(u11, b.x, u10 * a.x), fma(u11, b.y, u10 * a.y));
    } else if constexpr (V == V_RXL) {
        // [[p, i q], [i r, s]] with p, q, r, s real
        const double p = m[0], q = m[3], r = m[5], t = m[6];
        x0 = make_double2(fma(-q, b.y, p * a.x), fma(q, b.x, p * a.y));
        x1 = make_double2(fma(t, b.x, -r * a.y), fma(t, b.y, r * a.x));
    } else {
        x0 = cdot2(ldm(m, 0), a, ldm(m, 1), b);
        x1 = cdot2(ldm(m, 2), a, ldm(m, 3), b);
    }
}

template <int R, int A, int V, bool CTRL>
__device__ __forceinline__ void op_mat1(double2 (&v)[1 << R], const double *m, uint32_t rc) {
#pragma unroll
    for (int rho = 0; rho < (1 << R); ++rho) {
        if (rho & (1 << A)) continue;
        if (CTRL && (rho & rc) != rc) continue;
        mat1_pair<V>(v[rho], v[rho | (1 << A)], m);
    }
}

template <int R, int A, bool CTRL>
__device__ __forceinline__ void mat1_var(uint32_t var, double2 (&v)[1 << R], const double *m, uint32_t rc) {
    if (var == V_REAL) op_mat1<R, A, V_REAL, CTRL>(v, m, rc);
    else if (var == V_RXL) op_mat1<R, A, V_RXL, CTRL>(v, m, rc);
    else op_mat1<R, A, V_GEN, CTRL>(v, m, rc);
}

template <int R, int A>
__device__ __forceinline__ void dispatch_mat1(uint32_t a, uint32_t var, double2 (&v)[1 << R], const double *m,
                                              uint32_t rc) {
    if constexpr (A < R) {
        if (a == A) {
            if (rc) mat1_var<R, A, true>(var, v, m, rc);
            else mat1_var<R, A, false>(var, v, m, rc);
        } else {
            dispatch_mat1<R, A + 1>(a, var, v, m, rc);
        }
    }
}

template <int R, int A, int B>
__device__ __forceinline__ void op_mat2_perm(double2 (&v)[1 << R], const double *m, uint32_t code, uint32_t rc) {
    int src[4];
    uint32_t mode[4];
    double2 ph[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        src[r] = (code >> (24 + 2 * r)) & 3;
        mode[r] = (code >> (16 + 2 * r)) & 3;
        ph[r] = ldm(m, r);
    }
#pragma unroll
    for (int rho = 0; rho < (1 << R); ++rho) {
        if (rho & ((1 << A) | (1 << B))) continue;
        if ((rho & rc) != rc) continue;
        const int idx[4] = {rho, rho | (1 << B), rho | (1 << A), rho | (1 << A) | (1 << B)};
        const double2 x[4] = {v[idx[0]], v[idx[1]], v[idx[2]], v[idx[3]]};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            // select the source with compile-time register indices
            const double2 xs = src[r] == 0 ? x[0] : src[r] == 1 ? x[1] : src[r] == 2 ? x[2] : x[3];
            v[idx[r]] = mode[r] == 0 ? xs : (mode[r] == 1 ? cneg(xs) : cmul(xs, ph[r]));
        }
    }
}

template <int R, int A, int B>
__device__ __forceinline__ void op_mat2_gen(double2 (&v)[1 << R], const double *m, uint32_t rc) {
#pragma unroll
    for (int rho = 0; rho < (1 << R); ++rho) {
        if (rho & ((1 << A) | (1 << B))) continue;
        if ((rho & rc) != rc) continue;
        const int idx[4] = {rho, rho | (1 << B), rho | (1 << A), rho | (1 << A) | (1 << B)};
        const double2 x[4] = {v[idx[0]], v[idx[1]], v[idx[2]], v[idx[3]]};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double2 p = cdot2(ldm_v(m, 4 * r), x[0], ldm_v(m, 4 * r + 1), x[1]);
            const double2 q = cdot2(ldm_v(m, 4 * r + 2), x[2], ldm_v(m, 4 * r + 3), x[3]);
            v[idx[r]] = make_double2(p.x + q.x, p.y + q.y);
        }
    }
}

template <int R, int A, int B, bool PERM>
__device__ __forceinline__ void dispatch_mat2(uint32_t a, uint32_t b, double2 (&v)[1 << R], const double *m,
                                              uint32_t code, uint32_t rc) {
    if constexpr (A < R) {
        if constexpr (B < R) {
            if constexpr (A != B) {
                if (a == A && b == B) {
                    if constexpr (PERM) op_mat2_perm<R, A, B>(v, m, code, rc);
                    else op_mat2_gen<R, A, B>(v, m, rc);
                    return;
                }
            }
            dispatch_mat2<R, A, B + 1, PERM>(a, b, v, m, code, rc);
        } else {
            dispatch_mat2<R, A + 1, 0, PERM>(a, b, v, m, code, rc);
        }
    }
}

// diagonal with one register qubit at position P: two classes by bit P
template <int R, int P, bool CTRL>
__device__ __forceinline__ void dispatch_diag1(uint32_t p, double2 (&v)[1 << R], double2 f0, uint32_t m0, double2 f1,
                                               uint32_t m1, uint32_t rc) {
    if constexpr (P < R) {
        if (p == P) {
            scale_class<R, CTRL>(v, 1 << P, 0, f0, m0, rc);
            scale_class<R, CTRL>(v, 1 << P, 1 << P, f1, m1, rc);
        } else {
            dispatch_diag1<R, P + 1, CTRL>(p, v, f0, m0, f1, m1, rc);
        }
    }
}

// diagonal with two register qubits at positions (A, B): four classes (bitA, bitB)
template <int R, int A, int B, bool CTRL>
__device__ __forceinline__ void dispatch_diag2(uint32_t a, uint32_t b, double2 (&v)[1 << R], const double *m,
                                               uint32_t modes, uint32_t rc) {
    if constexpr (A < R) {
        if constexpr (B < R) {
            if constexpr (A != B) {
                if (a == A && b == B) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint32_t mc = (modes >> (2 * c)) & 3;
                        if (mc) scale_class<R, CTRL>(v, (1 << A) | (1 << B), ((c >> 1) << A) | ((c & 1) << B),
                                                     ldm(m, c), mc, rc);
                    }
                    return;
                }
            }
            dispatch_diag2<R, A, B + 1, CTRL>(a, b, v, m, modes, rc);
        } else {
            dispatch_diag2<R, A + 1, 0, CTRL>(a, b, v, m, modes, rc);
        }
    }
}

__device__ __forceinline__ uint32_t scalar_bit(uint32_t desc, uint32_t tpart, uint64_t base) {
    if (desc == kNoScalar) return 0;
    if (desc < (uint32_t)kScalarExt) return (tpart >> desc) & 1u;
    return (uint32_t)((base >> (desc - kScalarExt)) & 1ull);
}

template <int R, bool CTRL>
__device__ __forceinline__ void apply_diag(uint32_t code, uint32_t rs, const double *m, double2 (&v)[1 << R],
                                           uint32_t tpart, uint64_t base, uint32_t rc) {
    const uint32_t var = (code >> 4) & 15, a = (code >> 8) & 15, b = (code >> 12) & 15, modes = (code >> 16) & 0xff;
    if (var == D_AB) {
        dispatch_diag2<R, 0, 0, CTRL>(a, b, v, m, modes, rc);
        return;
    }
    const uint32_t sA = scalar_bit((rs >> 8) & 0xff, tpart, base), sB = scalar_bit((rs >> 16) & 0xff, tpart, base);
    if (var == D_NONE) {
        const uint32_t e = 2 * sA + sB;
        scale_class<R, CTRL>(v, 0, 0, ldm(m, e), (modes >> (2 * e)) & 3, rc);
    } else if (var == D_A) {
        const uint32_t e0 = sB, e1 = 2 + sB;
        dispatch_diag1<R, 0, CTRL>(a, v, ldm(m, e0), (modes >> (2 * e0)) & 3, ldm(m, e1), (modes >> (2 * e1)) & 3, rc);
    } else {
        const uint32_t e0 = 2 * sA, e1 = 2 * sA + 1;
        dispatch_diag1<R, 0, CTRL>(b, v, ldm(m, e0), (modes >> (2 * e0)) & 3, ldm(m, e1), (modes >> (2 * e1)) & 3, rc);
    }
}

template <int R>
__device__ __forceinline__ void apply_op(const DevOp *op, double2 (&v)[1 << R], uint32_t tpart, uint64_t base) {
    const uint4 h = *reinterpret_cast<const uint4 *>(op);
    const uint64_t ec = *(reinterpret_cast<const unsigned long long *>(op) + 2);
    const uint32_t code = h.x, rs = h.y, tc = h.z;
    // most ops carry no scalar control: the test on the (CTA-uniform) record first keeps
    // tpart / base, which the register allocator spills, out of the common path
    if ((tc | (uint32_t)ec | (uint32_t)(ec >> 32)) != 0u)
        if ((tpart & tc) != tc || (base & ec) != ec) return;  // a scalar control is 0 for this thread
    const uint32_t kind = code & 15, rc = rs & 0xff;
    const double *m = op->m;
    if (kind == K_MAT1) {
        dispatch_mat1<R, 0>((code >> 8) & 15, (code >> 4) & 15, v, m, rc);
    } else if (kind == K_MAT2) {
        if (((code >> 4) & 15) == V_PERM) dispatch_mat2<R, 0, 0, true>((code >> 8) & 15, (code >> 12) & 15, v, m, code, rc);
        else dispatch_mat2<R, 0, 0, false>((code >> 8) & 15, (code >> 12) & 15, v, m, code, rc);
    } else {
        if (rc) apply_diag<R, true>(code, rs, m, v, tpart, base, rc);
        else apply_diag<R, false>(code, rs, m, v, tpart, base, rc);
    }
}

// One CTA = one tile of 2^m amplitudes (tile qubits = pass->tile_mask).  The
// tile is streamed HBM -> shared memory (coalesced 128-bit loads), then each
// stage gathers 2^R amplitudes per thread over the stage's register qubits,
// applies the stage's ops in registers and scatters them back; the last
// stage's result streams back to HBM.  Tiles are independent (disjoint index
// sets), so there is no inter-CTA communication and no atomics.
// SMEM_OPS: the pass's op records are staged in shared memory once per
// (persistent) CTA and read as uniform broadcasts (global L1 reads per op and
// thread were the interpreter's main stall, long_scoreboard ~4 per issue)
// product-state amplitude from the 5-bit group tables (product_state_kernel's rule)
__device__ __forceinline__ double2 product_amp(const double2 *__restrict__ tab, int groups, uint64_t i) {
    double2 a = tab[i & 31];
    for (int g = 1; g < groups; ++g) {
        const double2 b = tab[32 * g + ((i >> (5 * g)) & 31)];
        a = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
    return a;
}

// ptab != nullptr: the tile is synthesised as the product state of those tables
// instead of read (the interpreted first pass of a product-start plan on a cold call)
template <int R, bool SMEM_OPS>
__global__ void __launch_bounds__(512) pass_kernel(double2 *__restrict__ psi, const DevPass *__restrict__ pass,
                                                   const DevStage *__restrict__ stages,
                                                   const DevOp *__restrict__ ops_g, uint64_t n_tiles,
                                                   const double2 *__restrict__ ptab, int groups) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = pass->m;
    const uint32_t nloc = 1u << m;
    double2 *tile = reinterpret_cast<double2 *>(smem_raw);
    uint64_t *lo_tab = reinterpret_cast<uint64_t *>(smem_raw + ((size_t)16 << m));
    uint64_t *hi_tab = lo_tab + (1 << kLoTabBits);
    const uint32_t T = blockDim.x;

    for (uint32_t e = threadIdx.x; e < (1u << kLoTabBits); e += T) lo_tab[e] = pass->lo_tab[e];
    for (uint32_t e = threadIdx.x; e < (1u << kHiTabBits); e += T) hi_tab[e] = pass->hi_tab[e];
    const int sb = pass->stage_begin, se = pass->stage_end;
    const DevOp *ops = ops_g;
    if constexpr (SMEM_OPS) {
        const int o0 = stages[sb].op_begin, o1 = stages[se - 1].op_end;
        DevOp *ops_s = reinterpret_cast<DevOp *>(hi_tab + (1 << kHiTabBits));
        const uint4 *src = reinterpret_cast<const uint4 *>(ops_g + o0);
        uint4 *dst = reinterpret_cast<uint4 *>(ops_s);
        const uint32_t words = (uint32_t)(o1 - o0) * (uint32_t)(sizeof(DevOp) / 16);
        for (uint32_t w = threadIdx.x; w < words; w += T) dst[w] = src[w];
        ops = ops_s - o0;  // ops[o] for o in [o0, o1)
    }

    for (uint64_t tile_id = blockIdx.x; tile_id < n_tiles; tile_id += gridDim.x) {
        uint64_t base = tile_id;
        for (int j = 0; j < m; ++j) base = insert_zero(base, pass->tq[j]);
        __syncthreads();
        if (ptab) {
            for (uint32_t i = threadIdx.x; i < nloc; i += T)
                tile[swz(i)] = product_amp(ptab, groups,
                                           base + (lo_tab[i & ((1u << kLoTabBits) - 1)] | hi_tab[i >> kLoTabBits]));
        } else {
            // T = nloc >> R (launch_pass): exactly 2^R elements per thread.  All loads are
            // issued before the first shared-memory store needs its data (the rolled loop
            // kept one load in flight per warp: its long-scoreboard wait was the kernel's
            // top stall, 12.7 % of all samples, ncu r02)
            double2 in[1 << R];
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) {
                const uint32_t i = threadIdx.x + (uint32_t)k * T;
                in[k] = __ldcs(psi + base + (lo_tab[i & ((1u << kLoTabBits) - 1)] | hi_tab[i >> kLoTabBits]));
            }
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) tile[swz(threadIdx.x + (uint32_t)k * T)] = in[k];
        }
        __syncthreads();

        for (int s = sb; s < se; ++s) {
            const DevStage *st = stages + s;
            const uint32_t rmask = st->reg_local_mask;
            uint32_t rm[R];
#pragma unroll
            for (int k = 0; k < R; ++k) rm[k] = 1u << st->rb[k];
            const uint32_t tpart = deposit32(threadIdx.x, (nloc - 1) & ~rmask);
            // swz is linear over GF(2) and tpart / register offsets have disjoint bits
            const uint32_t tsw = swz(tpart);
            double2 v[1 << R];
#pragma unroll
            for (int rho = 0; rho < (1 << R); ++rho) v[rho] = tile[tsw ^ swz(reg_offset<R>(rho, rm))];

            const int ob = st->op_begin, oe = st->op_end;
            for (int o = ob; o < oe; ++o) apply_op<R>(ops + o, v, tpart, base);
#pragma unroll
            for (int rho = 0; rho < (1 << R); ++rho) tile[tsw ^ swz(reg_offset<R>(rho, rm))] = v[rho];
            __syncthreads();
        }

#pragma unroll
        for (int k = 0; k < (1 << R); ++k) {
            const uint32_t i = threadIdx.x + (uint32_t)k * T;
            __stcs(psi + base + (lo_tab[i & ((1u << kLoTabBits) - 1)] | hi_tab[i >> kLoTabBits]), tile[swz(i)]);
        }
    }
}

// ---------------------------------------------------------------------------
// unfused single-gate kernel (one HBM sweep over the touched amplitudes per gate)
// ---------------------------------------------------------------------------

struct GateArgs {
    int nt, t0, t1, n_ins;
    uint64_t cmask;
    int ins[64];     // sorted qubits (targets + controls) to insert as zero bits
    double2 u[16];   // row-major
};

__global__ void __launch_bounds__(256) gate_kernel(double2 *__restrict__ psi, const GateArgs g, uint64_t n_groups) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_groups; k += stride) {
        uint64_t i = k;
        for (int j = 0; j < g.n_ins; ++j) i = insert_zero(i, g.ins[j]);
        i |= g.cmask;
        if (g.nt == 1) {
            const uint64_t j1 = i | (1ull << g.t0);
            const double2 x0 = psi[i], x1 = psi[j1];
            psi[i] = cdot2(g.u[0], x0, g.u[1], x1);
            psi[j1] = cdot2(g.u[2], x0, g.u[3], x1);
        } else {
            const uint64_t a = 1ull << g.t0, b = 1ull << g.t1;
            const uint64_t idx[4] = {i, i | b, i | a, i | a | b};
            double2 x[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) x[c] = psi[idx[c]];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double2 p = cdot2(g.u[4 * r], x[0], g.u[4 * r + 1], x[1]);
                const double2 q = cdot2(g.u[4 * r + 2], x[2], g.u[4 * r + 3], x[3]);
                psi[idx[r]] = make_double2(p.x + q.x, p.y + q.y);
            }
        }
    }
}

// diagonal gate: every amplitude whose controls are set gets d[target bits]
__global__ void __launch_bounds__(256) diag_kernel(double2 *__restrict__ psi, const GateArgs g, uint64_t n_idx) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_idx; k += stride) {
        uint64_t i = k;
        for (int j = 0; j < g.n_ins; ++j) i = insert_zero(i, g.ins[j]);  // controls only
        i |= g.cmask;
        const int sel = g.nt == 1 ? (int)((i >> g.t0) & 1) : (int)(2 * ((i >> g.t0) & 1) + ((i >> g.t1) & 1));
        psi[i] = cmul(psi[i], g.u[sel]);
    }
}

// ---------------------------------------------------------------------------
// state initialisation and readout
// ---------------------------------------------------------------------------

__global__ void set_basis_kernel(double2 *psi, uint64_t size, uint64_t index) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride)
        psi[i] = make_double2(i == index ? 1.0 : 0.0, 0.0);
}

// Product state (x)_q v_q from 5-bit group tables (product_tables with no register
// qubits): amplitude(i) = prod_g tab[32 g + ((i >> 5 g) & 31)].  The interpreted
// first pass of a product-start plan reads this state (cold calls, execute_plan_mixed).
__global__ void product_state_kernel(double2 *psi, uint64_t size, const double2 *__restrict__ tab, int groups) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        double2 a = tab[i & 31];
        for (int g = 1; g < groups; ++g) {
            const double2 b = tab[32 * g + ((i >> (5 * g)) & 31)];
            a = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
        }
        psi[i] = a;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// block-level reduction of up to 2 values; thread 0 writes partial[blockIdx.x*2 + {0,1}]
template <bool MAX>
__device__ __forceinline__ void block_reduce2(double a, double b, double *partial) {
    __shared__ double sa[32], sb[32];
    a = MAX ? warp_max(a) : warp_sum(a);
    b = MAX ? warp_max(b) : warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sa[w] = a;
        sb[w] = b;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        a = l < nw ? sa[l] : 0.0;
        b = l < nw ? sb[l] : 0.0;
        a = MAX ? warp_max(a) : warp_sum(a);
        b = MAX ? warp_max(b) : warp_sum(b);
        if (l == 0) {
            partial[2 * blockIdx.x] = a;
            partial[2 * blockIdx.x + 1] = b;
        }
    }
}

// mode 0: sum |a|^2; mode 1: sum |a|^2 over bit k == 0; mode 2: <psi|other>; mode 3: max |psi-other|
__global__ void __launch_bounds__(256) reduce_kernel(const double2 *__restrict__ psi, const double2 *__restrict__ other,
                                                     uint64_t size, int mode, int k, double *partial) {
    double a = 0.0, b = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t count = mode == 1 ? size >> 1 : size;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        if (mode == 0) {
            const double2 x = psi[j];
            a = fma(x.x, x.x, a);
            a = fma(x.y, x.y, a);
        } else if (mode == 1) {
            const double2 x = psi[insert_zero(j, k)];
            a = fma(x.x, x.x, a);
            a = fma(x.y, x.y, a);
        } else if (mode == 2) {
            const double2 x = psi[j], y = other[j];
            a = fma(x.x, y.x, a);  // Re(conj(x) y)
            a = fma(x.y, y.y, a);
            b = fma(x.x, y.y, b);  // Im(conj(x) y)
            b = fma(-x.y, y.x, b);
        } else {
            const double2 x = psi[j], y = other[j];
            a = fmax(a, hypot(x.x - y.x, x.y - y.y));
        }
    }
    if (mode == 3) block_reduce2<true>(a, b, partial);
    else block_reduce2<false>(a, b, partial);
}

// deterministic second stage: one block sums (or maxes) the per-block partials in order
__global__ void finish_kernel(const double *partial, int n_blocks, int mode, double *out) {
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n_blocks; i += blockDim.x) {
        if (mode == 3) {
            a = fmax(a, partial[2 * i]);
        } else {
            a += partial[2 * i];
            b += partial[2 * i + 1];
        }
    }
    __shared__ double sa[32], sb[32];
    a = mode == 3 ? warp_max(a) : warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sa[w] = a;
        sb[w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ra = sa[0], rb = sb[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            ra = mode == 3 ? fmax(ra, sa[i]) : ra + sa[i];
            rb += sb[i];
        }
        out[0] = ra;
        out[1] = rb;
    }
}

// zero amplitudes whose bit k != outcome, scale the rest (measure collapse, statevector.py:305-307)
__global__ void collapse_kernel(double2 *psi, uint64_t size, int k, int outcome, double scale) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        const double2 x = psi[i];
        if (k >= 0 && (int)((i >> k) & 1) != outcome) psi[i] = make_double2(0.0, 0.0);
        else psi[i] = make_double2(x.x * scale, x.y * scale);
    }
}

// probability histogram over m qubits (first listed = MSB); small tables in shared memory
__global__ void __launch_bounds__(256) pmeasure_kernel(const double2 *__restrict__ psi, uint64_t size, int m,
                                                       const int *__restrict__ qubits, double *partial) {
    extern __shared__ double hist[];
    const int bins = 1 << m;
    for (int b = threadIdx.x; b < bins; b += blockDim.x) hist[b] = 0.0;
    __syncthreads();
    int q[16];
    for (int p = 0; p < m; ++p) q[p] = qubits[p];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        const double2 x = psi[i];
        uint32_t key = 0;
        for (int p = 0; p < m; ++p) key |= (uint32_t)((i >> q[p]) & 1) << (m - 1 - p);
        atomicAdd(&hist[key], fma(x.x, x.x, x.y * x.y));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += blockDim.x) partial[(size_t)blockIdx.x * bins + b] = hist[b];
}

// small tables (<= 16 bins): per-thread register bins (no shared-memory
// atomics on a handful of addresses), fixed-order block and grid sums
struct QubitList {
    int q[16];
};

template <int M>
__global__ void __launch_bounds__(256) pmeasure_small_kernel(const double2 *__restrict__ psi, uint64_t size,
                                                             QubitList qubits, double *partial) {
    constexpr int B = 1 << M;
    double acc[B];
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = 0.0;
    int q[M];
#pragma unroll
    for (int p = 0; p < M; ++p) q[p] = qubits.q[p];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        const double2 x = psi[i];
        const double pr = fma(x.x, x.x, x.y * x.y);
        uint32_t key = 0;
#pragma unroll
        for (int p = 0; p < M; ++p) key |= (uint32_t)((i >> q[p]) & 1) << (M - 1 - p);
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] += key == (uint32_t)b ? pr : 0.0;
    }
    __shared__ double red[B][256 / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        double v = acc[b];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[b][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < B) {
        double s = 0.0;
        for (int w = 0; w < 256 / 32; ++w) s += red[threadIdx.x][w];
        partial[(size_t)blockIdx.x * B + threadIdx.x] = s;
    }
}

// Pauli string phase * X^x Z^z (Z first): out[i] = phase * (-1)^popc((i^x)&z) * in[i^x],
// in place over pairs {i, i^x} (noisy trajectories: errors moved to pass boundaries)
__global__ void pauli_kernel(double2 *__restrict__ psi, uint64_t size, uint64_t x, uint64_t z, double pre,
                             double pim) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t hi = x ? (1ull << (63 - __clzll((long long)x))) : 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        if (x && (i & hi)) continue;  // the partner handles the pair
        const uint64_t j = i ^ x;
        const double2 a = psi[i], b = psi[j];
        const double si = (__popcll(i & z) & 1) ? -1.0 : 1.0, sj = (__popcll(j & z) & 1) ? -1.0 : 1.0;
        // out[i] = phase * s(j) * in[j]; out[j] = phase * s(i) * in[i]
        const double2 bi = make_double2(sj * b.x, sj * b.y), aj = make_double2(si * a.x, si * a.y);
        psi[i] = make_double2(pre * bi.x - pim * bi.y, pre * bi.y + pim * bi.x);
        if (x) psi[j] = make_double2(pre * aj.x - pim * aj.y, pre * aj.y + pim * aj.x);
    }
}

// small tables: one 256-thread block per bin sums the per-block partials in a
// fixed order (strided per thread, then a fixed tree) - deterministic
__global__ void __launch_bounds__(256) pmeasure_finish_small(const double *partial, int n_blocks, int bins,
                                                             double *table) {
    __shared__ double red[256];
    const int b = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < n_blocks; i += 256) s += partial[(size_t)i * bins + b];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) table[b] = red[0];
}

__global__ void pmeasure_finish(const double *partial, int n_blocks, int bins, double *table) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= bins) return;
    double s = 0.0;
    for (int i = 0; i < n_blocks; ++i) s += partial[(size_t)i * bins + b];
    table[b] = s;
}

// large tables (m > 12): scatter with global atomics
__global__ void pmeasure_global_kernel(const double2 *__restrict__ psi, uint64_t size, int m,
                                       const int *__restrict__ qubits, double *table) {
    int q[64];
    for (int p = 0; p < m; ++p) q[p] = qubits[p];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
        const double2 x = psi[i];
        uint64_t key = 0;
        for (int p = 0; p < m; ++p) key |= ((i >> q[p]) & 1) << (m - 1 - p);
        atomicAdd(&table[key], fma(x.x, x.x, x.y * x.y));
    }
}

// reduced density matrix of nq in {1,2} qubits: rho[r][c] = sum_groups x_r conj(x_c)
template <int D>
__global__ void __launch_bounds__(256) rdm_kernel(const double2 *__restrict__ psi, uint64_t n_groups, int qa, int qb,
                                                  int ins0, int ins1, double *partial) {
    double acc[2 * D * D];
#pragma unroll
    for (int k = 0; k < 2 * D * D; ++k) acc[k] = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_groups; g += stride) {
        uint64_t i = insert_zero(g, ins0);
        if (D == 4) i = insert_zero(i, ins1);
        double2 x[D];
        if (D == 2) {
            x[0] = psi[i];
            x[1] = psi[i | (1ull << qa)];
        } else {
            const uint64_t a = 1ull << qa, b = 1ull << qb;
            x[0] = psi[i];
            x[1] = psi[i | b];
            x[2] = psi[i | a];
            x[3] = psi[i | a | b];
        }
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int c = 0; c < D; ++c) {
                // x_r * conj(x_c)
                acc[2 * (r * D + c)] = fma(x[r].x, x[c].x, fma(x[r].y, x[c].y, acc[2 * (r * D + c)]));
                acc[2 * (r * D + c) + 1] = fma(x[r].y, x[c].x, fma(-x[r].x, x[c].y, acc[2 * (r * D + c) + 1]));
            }
    }
    __shared__ double red[32][2 * D * D];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 2 * D * D; ++k) {
        const double v = warp_sum(acc[k]);
        if (l == 0) red[w][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * D * D) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i][threadIdx.x];
        partial[(size_t)blockIdx.x * 2 * D * D + threadIdx.x] = s;
    }
}

__global__ void rdm_finish(const double *partial, int n_blocks, int vals, double *out) {
    const int k = threadIdx.x;
    if (k >= vals) return;
    double s = 0.0;
    for (int i = 0; i < n_blocks; ++i) s += partial[(size_t)i * vals + k];
    out[k] = s;
}

// ---------------------------------------------------------------------------
// batched noisy trajectories (statevector.py:343-357 / noise.py:188-222 per trajectory):
// B trajectories are consecutive 2^nsub-amplitude blocks of one state (block b = blockIdx.y).
// One launch applies every trajectory's own dense gate U_b K_c(b) / sqrt(p) on the gate
// qubits, then accumulates that trajectory's reduced density of the NEXT noisy gate's qubits
// (its branch weights), so a noisy gate costs one HBM pass, not a weight sweep + an apply.
// Union qubits uq[0..NU) ascending; gate / next qubits are given as positions in the union
// (first listed = MSB).
// ---------------------------------------------------------------------------
struct NoisyArgs {
    int nsub;      // qubits per trajectory
    int uq[4];     // union of gate + next qubits, ascending
    int gk, nk;    // gate / next qubit counts (0..2)
    int gpos[2];   // union positions of the gate qubits, MSB first
    int npos[2];   // union positions of the next qubits, MSB first
};

// the per-trajectory matrix is re-read from shared memory (broadcast) at each use: volatile
// keeps the compiler from hoisting all 16 entries into registers, which would cap occupancy
__device__ __forceinline__ double2 vld(const volatile double2 *m, int k) { return make_double2(m[k].x, m[k].y); }

template <int NU, int P>
__device__ __forceinline__ void noisy_mat1_at(double2 (&x)[1 << NU], const volatile double2 *m) {
#pragma unroll
    for (int l = 0; l < (1 << NU); ++l) {
        if ((l >> P) & 1) continue;
        const double2 x0 = x[l], x1 = x[l | (1 << P)];
        x[l] = cdot2(vld(m, 0), x0, vld(m, 1), x1);
        x[l | (1 << P)] = cdot2(vld(m, 2), x0, vld(m, 3), x1);
    }
}

template <int NU, int PA, int PB>
__device__ __forceinline__ void noisy_mat2_at(double2 (&x)[1 << NU], const volatile double2 *m) {
    if constexpr (PA != PB && PA < NU && PB < NU) {
#pragma unroll
        for (int l = 0; l < (1 << NU); ++l) {
            if (((l >> PA) & 1) || ((l >> PB) & 1)) continue;
            const int idx[4] = {l, l | (1 << PB), l | (1 << PA), l | (1 << PA) | (1 << PB)};
            double2 y[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) y[c] = x[idx[c]];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double2 p = cdot2(vld(m, 4 * r), y[0], vld(m, 4 * r + 1), y[1]);
                const double2 q = cdot2(vld(m, 4 * r + 2), y[2], vld(m, 4 * r + 3), y[3]);
                x[idx[r]] = make_double2(p.x + q.x, p.y + q.y);
            }
        }
    }
}

// positions are runtime values but uniform per launch: a switch to compile-time
// instantiations keeps every register index static and lets the compiler allocate
// registers per case (max over cases, not the sum of predicated variants)
template <int NU>
__device__ __forceinline__ void noisy_mat1(double2 (&x)[1 << NU], const volatile double2 *m, int p0) {
    switch (p0) {
        case 0: noisy_mat1_at<NU, 0>(x, m); break;
        case 1: if constexpr (NU > 1) noisy_mat1_at<NU, 1>(x, m); break;
        case 2: if constexpr (NU > 2) noisy_mat1_at<NU, 2>(x, m); break;
        default: if constexpr (NU > 3) noisy_mat1_at<NU, 3>(x, m); break;
    }
}

template <int NU>
__device__ __forceinline__ void noisy_mat2(double2 (&x)[1 << NU], const volatile double2 *m, int p0, int p1) {
    switch (p0 * 4 + p1) {
        case 1: noisy_mat2_at<NU, 0, 1>(x, m); break;
        case 2: noisy_mat2_at<NU, 0, 2>(x, m); break;
        case 3: noisy_mat2_at<NU, 0, 3>(x, m); break;
        case 4: noisy_mat2_at<NU, 1, 0>(x, m); break;
        case 6: noisy_mat2_at<NU, 1, 2>(x, m); break;
        case 7: noisy_mat2_at<NU, 1, 3>(x, m); break;
        case 8: noisy_mat2_at<NU, 2, 0>(x, m); break;
        case 9: noisy_mat2_at<NU, 2, 1>(x, m); break;
        case 11: noisy_mat2_at<NU, 2, 3>(x, m); break;
        case 12: noisy_mat2_at<NU, 3, 0>(x, m); break;
        case 13: noisy_mat2_at<NU, 3, 1>(x, m); break;
        case 14: noisy_mat2_at<NU, 3, 2>(x, m); break;
        default: break;
    }
}

// rho is Hermitian: acc packs row r's diagonal (real) then its upper entries (re, im), D^2 doubles
__host__ __device__ constexpr int herm_index(int r, int c, int D) {
    return r + 2 * (r * (D - 1) - r * (r - 1) / 2) + (c == r ? 0 : 1 + 2 * (c - r - 1));
}

template <int NU, int D, int A>
__device__ __forceinline__ void noisy_rdm_at(const double2 (&x)[1 << NU], double (&acc)[A], int pa, int pb) {
#pragma unroll
    for (int l = 0; l < (1 << NU); ++l) {
        if (((l >> pa) & 1) || (D == 4 && ((l >> pb) & 1))) continue;
        int idx[4];
        if (D == 2) {
            idx[0] = l, idx[1] = l | (1 << pa), idx[2] = idx[3] = l;
        } else {
            idx[0] = l, idx[1] = l | (1 << pb), idx[2] = l | (1 << pa), idx[3] = l | (1 << pa) | (1 << pb);
        }
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int c = r; c < D; ++c) {
                const double2 xr = x[idx[r]], xc = x[idx[c]];
                const int k = herm_index(r, c, D);
                if (c == r) {
                    acc[k] = fma(xr.x, xr.x, fma(xr.y, xr.y, acc[k]));
                } else {  // x_r * conj(x_c)
                    acc[k] = fma(xr.x, xc.x, fma(xr.y, xc.y, acc[k]));
                    acc[k + 1] = fma(xr.y, xc.x, fma(-xr.x, xc.y, acc[k + 1]));
                }
            }
    }
}

template <int NU, int NK>
__device__ __forceinline__ void noisy_rdm(const double2 (&x)[1 << NU], double (&acc)[1 << (2 * NK)], int p0,
                                          int p1) {
    if constexpr (NK == 1) {
        switch (p0) {
            case 0: noisy_rdm_at<NU, 2>(x, acc, 0, 0); break;
            case 1: if constexpr (NU > 1) noisy_rdm_at<NU, 2>(x, acc, 1, 0); break;
            case 2: if constexpr (NU > 2) noisy_rdm_at<NU, 2>(x, acc, 2, 0); break;
            default: if constexpr (NU > 3) noisy_rdm_at<NU, 2>(x, acc, 3, 0); break;
        }
    } else if constexpr (NK == 2) {
#define QSV_RDM2(A_, B_) \
    if constexpr (A_ < NU && B_ < NU) noisy_rdm_at<NU, 4>(x, acc, A_, B_);
        switch (p0 * 4 + p1) {
            case 1: QSV_RDM2(0, 1) break;
            case 2: QSV_RDM2(0, 2) break;
            case 3: QSV_RDM2(0, 3) break;
            case 4: QSV_RDM2(1, 0) break;
            case 6: QSV_RDM2(1, 2) break;
            case 7: QSV_RDM2(1, 3) break;
            case 8: QSV_RDM2(2, 0) break;
            case 9: QSV_RDM2(2, 1) break;
            case 11: QSV_RDM2(2, 3) break;
            case 12: QSV_RDM2(3, 0) break;
            case 13: QSV_RDM2(3, 1) break;
            case 14: QSV_RDM2(3, 2) break;
            default: break;
        }
#undef QSV_RDM2
    }
}

// resident CTAs per SM the register budget is capped for (HBM-bound: occupancy hides latency)
template <int NU, int NK>
constexpr int noisy_min_blocks() { return NU <= 2 ? (NK == 2 ? 2 : 4) : (NU == 3 ? 2 : 1); }

template <int NU, int NK>
__global__ void __launch_bounds__(256, noisy_min_blocks<NU, NK>()) noisy_batch_kernel(double2 *__restrict__ psi, const NoisyArgs a,
                                                          const double2 *__restrict__ mats, double *partial) {
    constexpr int L = 1 << NU;
    constexpr int A = 1 << (2 * NK);  // packed Hermitian block: D^2 doubles
    const uint32_t b = blockIdx.y;
    __shared__ double2 m[16];
    if (threadIdx.x < 16) m[threadIdx.x] = mats[(size_t)b * 16 + threadIdx.x];
    __syncthreads();
    double acc[A];
#pragma unroll
    for (int k = 0; k < A; ++k) acc[k] = 0.0;
    // 32-bit offsets inside this trajectory's block (nsub <= 31): the 2^NU loop-invariant
    // union masks then cost one register each instead of two
    const uint32_t groups = 1u << (a.nsub - NU);
    double2 *__restrict__ pb = psi + ((uint64_t)b << a.nsub);
    uint32_t um[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        uint32_t o = 0;
#pragma unroll
        for (int p = 0; p < NU; ++p)
            if ((l >> p) & 1) o |= 1u << a.uq[p];
        um[l] = o;
    }
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        uint32_t i = g;
#pragma unroll
        for (int p = 0; p < NU; ++p) i = ((i >> a.uq[p]) << (a.uq[p] + 1)) | (i & ((1u << a.uq[p]) - 1));
        double2 x[L];
#pragma unroll
        for (int l = 0; l < L; ++l) x[l] = pb[i | um[l]];
        if (a.gk) {
            if (a.gk == 1)
                noisy_mat1<NU>(x, m, a.gpos[0]);
            else
                noisy_mat2<NU>(x, m, a.gpos[0], a.gpos[1]);
#pragma unroll
            for (int l = 0; l < L; ++l) pb[i | um[l]] = x[l];
        }
        if (NK) noisy_rdm<NU, NK>(x, acc, a.npos[0], a.npos[1]);
    }
    if (!NK) return;
    __shared__ double red[8][A];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < A; ++k) {
        const double v = warp_sum(acc[k]);
        if (l == 0) red[w][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // unpack into the row-major 4x4 complex slot layout: upper triangle + real diagonal of
        // the 2^NK x 2^NK block; every other slot 0 (the host mirrors the lower triangle)
        constexpr int D = 1 << NK;
        const int r = (threadIdx.x >> 1) >> 2, c = (threadIdx.x >> 1) & 3, part = threadIdx.x & 1;
        double s = 0.0;
        if (r < D && c < D && r <= c && !(r == c && part)) {
            const int k = herm_index(r, c, D) + part;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i][k];
        }
        partial[((size_t)b * gridDim.x + blockIdx.x) * 32 + threadIdx.x] = s;
    }
}

// per-trajectory fixed-order sum of the block partials
__global__ void noisy_batch_finish(const double *partial, int n_blocks, int vals, double *out) {
    const uint32_t b = blockIdx.x;
    const int k = threadIdx.x;
    if (k >= vals) return;
    double s = 0.0;
    for (int i = 0; i < n_blocks; ++i) s += partial[((size_t)b * n_blocks + i) * vals + k];
    out[(size_t)b * vals + k] = s;
}

// rows of `len` amplitudes at arbitrary offsets -> one packed buffer (partial-mode recombination)
__global__ void gather_rows_kernel(const double2 *__restrict__ psi, const uint64_t *__restrict__ offs, uint64_t len,
                                   double2 *__restrict__ out) {
    const uint64_t r = blockIdx.y;
    const uint64_t o = offs[r];
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len; k += (uint64_t)gridDim.x * blockDim.x)
        out[r * len + k] = psi[o + k];
}

}  // namespace qsv
