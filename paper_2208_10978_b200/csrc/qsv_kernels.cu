// qsv_kernels.cu -- hand-written sm_100a kernels of the state-vector engine.
//
// Every kernel here is HBM-bound or FP64/INT-issue bound; none is a GEMM, so
// no tcgen05 work is involved (FP64 complex arithmetic runs on the DFMA pipe).
//
//  K1/K2  tile_pass_kernel    one HBM pass (read + write of every amplitude)
//                             applying a fused program of dense 1q/2q gates,
//                             permutations, diagonal phases and Pauli-rotation
//                             groups to a 2^m-amplitude tile resident in SMEM.
//                             Replaces the per-gate loops of
//                             _cykernels.pyx:19-73 (apply_1q/apply_2q) driven by
//                             statevector.py:65-74 (evolve).
//  K3     see qsv_expect.cu (batched expectation sweep); here only the
//                             global fallback for flips wider than a tile.
//  K4     apply_pauli_kernel  out (+)= c * P psi  (_cykernels.pyx:76-102,
//                             statevector.py:91-95, 113-121).
//  K5     dot kernels         vdot / norm with a deterministic two-stage
//                             reduction (np.vdot, statevector.py:107, engine.py:75).
//  K6     set_basis_kernel    init_state (statevector.py:42-54).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "qsv_internal.h"

namespace qsv {

namespace {

constexpr int kTileThreads = 256;
constexpr int kRotPairs = 2;                                 // pairs held in registers per rotation sweep
constexpr int kTermChunk = 8;

__device__ __forceinline__ uint32_t insert0(uint32_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1u << b) - 1u));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// m0 * x + m1 * y
__device__ __forceinline__ double2 cmad2(double2 m0, double2 x, double2 m1, double2 y)
{
    double re = fma(m0.x, x.x, fma(-m0.y, x.y, fma(m1.x, y.x, -m1.y * y.y)));
    double im = fma(m0.x, x.y, fma(m0.y, x.x, fma(m1.x, y.y, m1.y * y.x)));
    return make_double2(re, im);
}

__device__ __forceinline__ double2 ldp2(const double *p)
{
    return make_double2(__ldg(p), __ldg(p + 1));
}

// Same load, but volatile so the compiler re-reads it (L1 hit) instead of
// keeping a whole 4x4 complex matrix live in registers across the loop.
__device__ __forceinline__ double2 ldp2_v(const double *p)
{
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// Tile base address: deposit the tile index bits into the complement
// positions.  One lane per complement bit, OR-reduced across the warp.
__device__ __forceinline__ uint64_t tile_base(uint64_t tile, int lane, int ncomp, int comp_lane)
{
    uint64_t bit = (lane < ncomp && ((tile >> lane) & 1ull)) ? (1ull << comp_lane) : 0ull;
    uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)bit);
    uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(bit >> 32));
    return ((uint64_t)hi << 32) | lo;
}

struct TileSmem {
    double2 *amp;      // 2^m amplitudes
    uint64_t *offhi;   // 2^(m-c) offsets of the non-contiguous tile bits
};

// Per-pass geometry tables (built on the host, uploaded with the program):
// offhi[2^(m-c)] offsets of the non-contiguous tile bits, comp[32] the
// physical positions of the tile-index bits.
__device__ __forceinline__ void load_geom(uint64_t *offhi, const uint64_t *g_offhi, int nhi)
{
    for (int i = threadIdx.x; i < nhi; i += blockDim.x) offhi[i] = __ldg(g_offhi + i);
}

// Offset (in amplitudes, relative to the tile base) of local index
// l = threadIdx.x + k*T.  The low c tile bits are the contiguous block.
template <int T>
__device__ __forceinline__ uint64_t tile_off(const uint64_t *offhi, int c, int k)
{
    const uint32_t l = threadIdx.x + k * T;
    return (l & ((1u << c) - 1u)) + offhi[l >> c];
}

template <int T>
__device__ __forceinline__ void load_tile(double2 *sm, const uint64_t *offhi, const double2 *psi,
                                          uint64_t base, int m, int c)
{
    const int per = (1 << m) / T;  // 0 when the tile is smaller than the block
    const double2 *p = psi + base;
    if (per == 0) {
        if ((int)threadIdx.x < (1 << m)) sm[threadIdx.x] = __ldcs(p + tile_off<T>(offhi, c, 0));
        return;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < per; k0 += 4) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < per) v[k] = __ldcs(p + tile_off<T>(offhi, c, k0 + k));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < per) sm[threadIdx.x + (k0 + k) * T] = v[k];
    }
}

template <int T>
__device__ __forceinline__ void store_tile(const double2 *sm, const uint64_t *offhi, double2 *psi,
                                           uint64_t base, int m, int c)
{
    const int per = (1 << m) / T;
    double2 *p = psi + base;
    if (per == 0) {
        if ((int)threadIdx.x < (1 << m)) __stcs(p + tile_off<T>(offhi, c, 0), sm[threadIdx.x]);
        return;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < per; k0 += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < per) __stcs(p + tile_off<T>(offhi, c, k0 + k), sm[threadIdx.x + (k0 + k) * T]);
    }
}

// ---- program ops on the SMEM tile ----------------------------------------

template <int T>
__device__ __forceinline__ void op_u1(double2 *sm, int m, int b, const double *P)
{
    const double2 m00 = ldp2(P), m01 = ldp2(P + 2), m10 = ldp2(P + 4), m11 = ldp2(P + 6);
    const int half = 1 << (m - 1);
#pragma unroll 2
    for (int i = threadIdx.x; i < half; i += T) {
        const uint32_t l0 = insert0(i, b), l1 = l0 | (1u << b);
        const double2 x = sm[l0], y = sm[l1];
        sm[l0] = cmad2(m00, x, m01, y);
        sm[l1] = cmad2(m10, x, m11, y);
    }
}

// 4x4 with rows indexed by 2*bit(a) + bit(b) (circuit.py:5-6, _cykernels.pyx:62-73).
template <int T>
__device__ __forceinline__ void op_u2(double2 *sm, int m, int a, int b, const double *P)
{
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    const int quarter = 1 << (m - 2);
#pragma unroll 1
#pragma unroll 2
    for (int i = threadIdx.x; i < quarter; i += T) {
        const uint32_t l = insert0(insert0(i, lo), hi);
        const uint32_t idx[4] = {l, l | (1u << b), l | (1u << a), l | (1u << a) | (1u << b)};
        double2 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = sm[idx[k]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double *R = P + 8 * r;
            double2 acc = cmad2(ldp2_v(R), x[0], ldp2_v(R + 2), x[1]);
            double2 acc2 = cmad2(ldp2_v(R + 4), x[2], ldp2_v(R + 6), x[3]);
            sm[idx[r]] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
        }
    }
}

template <int T>
__device__ __forceinline__ void op_swap_pairs(double2 *sm, int m, uint32_t fixed, uint32_t i0bit,
                                              uint32_t i1bit, int lo, int hi)
{
    // swap sm[l | fixed | i0bit] <-> sm[l | fixed | i1bit] over quads (lo, hi bits cleared)
    const int quarter = 1 << (m - 2);
#pragma unroll 2
    for (int i = threadIdx.x; i < quarter; i += T) {
        const uint32_t l = insert0(insert0(i, lo), hi) | fixed;
        const uint32_t p = l | i0bit, q = l | i1bit;
        const double2 x = sm[p], y = sm[q];
        sm[p] = y;
        sm[q] = x;
    }
}

template <int T>
__device__ __forceinline__ void op_x(double2 *sm, int m, int b)
{
    const int half = 1 << (m - 1);
#pragma unroll 2
    for (int i = threadIdx.x; i < half; i += T) {
        const uint32_t l0 = insert0(i, b), l1 = l0 | (1u << b);
        const double2 x = sm[l0], y = sm[l1];
        sm[l0] = y;
        sm[l1] = x;
    }
}

template <int T>
__device__ __forceinline__ void op_diag1(double2 *sm, int m, int b, const double *P)
{
    const double2 d0 = ldp2(P), d1 = ldp2(P + 2);
    const int tsize = 1 << m;
#pragma unroll 2
    for (int l = threadIdx.x; l < tsize; l += T) {
        sm[l] = cmul(((l >> b) & 1) ? d1 : d0, sm[l]);
    }
}

// kappa = i^q * s
__device__ __forceinline__ double2 kappa_of(int q, double s)
{
    switch (q & 3) {
        case 0: return make_double2(s, 0.0);
        case 1: return make_double2(0.0, s);
        case 2: return make_double2(-s, 0.0);
        default: return make_double2(0.0, -s);
    }
}

// Group of rotations exp(-i th/2 P) sharing the local flip mask f.  On the
// pair (l0, l1 = l0 ^ f):  a0' = c a0 + kappa sg(l1) a1,  a1' = c a1 + kappa sg(l0) a0
// with kappa = -i * i^{|y|} * sin(th/2) and sg(l) = (-1)^{popc(l & (y|z))}
// (reference P definition: _cykernels.pyx:84-102).
template <int T>
__device__ __forceinline__ void op_rotg(double2 *sm, int m, uint32_t f, int h, const RotRec *rots,
                                        int r0, int r1, uint64_t base)
{
    const int npairs = 1 << (m - 1);
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < npairs; i0 += T * kRotPairs) {
        double2 A[kRotPairs], B[kRotPairs];
        uint32_t L1[kRotPairs];
#pragma unroll
        for (int k = 0; k < kRotPairs; ++k) {
            const int i = i0 + k * T;
            const uint32_t l0 = insert0(i < npairs ? i : 0, h);
            L1[k] = l0 ^ f;
            A[k] = sm[l0];
            B[k] = sm[L1[k]];
        }
        for (int r = r0; r < r1; ++r) {
            const uint64_t s_hi = __ldg(&rots[r].s_hi);
            const uint32_t s_loc = __ldg(&rots[r].s_loc);
            const int q = __ldg(&rots[r].q);
            const double c = __ldg(&rots[r].c), s = __ldg(&rots[r].s);
            const uint32_t tp = __popcll(base & s_hi) & 1u;
            const uint32_t yodd = (q >> 2) & 1u;
            const double2 kap = kappa_of(q, s);
#pragma unroll
            for (int k = 0; k < kRotPairs; ++k) {
                const uint32_t s1 = (__popc(L1[k] & s_loc) & 1u) ^ tp;
                const uint32_t s0 = s1 ^ yodd;
                const double2 k1 = s1 ? make_double2(-kap.x, -kap.y) : kap;
                const double2 k0 = s0 ? make_double2(-kap.x, -kap.y) : kap;
                const double2 a = A[k], b = B[k];
                A[k] = cmad2(make_double2(c, 0.0), a, k1, b);
                B[k] = cmad2(make_double2(c, 0.0), b, k0, a);
            }
        }
#pragma unroll
        for (int k = 0; k < kRotPairs; ++k) {
            const int i = i0 + k * T;
            if (i < npairs) {
                sm[L1[k] ^ f] = A[k];
                sm[L1[k]] = B[k];
            }
        }
    }
}

// Diagonal (Z-only) rotations: a' = (c + kappa sg(l)) a, kappa = -i s.
template <int T>
__device__ __forceinline__ void op_rotd(double2 *sm, int m, const RotRec *rots, int r0, int r1,
                                        uint64_t base)
{
    const int tsize = 1 << m;
#pragma unroll 1
    for (int l0 = threadIdx.x; l0 < tsize; l0 += T * kRotPairs) {
        double2 A[kRotPairs];
#pragma unroll
        for (int k = 0; k < kRotPairs; ++k) {
            const int l = l0 + k * T;
            A[k] = sm[l < tsize ? l : 0];
        }
        for (int r = r0; r < r1; ++r) {
            const uint64_t s_hi = __ldg(&rots[r].s_hi);
            const uint32_t s_loc = __ldg(&rots[r].s_loc);
            const int q = __ldg(&rots[r].q);
            const double c = __ldg(&rots[r].c), s = __ldg(&rots[r].s);
            const uint32_t tp = __popcll(base & s_hi) & 1u;
            const double2 kap = kappa_of(q, s);
#pragma unroll
            for (int k = 0; k < kRotPairs; ++k) {
                const uint32_t l = l0 + k * T;
                const uint32_t sg = (__popc(l & s_loc) & 1u) ^ tp;
                const double2 kk = sg ? make_double2(-kap.x, -kap.y) : kap;
                A[k] = cmul(make_double2(c + kk.x, kk.y), A[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < kRotPairs; ++k) {
            const int l = l0 + k * T;
            if (l < tsize) sm[l] = A[k];
        }
    }
}

template <int T>
__global__ void __launch_bounds__(T, 2) tile_pass_kernel(double2 *__restrict__ psi, const TileDims g,
                                                      const uint64_t *__restrict__ g_offhi,
                                                      const int32_t *__restrict__ g_comp,
                                                      const OpRec *__restrict__ ops, int nops,
                                                      const RotRec *__restrict__ rots,
                                                      const double *__restrict__ params)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sm = reinterpret_cast<double2 *>(smem_raw);
    const int m = g.m, c = g.c;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(sm + (1 << m));
    load_geom(offhi, g_offhi, 1 << (m - c));
    const int lane = threadIdx.x & 31;
    const int comp_lane = __ldg(g_comp + lane);
    __syncthreads();
    const uint64_t ntiles = 1ull << g.ncomp;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t base = tile_base(tile, lane, g.ncomp, comp_lane);
        load_tile<T>(sm, offhi, psi, base, m, c);
        __syncthreads();
        for (int k = 0; k < nops; ++k) {
            const int type = __ldg(&ops[k].type);
            const int a = __ldg(&ops[k].a), b = __ldg(&ops[k].b);
            switch (type) {
                case OP_U1: op_u1<T>(sm, m, a, params + __ldg(&ops[k].p)); break;
                case OP_U2: op_u2<T>(sm, m, a, b, params + __ldg(&ops[k].p)); break;
                case OP_CX: {
                    const int lo = a < b ? a : b, hi = a < b ? b : a;
                    op_swap_pairs<T>(sm, m, 1u << a, 0u, 1u << b, lo, hi);
                    break;
                }
                case OP_SWAP: {
                    const int lo = a < b ? a : b, hi = a < b ? b : a;
                    op_swap_pairs<T>(sm, m, 0u, 1u << a, 1u << b, lo, hi);
                    break;
                }
                case OP_X: op_x<T>(sm, m, a); break;
                case OP_DIAG1: op_diag1<T>(sm, m, a, params + __ldg(&ops[k].p)); break;
                case OP_ROTG:
                    op_rotg<T>(sm, m, __ldg(&ops[k].f), __ldg(&ops[k].h), rots, __ldg(&ops[k].r0),
                               __ldg(&ops[k].r1), base);
                    break;
                case OP_ROTD:
                    op_rotd<T>(sm, m, rots, __ldg(&ops[k].r0), __ldg(&ops[k].r1), base);
                    break;
                default: break;
            }
            __syncthreads();
        }
        store_tile<T>(sm, offhi, psi, base, m, c);
        __syncthreads();
    }
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Column sums of partial[rows][cols] (per-CTA partial sums of a sweep).
// Block = 32 columns (lanes, coalesced) x 32 row slices (warps); each warp
// sums rows r = warp (mod 32), then lane-column partials are added in slice
// order: a fixed summation order, so results are deterministic.
__global__ void __launch_bounds__(1024) reduce_columns_kernel(const double *__restrict__ partial,
                                                              int rows, int cols,
                                                              const int32_t *__restrict__ map,
                                                              double *__restrict__ out)
{
    __shared__ double part[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (t < cols)
        for (int r = warp; r < rows; r += 32) s += partial[(size_t)r * cols + t];
    part[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && t < cols) {
        double v = 0.0;
        for (int w = 0; w < 32; ++w) v += part[w][lane];
        out[map ? map[t] : t] = v;
    }
}

// ---- K4 / K5 / K6 -------------------------------------------------------

__global__ void set_basis_kernel(double2 *__restrict__ psi, uint64_t dim, uint64_t index)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += stride)
        psi[j] = make_double2(j == index ? 1.0 : 0.0, 0.0);
}

// dst[j] (+)= coef * i^{|y|} * (-1)^{popc((j^f) & (y|z))} * src[j^f]
__global__ void apply_pauli_kernel(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                   uint64_t dim, uint64_t flip, uint64_t smask, double2 coef,
                                   int accumulate)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += stride) {
        const uint64_t i = j ^ flip;
        double2 v = cmul(coef, __ldg(src + i));
        if (__popcll(i & smask) & 1) v = make_double2(-v.x, -v.y);
        if (accumulate) {
            const double2 d = dst[j];
            v = make_double2(d.x + v.x, d.y + v.y);
        }
        dst[j] = v;
    }
}

// H|psi> for small states (L2-resident): one kernel over all strings,
// dst[j] = sum_t coef_t (-1)^{popc((j^f_t) & s_t)} src[j ^ f_t] accumulated in
// string order with the per-string kernel's arithmetic (bit-identical to S
// apply_pauli launches).  terms: [f, s] per string, coefs: i^{|y|}-folded.
__global__ void __launch_bounds__(256) apply_operator_small_kernel(
    const double2 *__restrict__ src, double2 *__restrict__ dst, uint64_t dim,
    const uint64_t *__restrict__ fs, const double2 *__restrict__ coefs, int S)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += stride) {
        double2 d = make_double2(0.0, 0.0);
        for (int t = 0; t < S; ++t) {
            const uint64_t i = j ^ __ldg(fs + 2 * t);
            double2 v = cmul(__ldg(coefs + t), __ldg(src + i));
            if (__popcll(i & __ldg(fs + 2 * t + 1)) & 1) v = make_double2(-v.x, -v.y);
            d = t == 0 ? v : make_double2(d.x + v.x, d.y + v.y);
        }
        dst[j] = d;
    }
}

// OP_GMAT tables on the device (the restatement of materialize_gmats,
// qsv_planner.cpp): one thread per (group, flip-pattern configuration)
// multiplies the group's rotations R = [[c, kappa sg1], [kappa sg0, c]],
// kappa = i^q sin, and writes the table for common parity 0 and its
// Z-conjugate for parity 1 at base + dst.
__global__ void gmat_fill_kernel(char *__restrict__ base, const GmatJob *__restrict__ jobs, int njobs,
                                 const double2 *__restrict__ cs, const int32_t *__restrict__ q,
                                 const uint8_t *__restrict__ yF)
{
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = id >> 3, cfg = id & 7;
    if (j >= njobs) return;
    const GmatJob g = jobs[j];
    const int ncfg = 1 << (g.w - 1);
    if (cfg >= ncfg) return;
    uint32_t r1 = 1u << g.H;
    for (int c = 0, b = 0; b < 8; ++b) {  // flip bits ascending, H skipped
        if (!((g.F >> b) & 1) || b == g.H) continue;
        if ((cfg >> c) & 1) r1 |= 1u << b;
        ++c;
    }
    double M[8] = {1, 0, 0, 0, 0, 0, 1, 0};
    for (int r = g.r0; r < g.r1; ++r) {
        const double2 csr = cs[r];
        const int qq = q[r];
        double kre = 0.0, kim = 0.0;
        switch (qq & 3) {
            case 0: kre = csr.y; break;
            case 1: kim = csr.y; break;
            case 2: kre = -csr.y; break;
            default: kim = -csr.y; break;
        }
        const int s1 = __popc(r1 & yF[g.yf + (r - g.r0)]) & 1;
        const int s0 = s1 ^ ((qq >> 2) & 1);
        const double b_re = s1 ? -kre : kre, b_im = s1 ? -kim : kim;
        const double c_re = s0 ? -kre : kre, c_im = s0 ? -kim : kim;
        const double cr = csr.x;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double a0r = M[2 * k], a0i = M[2 * k + 1];
            const double a1r = M[4 + 2 * k], a1i = M[4 + 2 * k + 1];
            M[2 * k] = cr * a0r + (b_re * a1r - b_im * a1i);
            M[2 * k + 1] = cr * a0i + (b_re * a1i + b_im * a1r);
            M[4 + 2 * k] = cr * a1r + (c_re * a0r - c_im * a0i);
            M[4 + 2 * k + 1] = cr * a1i + (c_re * a0i + c_im * a0r);
        }
    }
    double *d0 = reinterpret_cast<double *>(base + g.dst) + 8 * cfg;
    double *d1 = reinterpret_cast<double *>(base + g.dst) + 8 * (ncfg + cfg);
#pragma unroll
    for (int i = 0; i < 8; ++i) d0[i] = M[i];
    d1[0] = M[0];
    d1[1] = M[1];
    d1[2] = -M[2];
    d1[3] = -M[3];
    d1[4] = -M[4];
    d1[5] = -M[5];
    d1[6] = M[6];
    d1[7] = M[7];
}

// mode 0: sum conj(a) b ; mode 1: sum |a|^2 (imag = 0)
template <int T>
__global__ void __launch_bounds__(T) dot_partial_kernel(const double2 *__restrict__ a,
                                                        const double2 *__restrict__ b, uint64_t dim,
                                                        int mode, double *__restrict__ partial)
{
    double re = 0.0, im = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * T;
    for (uint64_t j = (uint64_t)blockIdx.x * T + threadIdx.x; j < dim; j += stride) {
        const double2 x = __ldcs(a + j);
        if (mode == 1) {
            re = fma(x.x, x.x, fma(x.y, x.y, re));
        } else {
            const double2 y = __ldcs(b + j);
            re = fma(x.x, y.x, fma(x.y, y.y, re));
            im = fma(x.x, y.y, fma(-x.y, y.x, im));
        }
    }
    __shared__ double sre[T / 32], sim[T / 32];
    re = warp_sum(re);
    im = warp_sum(im);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sre[warp] = re;
        sim[warp] = im;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0, i = 0.0;
        for (int w = 0; w < T / 32; ++w) {
            r += sre[w];
            i += sim[w];
        }
        partial[2 * blockIdx.x] = r;
        partial[2 * blockIdx.x + 1] = i;
    }
}

__global__ void dot_final_kernel(const double *__restrict__ partial, int nblocks,
                                 double *__restrict__ out2)
{
    // single warp, fixed order: lane-strided partial sums then a fixed shuffle tree
    double re = 0.0, im = 0.0;
    for (int k = threadIdx.x; k < nblocks; k += 32) {
        re += partial[2 * k];
        im += partial[2 * k + 1];
    }
    re = warp_sum(re);
    im = warp_sum(im);
    if (threadIdx.x == 0) {
        out2[0] = re;
        out2[1] = im;
    }
}

__global__ void axpby_kernel(double2 *__restrict__ y, const double2 *__restrict__ x, uint64_t dim,
                             double2 alpha, double2 beta)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += stride) {
        const double2 a = cmul(alpha, y[j]);
        const double2 b = cmul(beta, __ldg(x + j));
        y[j] = make_double2(a.x + b.x, a.y + b.y);
    }
}

// ---- global (non-tile) fallbacks for flips wider than a tile -------------

__device__ __forceinline__ uint64_t insert0_64(uint64_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1ull << b) - 1ull));
}

// Rotation group with an arbitrary flip mask, pairs (j0, j0 ^ flip) over HBM.
__global__ void rot_global_kernel(double2 *__restrict__ psi, uint64_t npairs, uint64_t flip, int h,
                                  const RotRec *__restrict__ rots, int nrot)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
        const uint64_t j0 = insert0_64(i, h), j1 = j0 ^ flip;
        double2 a = psi[j0], b = psi[j1];
        for (int r = 0; r < nrot; ++r) {
            const uint64_t sm = __ldg(&rots[r].s_hi);
            const int q = __ldg(&rots[r].q);
            const double c = __ldg(&rots[r].c), s = __ldg(&rots[r].s);
            const uint32_t s1 = __popcll(j1 & sm) & 1u, s0 = s1 ^ ((q >> 2) & 1u);
            const double2 kap = kappa_of(q, s);
            const double2 k1 = s1 ? make_double2(-kap.x, -kap.y) : kap;
            const double2 k0 = s0 ? make_double2(-kap.x, -kap.y) : kap;
            const double2 na = cmad2(make_double2(c, 0.0), a, k1, b);
            const double2 nb = cmad2(make_double2(c, 0.0), b, k0, a);
            a = na;
            b = nb;
        }
        psi[j0] = a;
        psi[j1] = b;
    }
}

// Flip groups with arbitrary flip masks: per-block per-term partial sums.
template <int T>
__global__ void __launch_bounds__(T) expect_global_kernel(const double2 *__restrict__ psi, int n,
                                                          const GroupRec *__restrict__ groups,
                                                          const uint64_t *__restrict__ gflip,
                                                          int ngroups,
                                                          const TermRec *__restrict__ terms,
                                                          int nterms, double *__restrict__ partial)
{
    __shared__ double red[T / 32][kTermChunk];
    const uint64_t npairs = 1ull << (n - 1);
    const uint64_t stride = (uint64_t)gridDim.x * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int gi = 0; gi < ngroups; ++gi) {
        const uint64_t f = __ldg(&gflip[gi]);
        const int h = __ldg(&groups[gi].h);
        const int t0g = __ldg(&groups[gi].t0), t1g = __ldg(&groups[gi].t1);
        for (int t0 = t0g; t0 < t1g; t0 += kTermChunk) {
            const int nt = min(kTermChunk, t1g - t0);
            uint64_t sl[kTermChunk];
            int ui[kTermChunk];
            double a8[kTermChunk];
#pragma unroll
            for (int k = 0; k < kTermChunk; ++k) {
                sl[k] = k < nt ? __ldg(&terms[t0 + k].s_hi) : 0ull;
                ui[k] = k < nt ? __ldg(&terms[t0 + k].use_im) : 0;
                a8[k] = 0.0;
            }
            for (uint64_t i = (uint64_t)blockIdx.x * T + threadIdx.x; i < npairs; i += stride) {
                const uint64_t j0 = insert0_64(i, h), j1 = j0 ^ f;
                const double2 x = psi[j0], y = psi[j1];
                const double re = fma(x.x, y.x, x.y * y.y);
                const double im = fma(x.x, y.y, -x.y * y.x);
#pragma unroll
                for (int k = 0; k < kTermChunk; ++k) {
                    if (k < nt) {
                        const double v = ui[k] ? im : re;
                        a8[k] += (__popcll(j0 & sl[k]) & 1u) ? -v : v;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kTermChunk; ++k) {
                const double s = warp_sum(a8[k]);
                if (lane == 0) red[warp][k] = s;
            }
            __syncthreads();
            if (threadIdx.x < nt) {
                double s = 0.0;
                for (int w = 0; w < T / 32; ++w) s += red[w][threadIdx.x];
                partial[(size_t)blockIdx.x * nterms + t0 + threadIdx.x] =
                    s * __ldg(&terms[t0 + threadIdx.x].scale);
            }
            __syncthreads();
        }
    }
}

int g_num_sms[64] = {0};

}  // namespace

int elementwise_grid(uint64_t dim, int device)
{
    const uint64_t want = (dim + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms(device) * 8;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

int num_sms(int device)
{
    if (device < 0 || device >= 64) return 148;
    if (!g_num_sms[device]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
            v = 148;
        g_num_sms[device] = v;
    }
    return g_num_sms[device];
}

static size_t tile_smem_bytes(const TileDims &g)
{
    return ((size_t)16 << g.m) + ((size_t)8 << (g.m - g.c));
}

cudaError_t launch_tile_pass(double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                             const int32_t *d_comp, const OpRec *d_ops, int nops,
                             const RotRec *d_rots, const double *d_params, cudaStream_t st)
{
    static PerDeviceOnce once;
    cudaError_t ea = once.run([] {
        return cudaFuncSetAttribute(tile_pass_kernel<kTileThreads>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(((size_t)16 << kMaxTileBits) + 8192));
    });
    if (ea != cudaSuccess) return ea;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = tile_smem_bytes(g);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, tile_pass_kernel<kTileThreads>, kTileThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << g.ncomp;
    const uint64_t cap = (uint64_t)num_sms(dev) * per_sm;
    const int grid = (int)(ntiles < cap ? ntiles : cap);
    tile_pass_kernel<kTileThreads><<<grid, kTileThreads, smem, st>>>(psi, g, d_offhi, d_comp, d_ops,
                                                                     nops, d_rots, d_params);
    return cudaGetLastError();
}

cudaError_t launch_reduce_columns(const double *partial, int rows, int cols, const int32_t *d_map,
                                  double *out, cudaStream_t st)
{
    if (cols <= 0) return cudaSuccess;
    reduce_columns_kernel<<<(cols + 31) / 32, 1024, 0, st>>>(partial, rows, cols, d_map, out);
    return cudaGetLastError();
}

// Relayout chunk swap over peer memory (qsv_dist.cpp): a[i] <-> b[i] for
// i < n, where b may live on another GPU (NVLink / NVSwitch P2P loads and
// stores; the same device when two shards share one).  Each element is read
// once and written once on each side -- no staging copy -- and the two
// devices of a pair each run the swap on one half, so both directions of the
// link and both GPUs' load/store units are busy.  Four 16-B elements per
// thread are in flight before any store (peer latency ~1-2 us).
__global__ void __launch_bounds__(256) swap_chunks_kernel(double2 *__restrict__ a, double2 *__restrict__ b,
                                                          uint64_t n)
{
    constexpr int U = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        double2 va[U], vb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            va[u] = __ldcs(a + i + u * stride);
            vb[u] = __ldcs(b + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            __stcs(a + i + u * stride, vb[u]);
            __stcs(b + i + u * stride, va[u]);
        }
    }
    for (; i < n; i += stride) {
        const double2 va = __ldcs(a + i), vb = __ldcs(b + i);
        __stcs(a + i, vb);
        __stcs(b + i, va);
    }
}

cudaError_t launch_swap_chunks(double2 *a, double2 *b, uint64_t n, int sms, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    const uint64_t want = (n + 255) / 256;
    const int grid = (int)std::min<uint64_t>(want, (uint64_t)sms * 8);
    swap_chunks_kernel<<<grid, 256, 0, st>>>(a, b, n);
    return cudaGetLastError();
}

cudaError_t launch_set_basis(double2 *psi, uint64_t dim, uint64_t index, cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    set_basis_kernel<<<elementwise_grid(dim, dev), 256, 0, st>>>(psi, dim, index);
    return cudaGetLastError();
}

cudaError_t launch_gmat_fill(char *base, const GmatJob *d_jobs, int njobs, const double2 *d_cs,
                             const int32_t *d_q, const uint8_t *d_yF, cudaStream_t st)
{
    if (njobs <= 0) return cudaSuccess;
    const int threads = 8 * njobs;
    gmat_fill_kernel<<<(threads + 127) / 128, 128, 0, st>>>(base, d_jobs, njobs, d_cs, d_q, d_yF);
    return cudaGetLastError();
}

cudaError_t launch_apply_operator_small(const double2 *src, double2 *dst, uint64_t dim,
                                        const uint64_t *d_fs, const double2 *d_coefs, int S,
                                        cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t want = (dim + 255) / 256;
    const int grid = (int)(want ? want : 1);
    apply_operator_small_kernel<<<grid, 256, 0, st>>>(src, dst, dim, d_fs, d_coefs, S);
    return cudaGetLastError();
}

cudaError_t launch_apply_pauli(const double2 *src, double2 *dst, uint64_t dim, uint64_t x,
                               uint64_t y, uint64_t z, double cre, double cim, int accumulate,
                               cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    // fold the global phase i^{|y| mod 4} (_cykernels.pyx:84-94) into the coefficient
    const int wy = __builtin_popcountll(y) & 3;
    double pre = 1.0, pim = 0.0;
    if (wy == 1) { pre = 0.0; pim = 1.0; }
    else if (wy == 2) { pre = -1.0; }
    else if (wy == 3) { pre = 0.0; pim = -1.0; }
    const double2 coef = make_double2(cre * pre - cim * pim, cre * pim + cim * pre);
    apply_pauli_kernel<<<elementwise_grid(dim, dev), 256, 0, st>>>(src, dst, dim, x | y, y | z,
                                                                   coef, accumulate);
    return cudaGetLastError();
}

cudaError_t launch_dot(const double2 *a, const double2 *b, uint64_t dim, double *d_partial,
                       double *d_out2, int mode, cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    int grid = num_sms(dev) * 4;
    const uint64_t want = (dim + 255) / 256;
    if ((uint64_t)grid > want) grid = (int)(want ? want : 1);
    dot_partial_kernel<256><<<grid, 256, 0, st>>>(a, b, dim, mode, d_partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dot_final_kernel<<<1, 32, 0, st>>>(d_partial, grid, d_out2);
    return cudaGetLastError();
}

cudaError_t launch_axpby(double2 *y, const double2 *x, uint64_t dim, double are, double aim,
                         double bre, double bim, cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    axpby_kernel<<<elementwise_grid(dim, dev), 256, 0, st>>>(y, x, dim, make_double2(are, aim),
                                                             make_double2(bre, bim));
    return cudaGetLastError();
}

cudaError_t launch_rot_global(double2 *psi, int n, uint64_t flip, const RotRec *d_rots, int nrot,
                              cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t npairs = 1ull << (n - 1);
    const int h = 63 - __builtin_clzll(flip);
    rot_global_kernel<<<elementwise_grid(npairs, dev), 256, 0, st>>>(psi, npairs, flip, h, d_rots,
                                                                      nrot);
    return cudaGetLastError();
}

int expect_global_grid(int n)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t npairs = 1ull << (n - 1);
    const uint64_t want = (npairs + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms(dev) * 4;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_expect_global(const double2 *psi, int n, const GroupRec *d_groups,
                                 const uint64_t *d_gflip, int ngroups, const TermRec *d_terms,
                                 int nterms, double *d_partial, int *grid_out, cudaStream_t st)
{
    const int grid = expect_global_grid(n);
    *grid_out = grid;
    expect_global_kernel<256><<<grid, 256, 0, st>>>(psi, n, d_groups, d_gflip, ngroups, d_terms,
                                                    nterms, d_partial);
    return cudaGetLastError();
}

}  // namespace qsv
