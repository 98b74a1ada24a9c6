// qsv_tile_block.cu -- K1/K2 v2: register-blocked tile pass (sm_100a).
//
// One launch = one HBM pass: every CTA streams 2^m-amplitude tiles (m <= 12,
// 64 KiB) of the state through shared memory and applies a planner-built
// program of *blocks*.  A block names <= 4 tile bits B; each thread gathers
// the 16 amplitudes of one coset of B from SMEM into registers, applies all
// of the block's ops there (dense 1q/2q gates, diagonal phases, same-flip
// Pauli-rotation groups), and scatters them back: one SMEM round trip and
// one barrier per block instead of per gate.  Permutation gates (CNOT, SWAP,
// X) never touch data: the planner folds them into a GF(2)-affine map from
// logical tile index to SMEM slot, and every gather / scatter / store goes
// through that map.  SMEM slots are XOR-swizzled (granule ^= fold3(slot)) so
// the strided coset gathers stay close to conflict-free.
//
// Reference semantics: the per-gate loops of _cykernels.pyx:19-73 driven by
// statevector.py:65-74; Pauli rotations exp(-i t/2 P) with P as in
// _cykernels.pyx:76-102.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qsv_internal.h"

namespace qsv {

namespace {

constexpr int kRB = kBlockBits;              // register bits per block (qsv_internal.h)
constexpr int kR = 1 << kRB;                  // amplitudes per thread
constexpr int kT = (1 << kMaxTileBits) / kR;  // threads per CTA: one coset each
constexpr int kTB = kMaxTileBits - kRB;       // thread-index bits of a full tile

__device__ __forceinline__ uint32_t ins0(uint32_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1u << b) - 1u));
}

// GF(2)-linear swizzle (qsv_internal.h tile_swz).  Bijective on [0, 2^m).
__device__ __forceinline__ uint32_t swz(uint32_t l) { return tile_swz(l); }

__device__ __forceinline__ double2 cfma2(double2 m0, double2 x, double2 m1, double2 y)
{
    double re = fma(m0.x, x.x, fma(-m0.y, x.y, fma(m1.x, y.x, -m1.y * y.y)));
    double im = fma(m0.x, x.y, fma(m0.y, x.x, fma(m1.x, y.y, m1.y * y.x)));
    return make_double2(re, im);
}

__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

// volatile (non-hoistable) variant: re-read from L1 instead of pinning a whole
// 4x4 complex matrix in registers
__device__ __forceinline__ double2 ld2v(const double *p)
{
    double2 v;
    asm volatile("ld.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));  // generic: SMEM or global
    return v;
}

__device__ __forceinline__ uint64_t tbase(uint64_t tile, int lane, int ncomp, int comp_lane)
{
    uint64_t bit = (lane < ncomp && ((tile >> lane) & 1ull)) ? (1ull << comp_lane) : 0ull;
    uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)bit);
    uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(bit >> 32));
    return ((uint64_t)hi << 32) | lo;
}

// ---- register ops on a[16] (block-local bit indices are template args) ----

template <int J>
__device__ __forceinline__ void r_u1(double2 (&a)[kR], const double *P)
{
    const double2 m00 = ld2(P), m01 = ld2(P + 2), m10 = ld2(P + 4), m11 = ld2(P + 6);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        if (r & (1 << J)) continue;
        const double2 x = a[r], y = a[r | (1 << J)];
        a[r] = cfma2(m00, x, m01, y);
        a[r | (1 << J)] = cfma2(m10, x, m11, y);
    }
}

template <int JA, int JB>
__device__ __forceinline__ void r_u2(double2 (&a)[kR], const double *P)
{
    // quad by quad; only the four inputs are copied, each output row goes
    // straight back into a[], matrix rows re-read from SMEM (broadcast LDS)
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        if (r & ((1 << JA) | (1 << JB))) continue;
        const int i00 = r, i01 = r | (1 << JB), i10 = r | (1 << JA), i11 = r | (1 << JA) | (1 << JB);
        const double2 x0 = a[i00], x1 = a[i01], x2 = a[i10], x3 = a[i11];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double *R = P + 8 * k;
            const double2 p = cfma2(ld2v(R), x0, ld2v(R + 2), x1);
            const double2 q = cfma2(ld2v(R + 4), x2, ld2v(R + 6), x3);
            a[k == 0 ? i00 : k == 1 ? i01 : k == 2 ? i10 : i11] = make_double2(p.x + q.x, p.y + q.y);
        }
    }
}

__device__ __forceinline__ double2 cmulc(double2 d, double2 x)
{
    return make_double2(fma(d.x, x.x, -d.y * x.y), fma(d.x, x.y, d.y * x.x));
}

template <int J>
__device__ __forceinline__ void r_diag_in(double2 (&a)[kR], double2 d0, double2 d1)
{
#pragma unroll
    for (int r = 0; r < kR; ++r) a[r] = cmulc((r & (1 << J)) ? d1 : d0, a[r]);
}

// a0' = c a0 + k1 a1 where k1 = +-(i^q s) ; q odd -> imaginary
__device__ __forceinline__ double2 rot_mix(double c, double2 a0, double k, bool imag, double2 a1)
{
    if (imag) return make_double2(fma(c, a0.x, -k * a1.y), fma(c, a0.y, k * a1.x));
    return make_double2(fma(c, a0.x, k * a1.x), fma(c, a0.y, k * a1.y));
}

// Same-flip rotation group on the block-local flip F.  The sign of amplitude
// r is tpar ^ parity(r & sB) ^ thread parity (bits outside the block).
template <int F>
__device__ __forceinline__ void r_rotg(double2 (&a)[kR], const RotRec *rots, int r0, int r1,
                                       uint64_t base, uint32_t tid)
{
    constexpr int H = 31 - __builtin_clz(F);
#pragma unroll 1
    for (int k = r0; k < r1; ++k) {
        const uint64_t s_hi = (rots[k].s_hi);
        const int q = (rots[k].q);
        const double c = (rots[k].c), s = (rots[k].s);
        const uint32_t sB = (q >> 8) & (kR - 1u);
        const uint32_t par = (__popcll(base & s_hi) + __popc(tid & ((uint32_t)q >> 12))) & 1u;
        const uint32_t yodd = (q >> 2) & 1u;
        const bool imag = q & 1;
        const double kk = (q & 2) ? -s : s;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            if (r & (1 << H)) continue;
            const int r1i = r ^ F;
            const uint32_t s1 = par ^ (__popc((uint32_t)r1i & sB) & 1u);
            const uint32_t s0 = s1 ^ yodd;
            const double k1 = s1 ? -kk : kk, k0 = s0 ? -kk : kk;
            const double2 x = a[r], y = a[r1i];
            a[r] = rot_mix(c, x, k1, imag, y);
            a[r1i] = rot_mix(c, y, k0, imag, x);
        }
    }
}

__device__ __forceinline__ void r_rotd(double2 (&a)[kR], const RotRec *rots, int r0, int r1,
                                       uint64_t base, uint32_t tid)
{
#pragma unroll 1
    for (int k = r0; k < r1; ++k) {
        const uint64_t s_hi = (rots[k].s_hi);
        const int q = (rots[k].q);
        const double c = (rots[k].c), s = (rots[k].s);
        const uint32_t sB = (q >> 8) & (kR - 1u);
        const uint32_t par = (__popcll(base & s_hi) + __popc(tid & ((uint32_t)q >> 12))) & 1u;
        // diagonal: a *= c + kappa sg, kappa = -i s (q = 3)
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            const uint32_t sg = par ^ (__popc((uint32_t)r & sB) & 1u);
            const double ks = sg ? s : -s;  // imaginary part of (c - i s sg)
            const double2 x = a[r];
            a[r] = make_double2(fma(c, x.x, -ks * x.y), fma(c, x.y, ks * x.x));
        }
    }
}

__host__ __device__ constexpr int popc_c(int v) { return v ? (v & 1) + popc_c(v >> 1) : 0; }

// index of r1's flip-bit pattern (bits of F except H, compressed ascending);
// folds to a constant inside the unrolled pair loops
template <int F, int H>
__device__ __forceinline__ int cfg_of(int r1)
{
    int out = 0, k = 0;
#pragma unroll
    for (int b = 0; b < kRB; ++b) {
        if (((F >> b) & 1) && b != H) {
            out |= ((r1 >> b) & 1) << k;
            ++k;
        }
    }
    return out;
}

// Fused same-flip group (OP_GMAT): per pair, the product of the group's
// rotations is one 2x2 picked by (common sign parity cp, flip pattern cfg).
template <int F>
__device__ __forceinline__ void r_gmat(double2 (&a)[kR], const double *T, const RotRec *rc,
                                       uint64_t base, uint32_t tid)
{
    constexpr int H = 31 - __builtin_clz(F);
    constexpr int NCFG = 1 << (popc_c(F) - 1);
    const uint64_t s_hi = (rc->s_hi);
    const int q = (rc->q);
    const uint32_t zB = (q >> 8) & (kR - 1u);
    const uint32_t par0 = (__popcll(base & s_hi) + __popc(tid & ((uint32_t)q >> 12))) & 1u;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        if (r & (1 << H)) continue;
        const int r1 = r ^ F;
        const uint32_t cp = par0 ^ (__popc((uint32_t)r1 & zB) & 1u);
        const double *M = T + 8 * ((int)cp * NCFG + cfg_of<F, H>(r1));
        const double2 m00 = ld2(M), m01 = ld2(M + 2), m10 = ld2(M + 4), m11 = ld2(M + 6);
        const double2 x = a[r], y = a[r1];
        a[r] = cfma2(m00, x, m01, y);
        a[r1] = cfma2(m10, x, m11, y);
    }
}

__device__ __forceinline__ void dispatch_gmat(int F, double2 (&a)[kR], const double *T,
                                              const RotRec *rc, uint64_t base, uint32_t tid)
{
    switch (F) {
#define QSV_GMAT_CASE(f) case f: r_gmat<f>(a, T, rc, base, tid); break;
        QSV_GMAT_CASE(1) QSV_GMAT_CASE(2) QSV_GMAT_CASE(3) QSV_GMAT_CASE(4) QSV_GMAT_CASE(5)
        QSV_GMAT_CASE(6) QSV_GMAT_CASE(7)
#if QSV_BLOCK_BITS > 3
        QSV_GMAT_CASE(8) QSV_GMAT_CASE(9) QSV_GMAT_CASE(10)
        QSV_GMAT_CASE(11) QSV_GMAT_CASE(12) QSV_GMAT_CASE(13) QSV_GMAT_CASE(14) QSV_GMAT_CASE(15)
#endif
#undef QSV_GMAT_CASE
        default: break;
    }
}

__device__ __forceinline__ void dispatch_rotg(int F, double2 (&a)[kR], const RotRec *rots, int r0,
                                              int r1, uint64_t base, uint32_t tid)
{
    switch (F) {
#define QSV_ROTG_CASE(f) case f: r_rotg<f>(a, rots, r0, r1, base, tid); break;
        QSV_ROTG_CASE(1) QSV_ROTG_CASE(2) QSV_ROTG_CASE(3) QSV_ROTG_CASE(4) QSV_ROTG_CASE(5)
        QSV_ROTG_CASE(6) QSV_ROTG_CASE(7)
#if QSV_BLOCK_BITS > 3
        QSV_ROTG_CASE(8) QSV_ROTG_CASE(9) QSV_ROTG_CASE(10)
        QSV_ROTG_CASE(11) QSV_ROTG_CASE(12) QSV_ROTG_CASE(13) QSV_ROTG_CASE(14) QSV_ROTG_CASE(15)
#endif
#undef QSV_ROTG_CASE
        default: break;
    }
}

__device__ __forceinline__ void dispatch_u1(int j, double2 (&a)[kR], const double *P)
{
    switch (j) {
        case 0: r_u1<0>(a, P); break;
        case 1: r_u1<1>(a, P); break;
#if QSV_BLOCK_BITS > 3
        case 2: r_u1<2>(a, P); break;
        default: r_u1<3>(a, P); break;
#else
        default: r_u1<2>(a, P); break;
#endif
    }
}

template <template <int, int> class OPW>
__device__ __forceinline__ void dispatch_pair(int ja, int jb, double2 (&a)[kR], const double *P)
{
    switch (ja * 4 + jb) {
        case 1: OPW<0, 1>::run(a, P); break;
        case 2: OPW<0, 2>::run(a, P); break;
        case 4: OPW<1, 0>::run(a, P); break;
        case 6: OPW<1, 2>::run(a, P); break;
        case 8: OPW<2, 0>::run(a, P); break;
        case 9: OPW<2, 1>::run(a, P); break;
#if QSV_BLOCK_BITS > 3
        case 3: OPW<0, 3>::run(a, P); break;
        case 7: OPW<1, 3>::run(a, P); break;
        case 11: OPW<2, 3>::run(a, P); break;
        case 12: OPW<3, 0>::run(a, P); break;
        case 13: OPW<3, 1>::run(a, P); break;
        case 14: OPW<3, 2>::run(a, P); break;
#endif
        default: break;
    }
}

template <int A, int B> struct W_u2 { __device__ static void run(double2 (&a)[kR], const double *P) { r_u2<A, B>(a, P); } };
// OP_U1C: 2x2 on bit A, matrix P (bit B = 0) or P + 8 (bit B = 1)
template <int A, int B> struct W_u1c {
    __device__ static void run(double2 (&a)[kR], const double *P)
    {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            if (r & (1 << A)) continue;
            const double *Q = P + 8 * ((r >> B) & 1);
            const double2 m00 = ld2(Q), m01 = ld2(Q + 2), m10 = ld2(Q + 4), m11 = ld2(Q + 6);
            const double2 x = a[r], y = a[r | (1 << A)];
            a[r] = cfma2(m00, x, m01, y);
            a[r | (1 << A)] = cfma2(m10, x, m11, y);
        }
    }
};

// in-register permutations (block-local bits): CNOT control A target B, SWAP, X
template <int A, int B> struct W_cx {
    __device__ static void run(double2 (&a)[kR], const double *)
    {
#pragma unroll
        for (int r = 0; r < kR; ++r)
            if ((r & (1 << A)) && !(r & (1 << B))) {
                const double2 t = a[r];
                a[r] = a[r | (1 << B)];
                a[r | (1 << B)] = t;
            }
    }
};
template <int A, int B> struct W_swap {
    __device__ static void run(double2 (&a)[kR], const double *)
    {
#pragma unroll
        for (int r = 0; r < kR; ++r)
            if ((r & (1 << A)) && !(r & (1 << B))) {
                const int q = r ^ (1 << A) ^ (1 << B);
                const double2 t = a[r];
                a[r] = a[q];
                a[q] = t;
            }
    }
};
template <int J>
__device__ __forceinline__ void r_x(double2 (&a)[kR])
{
#pragma unroll
    for (int r = 0; r < kR; ++r)
        if (!(r & (1 << J))) {
            const double2 t = a[r];
            a[r] = a[r | (1 << J)];
            a[r | (1 << J)] = t;
        }
}

// Slot of logical tile index l under the block's affine map (kind-1 blocks).
__device__ __forceinline__ uint32_t map_slot(uint32_t l, int m, uint32_t tswz, const uint16_t *cols)
{
    uint32_t o = tswz;
    for (int b = 0; b < m; ++b)
        if ((l >> b) & 1u) o ^= cols[b];
    return o;
}

// Wide-flip rotation group (flip with more than 4 in-tile bits) straight on SMEM.
__device__ void smem_rotg(double2 *sm, int m, uint32_t f, int h, const RotRec *rots, int r0,
                          int r1, uint64_t base, uint32_t tswz, const uint16_t *cols, uint32_t tid)
{
    const int npairs = 1 << (m - 1);
    for (int i = tid; i < npairs; i += kT) {
        const uint32_t l0 = ins0(i, h), l1 = l0 ^ f;
        const uint32_t p0 = map_slot(l0, m, tswz, cols), p1 = map_slot(l1, m, tswz, cols);
        double2 a0 = sm[p0], a1 = sm[p1];
        for (int k = r0; k < r1; ++k) {
            const uint64_t s_hi = (rots[k].s_hi);
            const uint32_t s_loc = (rots[k].s_loc);
            const int q = (rots[k].q);
            const double c = (rots[k].c), s = (rots[k].s);
            const uint32_t s1 = (__popcll(base & s_hi) + __popc(l1 & s_loc)) & 1u;
            const uint32_t s0 = s1 ^ ((q >> 2) & 1u);
            const double kk = (q & 2) ? -s : s;
            const bool imag = q & 1;
            const double2 x = a0, y = a1;
            a0 = rot_mix(c, x, s1 ? -kk : kk, imag, y);
            a1 = rot_mix(c, y, s0 ? -kk : kk, imag, x);
        }
        sm[p0] = a0;
        sm[p1] = a1;
    }
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc)
{
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issue the asynchronous (LDGSTS) loads of one tile into a swizzled SMEM buffer.
__device__ __forceinline__ void issue_tile_load(double2 *buf, const double2 *src, const uint64_t *offhi,
                                                int tsize, int c, uint32_t cmask)
{
#pragma unroll 4
    for (int l = threadIdx.x; l < tsize; l += kT) cp_async16(buf + swz(l), src + (l & cmask) + offhi[l >> c]);
}

// Consumer barrier: BAR = 0 -> whole CTA; otherwise named barrier BAR over
// the kT compute threads (warp-specialised kernel).
template <int BAR>
__device__ __forceinline__ void block_sync(int bar_id)
{
    if (BAR == 0) __syncthreads();
    else if (BAR > 0) asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(kT) : "memory");
    else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kT) : "memory");
}

// Run a pass's register blocks on one SMEM tile (all kT compute threads).
template <bool LITE, int BAR>
__device__ __forceinline__ void run_blocks(double2 *sm, const BlockRec *blocks, int nblocks,
                                           const OpRec *ops, const RotRec *rots,
                                           const double *params, uint64_t base, uint32_t tid, int m,
                                           int bar_id = 0)
{
    const int ncos = (1 << m) >> kRB;  // cosets per block (m >= 4)
    const int tbits = m - kRB;         // thread-index bits of a block
    for (int bi = 0; bi < nblocks; ++bi) {
        const BlockRec *B = blocks + bi;
        const int kind = B->kind;
        const int op0 = B->op0, op1 = B->op1;
        if (kind == 0) {
            if ((int)tid < ncos) {
                uint32_t sb = B->tswz;
                for (int i = 0; i < tbits; ++i)
                    if ((tid >> i) & 1u) sb ^= B->cols[i];
                uint32_t e[kRB];
#pragma unroll
                for (int j = 0; j < kRB; ++j) e[j] = B->cols[kTB + j];
                double2 a[kR];
#pragma unroll
                for (int r = 0; r < kR; ++r) {
                    uint32_t o = 0;
#pragma unroll
                    for (int j = 0; j < kRB; ++j) o ^= ((r >> j) & 1) ? e[j] : 0u;
                    a[r] = sm[sb ^ o];
                }
#pragma unroll 1
                for (int k = op0; k < op1; ++k) {
                    const int4 w0 = reinterpret_cast<const int4 *>(ops + k)[0];
                    const int4 w1 = reinterpret_cast<const int4 *>(ops + k)[1];
                    const int type = w0.x, oa = w0.y, ob = w0.z;
                    switch (type) {
                        case OP_U1: dispatch_u1(oa, a, params + w1.z); break;
                        case OP_U1C: dispatch_pair<W_u1c>(oa, ob, a, params + w1.z); break;
                        case OP_U2:
                            if (!LITE) dispatch_pair<W_u2>(oa, ob, a, params + w1.z);
                            break;
                        case OP_CX: dispatch_pair<W_cx>(oa, ob, a, params); break;
                        case OP_SWAP: dispatch_pair<W_swap>(oa, ob, a, params); break;
                        case OP_X:
                            switch (oa) {
                                case 0: r_x<0>(a); break;
                                case 1: r_x<1>(a); break;
                                case 2: r_x<2>(a); break;
                                default: r_x<3>(a); break;
                            }
                            break;
                        case OP_DIAG1: {
                            const double *P = params + w1.z;
                            const double2 d0 = ld2(P), d1 = ld2(P + 2);
                            if (oa >= 0) {
                                switch (oa) {
                                    case 0: r_diag_in<0>(a, d0, d1); break;
                                    case 1: r_diag_in<1>(a, d0, d1); break;
#if QSV_BLOCK_BITS > 3
                                    case 2: r_diag_in<2>(a, d0, d1); break;
                                    default: r_diag_in<3>(a, d0, d1); break;
#else
                                    default: r_diag_in<2>(a, d0, d1); break;
#endif
                                }
                            } else {
                                const double2 d = ((tid >> ob) & 1u) ? d1 : d0;
#pragma unroll
                                for (int r = 0; r < kR; ++r) a[r] = cmulc(d, a[r]);
                            }
                            break;
                        }
                        case OP_ROTG: dispatch_rotg(w1.w, a, rots, w1.x, w1.y, base, tid); break;
                        case OP_ROTD: r_rotd(a, rots, w1.x, w1.y, base, tid); break;
                        case OP_GMAT:
                            dispatch_gmat(w1.w, a, params + w1.z, rots + w1.x, base, tid);
                            break;
                        default: break;
                    }
                }
#pragma unroll
                for (int r = 0; r < kR; ++r) {
                    uint32_t o = 0;
#pragma unroll
                    for (int j = 0; j < kRB; ++j) o ^= ((r >> j) & 1) ? e[j] : 0u;
                    sm[sb ^ o] = a[r];
                }
            }
        } else if (!LITE) {
            uint16_t cols[12];
#pragma unroll
            for (int b = 0; b < 12; ++b) cols[b] = B->cols[b];
            smem_rotg(sm, m, ops[op0].f, ops[op0].h, rots, ops[op0].r0, ops[op0].r1, base,
                      B->tswz, cols, tid);
        }
        block_sync<BAR>(bar_id);
    }
}

// Persistent CTA (one per SM): double-buffered tiles -- while the register
// blocks run on tile i, the LDGSTS copies of tile i+1 stream into the other
// buffer, so HBM traffic overlaps the DFMA / SMEM work.  g_geo[0..31] are the
// tile-index bit positions, g_geo[32..43] the swizzled columns of the pass's
// final map and g_geo[44] its swizzled translation (used by the store).
// Program of one pass (pass-local indices).  STAGED: copied into shared
// memory once per CTA so every per-tile decode is an LDS.
struct PassProgram {
    const BlockRec *blocks;
    const OpRec *ops;
    const RotRec *rots;
    const double *params;
    int nblocks, nops, nrots, nparams;
};

// LITE: passes without U2 / wide-flip groups -> <= 128 registers, a single
// SMEM tile buffer, two CTAs per SM (16 warps) that overlap each other's
// loads and compute.  Otherwise one CTA per SM with a double-buffered tile.
template <bool STAGED, bool LITE>
__global__ void __launch_bounds__(kT, LITE ? 2 : 1)
tile_block_kernel(double2 *__restrict__ psi, const TileDims g, const uint64_t *__restrict__ g_offhi,
                  const int32_t *__restrict__ g_geo, const PassProgram prog)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NBUF = LITE ? 1 : 2;
    const int m = g.m, c = g.c;
    const int tsize = 1 << m;
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);  // NBUF x tsize
    uint64_t *offhi = reinterpret_cast<uint64_t *>(bufs + NBUF * tsize);
    for (int i = threadIdx.x; i < (1 << (m - c)); i += kT) offhi[i] = __ldg(g_offhi + i);
    const BlockRec *blocks = prog.blocks;
    const OpRec *ops = prog.ops;
    const RotRec *rots = prog.rots;
    const double *params = prog.params;
    const int nblocks = prog.nblocks;
    if (STAGED) {
        // layout after offhi (16 B aligned): params | rots | ops | blocks
        double *sp = reinterpret_cast<double *>(offhi + (1 << (m - c)) + ((1 << (m - c)) & 1));
        RotRec *sr = reinterpret_cast<RotRec *>(sp + ((prog.nparams + 1) & ~1));
        OpRec *so = reinterpret_cast<OpRec *>(sr + prog.nrots);
        BlockRec *sb = reinterpret_cast<BlockRec *>(so + prog.nops);
        for (int i = threadIdx.x; i < prog.nparams; i += kT) sp[i] = __ldg(prog.params + i);
        const int4 *gs = reinterpret_cast<const int4 *>(prog.rots);
        for (int i = threadIdx.x; i < prog.nrots * 2; i += kT) reinterpret_cast<int4 *>(sr)[i] = __ldg(gs + i);
        gs = reinterpret_cast<const int4 *>(prog.ops);
        for (int i = threadIdx.x; i < prog.nops * 2; i += kT) reinterpret_cast<int4 *>(so)[i] = __ldg(gs + i);
        gs = reinterpret_cast<const int4 *>(prog.blocks);
        for (int i = threadIdx.x; i < prog.nblocks * 3; i += kT) reinterpret_cast<int4 *>(sb)[i] = __ldg(gs + i);
        params = sp;
        rots = sr;
        ops = so;
        blocks = sb;
    }
    const uint32_t tid = threadIdx.x;
    const int lane = tid & 31;
    const int comp_lane = __ldg(g_geo + lane);
    const uint32_t cmask = (1u << c) - 1u;
    // store map: slot of logical l = tid + k*kT
    uint32_t st_base = (uint32_t)__ldg(g_geo + 44);
    for (int i = 0; i < kTB && i < m; ++i)
        if ((tid >> i) & 1u) st_base ^= (uint32_t)__ldg(g_geo + 32 + i);
    __syncthreads();
    const uint64_t ntiles = 1ull << g.ncomp;
    uint64_t tile = blockIdx.x;
    if (tile >= ntiles) return;
    uint64_t base = tbase(tile, lane, g.ncomp, comp_lane);
    issue_tile_load(bufs, psi + base, offhi, tsize, c, cmask);
    cp_async_commit();
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        double2 *sm = bufs + (NBUF == 2 ? (it & 1) * tsize : 0);
        const uint64_t next = tile + gridDim.x;
        if (NBUF == 2) {
            if (next < ntiles) {
                const uint64_t nb = tbase(next, lane, g.ncomp, comp_lane);
                issue_tile_load(bufs + ((it + 1) & 1) * tsize, psi + nb, offhi, tsize, c, cmask);
            }
            cp_async_commit();
            cp_async_wait<1>();  // this tile's copies have landed (the next tile's may be in flight)
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        run_blocks<LITE, 0>(sm, blocks, nblocks, ops, rots, params, base, tid, m);
        // ---- store through the pass's final map (streaming STG) ----
        double2 *dst = psi + base;
        if (tsize >= kT) {
#pragma unroll 4
            for (int k = 0; k < (tsize >> kTB); ++k) {
                uint32_t sk = 0;
                for (int j = 0; j < kRB; ++j)
                    if ((k >> j) & 1) sk ^= (uint32_t)__ldg(g_geo + 32 + kTB + j);
                const uint32_t l = tid + k * kT;
                __stcs(dst + (l & cmask) + offhi[l >> c], sm[st_base ^ sk]);
            }
        } else if ((int)tid < tsize) {
            __stcs(dst + (tid & cmask) + offhi[tid >> c], sm[st_base]);
        }
        __syncthreads();
        if (next < ntiles) {
            base = tbase(next, lane, g.ncomp, comp_lane);
            if (NBUF == 1) {  // single buffer: the next tile's load starts after the store
                issue_tile_load(bufs, psi + base, offhi, tsize, c, cmask);
                cp_async_commit();
            }
        }
    }
    cp_async_wait<0>();
}


// ---- mbarrier / async-copy helpers of the ring pipeline ----
constexpr int kStages = 3;

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "QSV_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra QSV_WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *b)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

// ---------------------------------------------------------------------------
// Two-group ring pass (m = 12, no U2 / wide-flip blocks): one persistent CTA
// per SM, 512 threads = two groups of 8 warps at <= 128 registers (the whole
// register file), sharing a 3-stage ring of 64 KiB tiles.  Group g takes the
// CTA's tiles it = g, g+2, ...; tile it lives in stage it % 3.  After
// computing and storing tile it, the group refills that stage with tile it+3
// (which the *other* group will compute), so one tile load is always in
// flight while both groups run FP64 work: HBM streaming overlaps compute.
// Tile it's arrival barrier is full[it % 3 + 3 * ((it / 3) & 1)], completed
// by the 256 noinc cp.async arrivals of the loading group.  Two barriers per
// stage: a group may reach tile it before the other group's tile it - 3 of
// the same stage has landed, or after tile it's own load already landed, and a
// parity wait can only tell the current phase from the previous one -- with
// the barrier reused every 6 tiles (always by the same group) the phase being
// waited on is always the current or the just-completed one.  Each group syncs
// its own blocks on named barrier 1 + g.
constexpr int kRingThreads = 2 * kT;

__device__ __forceinline__ int ring_bar(int it) { return it % kStages + kStages * ((it / kStages) & 1); }

template <bool STAGED>
__global__ void __launch_bounds__(kRingThreads, 1)
tile_ring_kernel(double2 *__restrict__ psi, const TileDims g, const uint64_t *__restrict__ g_offhi,
                 const int32_t *__restrict__ g_geo, const PassProgram prog)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int m = kMaxTileBits;
    constexpr int tsize = 1 << m;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);            // [2 * kStages]
    uint32_t *st_k = reinterpret_cast<uint32_t *>(full + 2 * kStages);  // [16]
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw + 256);        // kStages x tsize
    const int c = g.c;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(bufs + kStages * tsize);
    const int nhi = 1 << (m - c);
    const uint32_t tid_all = threadIdx.x;
    for (int i = tid_all; i < nhi; i += kRingThreads) offhi[i] = __ldg(g_offhi + i);
    const BlockRec *blocks = prog.blocks;
    const OpRec *ops = prog.ops;
    const RotRec *rots = prog.rots;
    const double *params = prog.params;
    if (STAGED) {
        double *sp = reinterpret_cast<double *>(offhi + nhi + (nhi & 1));
        RotRec *sr = reinterpret_cast<RotRec *>(sp + ((prog.nparams + 1) & ~1));
        OpRec *so = reinterpret_cast<OpRec *>(sr + prog.nrots);
        BlockRec *sb = reinterpret_cast<BlockRec *>(so + prog.nops);
        for (int i = tid_all; i < prog.nparams; i += kRingThreads) sp[i] = __ldg(prog.params + i);
        const int4 *gs = reinterpret_cast<const int4 *>(prog.rots);
        for (int i = tid_all; i < prog.nrots * 2; i += kRingThreads) reinterpret_cast<int4 *>(sr)[i] = __ldg(gs + i);
        gs = reinterpret_cast<const int4 *>(prog.ops);
        for (int i = tid_all; i < prog.nops * 2; i += kRingThreads) reinterpret_cast<int4 *>(so)[i] = __ldg(gs + i);
        gs = reinterpret_cast<const int4 *>(prog.blocks);
        for (int i = tid_all; i < prog.nblocks * 3; i += kRingThreads) reinterpret_cast<int4 *>(sb)[i] = __ldg(gs + i);
        params = sp;
        rots = sr;
        ops = so;
        blocks = sb;
    }
    // store map of logical l = tid + kT * k: bits 0..7 from tid, 8..11 from k
    if (tid_all < 16) {
        uint32_t v = 0;
        for (int j = 0; j < 4; ++j)
            if ((tid_all >> j) & 1u) v ^= (uint32_t)__ldg(g_geo + 32 + kTB + j);
        st_k[tid_all] = v;
    }
    if (tid_all == 0) {
        for (int st = 0; st < 2 * kStages; ++st) mbar_init(full + st, kT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint64_t ntiles = 1ull << g.ncomp;
    if ((uint64_t)blockIdx.x >= ntiles) return;
    const int T = (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1;
    const int grp = (int)(tid_all / kT);
    const uint32_t tid = tid_all % kT;
    const int bar_id = 1 + grp;
    const int lane = tid & 31;
    const int comp_lane = __ldg(g_geo + lane);
    const uint32_t cmask = (1u << c) - 1u;
    uint32_t st_base = (uint32_t)__ldg(g_geo + 44);
    for (int i = 0; i < kTB; ++i)
        if ((tid >> i) & 1u) st_base ^= (uint32_t)__ldg(g_geo + 32 + i);

    auto load = [&](int it) {
        const uint64_t tile = blockIdx.x + (uint64_t)it * gridDim.x;
        const uint64_t b = tbase(tile, lane, g.ncomp, comp_lane);
        double2 *buf = bufs + (it % kStages) * tsize;
        const double2 *src = psi + b;
#pragma unroll 4
        for (int k = 0; k < tsize / kT; ++k) {
            const uint32_t l = tid + k * kT;
            cp_async16(buf + swz(l), src + (l & cmask) + offhi[l >> c]);
        }
        cp_async_mbar_arrive(full + ring_bar(it));
    };
    // prologue: group 0 loads tiles 0 and 2, group 1 loads tile 1
    if (grp == 0) {
        load(0);
        if (T > 2) load(2);
    } else if (T > 1) {
        load(1);
    }
    for (int it = grp; it < T; it += 2) {
        const int st = it % kStages;
        const uint64_t tile = blockIdx.x + (uint64_t)it * gridDim.x;
        const uint64_t base = tbase(tile, lane, g.ncomp, comp_lane);
        mbar_wait(full + ring_bar(it), (uint32_t)((it / (2 * kStages)) & 1));
        double2 *sm = bufs + st * tsize;
        run_blocks<true, -1>(sm, blocks, prog.nblocks, ops, rots, params, base, tid, m, bar_id);
        // run_blocks ends with a group barrier: the tile is final in SMEM
        double2 *dst = psi + base;
#pragma unroll 4
        for (int k = 0; k < tsize / kT; ++k) {
            const uint32_t l = tid + k * kT;
            __stcs(dst + (l & cmask) + offhi[l >> c], sm[st_base ^ st_k[k]]);
        }
        if (it + kStages < T) {
            block_sync<-1>(bar_id);  // every thread of the group is done reading stage st
            load(it + kStages);
        }
    }
    cp_async_wait<0>();
}
}  // namespace

cudaError_t launch_tile_blocks(double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                               const int32_t *d_geo, const BlockRec *d_blocks, int nblocks,
                               const OpRec *d_ops, int nops, const RotRec *d_rots, int nrots,
                               const double *d_params, int nparams, bool lite, cudaStream_t st)
{
    static PerDeviceOnce once;
    const int max_smem = 227 * 1024;
    cudaError_t ea = once.run([] {
        cudaError_t e = cudaFuncSetAttribute(tile_block_kernel<true, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(tile_block_kernel<false, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(tile_block_kernel<true, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
    });
    if (ea != cudaSuccess) return ea;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t nhi = (size_t)1 << (g.m - g.c);
    const size_t prog_bytes = 8 * (size_t)((nparams + 1) & ~1) + sizeof(RotRec) * nrots +
                              sizeof(OpRec) * nops + sizeof(BlockRec) * nblocks;
    const size_t lite_base = ((size_t)16 << g.m) + 8 * (nhi + (nhi & 1));
    const size_t full_base = ((size_t)32 << g.m) + 8 * (nhi + (nhi & 1));
    PassProgram prog{d_blocks, d_ops, d_rots, d_params, nblocks, nops, nrots, nparams};
    const uint64_t ntiles = 1ull << g.ncomp;
    static const char *env_grid = getenv("QSV_TILE_GRID");  // debug: cap the persistent grid
    auto grid_for = [&](int per_sm) {
        uint64_t cap = (uint64_t)num_sms(dev) * (per_sm > 0 ? per_sm : 1);
        if (env_grid && atoi(env_grid) > 0) cap = (uint64_t)atoi(env_grid);
        return (int)(ntiles < cap ? ntiles : cap);
    };
    static const char *env_ring = getenv("QSV_TILE_RING");  // 0: disable the ring kernel
    if (lite && g.m == kMaxTileBits && !(env_ring && env_ring[0] == '0')) {
        static PerDeviceOnce ring_once;
        cudaError_t er = ring_once.run([] {
            cudaError_t e = cudaFuncSetAttribute(tile_ring_kernel<true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            if (e != cudaSuccess) return e;
            return cudaFuncSetAttribute(tile_ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024);
        });
        if (er != cudaSuccess) return er;
        const size_t rb = 256 + ((size_t)kStages * 16 << g.m) + 8 * (nhi + (nhi & 1));
        const bool rs = rb + prog_bytes <= (size_t)max_smem;
        const size_t smem = rs ? rb + prog_bytes : rb;
        if (rs)
            tile_ring_kernel<true><<<grid_for(1), kRingThreads, smem, st>>>(psi, g, d_offhi, d_geo, prog);
        else
            tile_ring_kernel<false><<<grid_for(1), kRingThreads, smem, st>>>(psi, g, d_offhi, d_geo, prog);
        return cudaGetLastError();
    }
    // two CTAs per SM need <= ~113 KB each: single tile buffer + staged program
    if (lite && lite_base + prog_bytes <= (size_t)112 * 1024) {
        const size_t smem = lite_base + prog_bytes;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_block_kernel<true, true>, kT, smem);
        tile_block_kernel<true, true><<<grid_for(per_sm), kT, smem, st>>>(psi, g, d_offhi, d_geo, prog);
        return cudaGetLastError();
    }
    const bool staged = full_base + prog_bytes <= (size_t)max_smem;
    const size_t smem = staged ? full_base + prog_bytes : full_base;
    if (staged)
        tile_block_kernel<true, false><<<grid_for(1), kT, smem, st>>>(psi, g, d_offhi, d_geo, prog);
    else
        tile_block_kernel<false, false><<<grid_for(1), kT, smem, st>>>(psi, g, d_offhi, d_geo, prog);
    return cudaGetLastError();
}

}  // namespace qsv
