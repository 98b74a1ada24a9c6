// qsv_small.cu -- small-state rotation programs (config 1: 12 q, 1,872 UCC
// rotations in 261 same-flip groups).
//
// The reference applies each rotation as its decomposed gate list
// (statevector.py:65-74 over circuit.py:271-281's pauli_evolution blocks);
// the planner recognises the blocks as exp(-i theta/2 P) (match_block).  For
// a state of <= 12 qubits the tile passes run on ONE SM with straight-line
// code that executes once per warp, so they are bound by instruction fetch
// (profiles/r02_ucc12_compact_ab.txt).  Here the whole program is one CTA
// with the state resident in shared memory, walking the same-flip rotation
// groups with a small loop body: per group, every thread applies the group's
// fused 2x2 matrix to 4 (or 8) pairs (lo, lo ^ xm) that share a config,
// so it loads that matrix once.
//
// Algebra (P = i^ny X^xm Z^zm per string, zm = Y|Z positions, ny = |Y|):
//   P|lo> = i^ny (-1)^(zm.lo) |lo^xm>,  (-1)^(zm.hi) = (-1)^(zm.lo) (-1)^ny,
// so exp(-i theta/2 P) acts on (psi_lo, psi_hi) as
//   [[c, -i s i^ny g sigma (-1)^ny], [-i s i^ny g sigma, c]]
// with g = (-1)^(z0.lo) common to the group and sigma = (-1)^(d.lo) for the
// string's phase-mask difference d = zm ^ z0 (in the span of <= 3 basis
// vectors b_j: sigma is fixed by the 3 parities b_j.lo).  g enters every
// off-diagonal entry, so the fused product is D M D with D = diag(1, g): 16
// matrices per group (8 configs x g).  A pair's config is linear in its pair
// index p, so the pairs p0 ^ span(u) for u in the null space of the four
// parity masks all share p0's config (SmallGroup.lu).  The matrices of a
// chunk of groups are built by the CTA itself at the start of the chunk from
// the raw angles (sincos on device).
//
// Invariant classes: a GF(2) functional w with parity(w & xm) = 0 for every
// flip of the program is conserved by every rotation, so the amplitudes split
// into classes that never mix.  A particle-number-conserving ansatz (UCC
// singles and doubles: even-weight flips) conserves the parity of the index;
// an evolve from a basis state (every energy evaluation) therefore only ever
// touches that state's class -- half of the pairs -- and the other half stays
// exactly zero.  The kernel enumerates the pairs of the reachable classes only.
//
// Bound: shared-memory bandwidth and latency on one SM.  Per group each
// reachable amplitude is read and written once plus one 64-B matrix per
// thread: config 1 (one class of 2,048 amplitudes, 256 threads x 4 pairs)
// 160 us for 261 groups (262 us without the class restriction, 280 us as tile
// passes).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "qsv_internal.h"
#include "qsv_planner.h"

namespace qsv {

// Shared-memory budget per chunk (the state takes 2^n x 16 B <= 64 KiB).
constexpr int kSmallChunkRots = 2048;  // angles: 32 KiB of (cos, sin)
constexpr int kSmallChunkGroups = 80;  // matrices: 80 x 16 configs x 80 B = 100 KiB
constexpr int kRow = 5;                // double2 per matrix row (4 used; 80 B spreads rows over banks)
size_t small_smem_bytes(int n);
static_assert(sizeof(SmallGroup) % 4 == 0, "group records are copied as words");

static inline uint32_t parity32(uint32_t v) { return (uint32_t)__builtin_popcount(v) & 1u; }

bool build_small_program(int n, const std::vector<Rot> &R, SmallProgram &sp)
{
    sp = SmallProgram();
    if (n < kSmallMinQubits || n > kSmallMaxQubits || R.empty()) return false;
    for (const Rot &r : R)
        if ((r.x | r.y) == 0) return false;  // diagonal strings: not handled here
    const uint32_t pmask = (1u << (n - 1)) - 1u;  // pair-index space
    size_t k = 0;
    while (k < R.size()) {
        SmallGroup g{};
        const uint32_t xm = (uint32_t)(R[k].x | R[k].y);
        const uint32_t z0 = (uint32_t)(R[k].y | R[k].z);
        uint32_t b[3] = {0, 0, 0};
        g.xm = xm;
        g.h = 31 - __builtin_clz(xm);
        g.r0 = (int32_t)k;
        int dim = 0;
        size_t e = k;
        for (; e < R.size(); ++e) {
            if ((uint32_t)(R[e].x | R[e].y) != xm) break;
            const uint32_t d = (uint32_t)(R[e].y | R[e].z) ^ z0;
            int coord = -1;
            for (int cbits = 0; cbits < (1 << dim) && coord < 0; ++cbits) {
                uint32_t v = 0;
                for (int j = 0; j < dim; ++j)
                    if ((cbits >> j) & 1) v ^= b[j];
                if (v == d) coord = cbits;
            }
            if (coord < 0) {
                if (dim == 3) break;  // a fourth independent difference: next group
                b[dim] = d;
                coord = 1 << dim;
                ++dim;
            }
            const int ny = __builtin_popcountll(R[e].y);
            sp.meta.push_back((ny & 3) | ((ny & 1) << 2) | (coord << 3));
            sp.src.push_back(R[e].src);
        }
        g.r1 = (int32_t)e;
        g.dimb = dim;
        const uint32_t lowm = (1u << g.h) - 1u;
        const uint32_t ms[4] = {b[0], b[1], b[2], z0};
        for (int j = 0; j < 4; ++j) g.pm[j] = (ms[j] & lowm) | ((ms[j] >> 1) & ~lowm);
        sp.groups.push_back(g);
        k = e;
    }
    // Invariant classes: every functional w with parity(w & xm) = 0 for all
    // flips is conserved by every rotation (a pair lo, lo ^ xm has one value
    // of it), so the 2^n amplitudes split into independent classes.  A
    // particle-number-conserving ansatz (even-weight flips: UCC singles and
    // doubles) conserves the total parity; an evolve from a basis state then
    // only ever touches that state's class -- half the pairs.
    std::vector<uint32_t> flips;
    for (const SmallGroup &g : sp.groups)
        if (std::find(flips.begin(), flips.end(), g.xm) == flips.end()) flips.push_back(g.xm);
    uint32_t W[3] = {0, 0, 0};
    int nw = 0;
    for (uint32_t w = (1u << n) - 1u; w > 0 && nw < 3; --w) {
        bool inv = true;
        for (uint32_t x : flips)
            if (parity32(w & x)) { inv = false; break; }
        if (!inv) continue;
        uint32_t r = w;
        for (int i = 0; i < nw; ++i)
            if ((r >> (31 - __builtin_clz(W[i]))) & 1u) r ^= W[i];
        if (!r) continue;
        const int pv = 31 - __builtin_clz(r);
        for (int i = 0; i < nw; ++i)
            if ((W[i] >> pv) & 1u) W[i] ^= r;
        W[nw++] = r;
    }
    // 4 pairs per thread share a matrix load; classes used: keep >= 32
    // threads busy per class at this n
    int ncls = nw;
    const int share = 2;
    while (ncls > 0 && (n - 1) - ncls - share < 5) --ncls;
    if ((n - 1) - ncls - share < 5) return false;
    sp.ncls = ncls;
    sp.share = share;
    for (int i = 0; i < ncls; ++i) sp.w[i] = W[i];
    for (SmallGroup &g : sp.groups) {
        const uint32_t lowm = (1u << g.h) - 1u;
        uint32_t wp[3] = {0, 0, 0};
        for (int i = 0; i < ncls; ++i) wp[i] = (W[i] & lowm) | ((W[i] >> 1) & ~lowm);
        // share null-space vectors of the four parity masks and the class
        // rows, reduced so each owns its pivot (its highest bit, as high as
        // possible: the thread-to-pair map keeps the low bits consecutive)
        uint32_t u[2] = {0, 0};
        int nu = 0;
        for (uint32_t v = pmask; v > 0 && nu < share; --v) {
            bool in_null = true;
            for (int j = 0; j < 4; ++j) in_null &= parity32(v & g.pm[j]) == 0;
            for (int j = 0; j < ncls; ++j) in_null &= parity32(v & wp[j]) == 0;
            if (!in_null) continue;
            uint32_t r = v;
            for (int i = 0; i < nu; ++i)
                if ((r >> (31 - __builtin_clz(u[i]))) & 1u) r ^= u[i];
            if (!r) continue;
            const int pv = 31 - __builtin_clz(r);  // not an earlier pivot: r is reduced by them
            for (int i = 0; i < nu; ++i)
                if ((u[i] >> pv) & 1u) u[i] ^= r;  // earlier vectors must not carry the new pivot
            u[nu++] = r;
        }
        if (nu < share) return false;
        uint32_t upiv = 0;
        for (int i = 0; i < nu; ++i) {
            upiv |= 1u << (31 - __builtin_clz(u[i]));
            g.lu[i] = (u[i] & lowm) | ((u[i] & ~lowm) << 1);
        }
        // class rows in reduced echelon form over pivots that are not u pivots
        for (int i = 0; i < ncls; ++i) {
            uint32_t r = wp[i], cb = 1u << i;
            for (int j = 0; j < i; ++j)
                if ((r >> g.cpiv[j]) & 1u) { r ^= g.crow[j]; cb ^= g.comb[j]; }
            const uint32_t avail = r & ~upiv;
            if (!avail) return false;
            const int pv = 31 - __builtin_clz(avail);
            for (int j = 0; j < i; ++j)
                if ((g.crow[j] >> pv) & 1u) { g.crow[j] ^= r; g.comb[j] ^= cb; }
            g.crow[i] = r;
            g.comb[i] = cb;
            g.cpiv[i] = pv;
        }
        int nz = 0;
        for (int i = 0; i < nu; ++i) g.zpos[nz++] = 31 - __builtin_clz(u[i]);
        for (int i = 0; i < ncls; ++i) g.zpos[nz++] = g.cpiv[i];
        std::sort(g.zpos, g.zpos + nz);
    }
    // chunks of groups whose angles and matrices fit the shared tables
    int g0 = 0;
    const int ng = (int)sp.groups.size();
    while (g0 < ng) {
        int g1 = g0;
        while (g1 < ng && g1 - g0 < kSmallChunkGroups &&
               sp.groups[g1].r1 - sp.groups[g0].r0 <= kSmallChunkRots)
            ++g1;
        if (g1 == g0) return false;  // one group alone exceeds the table (> 2048 rotations)
        sp.chunks.push_back(g0);
        sp.chunks.push_back(g1);
        g0 = g1;
    }
    sp.valid = true;
    return true;
}

namespace {

// Slot of amplitude l: the low 3 bits (16-B granule within a 128-B row) are
// flipped by bit 3, so any three of the bits 0-3 -- the bits a quarter warp's
// 8 pairs vary once the pivot bit is skipped -- reach 8 distinct granules.
__device__ __forceinline__ uint32_t sslot(uint32_t l) { return l ^ (((l >> 3) & 1u) * 7u); }

__device__ __forceinline__ uint32_t par(uint32_t v) { return (uint32_t)__popc(v) & 1u; }

// i^k * v for a real v
__device__ __forceinline__ double2 ipow(int k, double v)
{
    switch (k & 3) {
        case 0: return make_double2(v, 0.0);
        case 1: return make_double2(0.0, v);
        case 2: return make_double2(-v, 0.0);
        default: return make_double2(0.0, -v);
    }
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c)
{
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// S = log2 pairs per thread sharing one matrix load; 2^(11 - S) threads
constexpr int kMaxThreads = 512;

// One CTA of (pairs in a class) / 2^S threads; per group every thread
// applies the group's matrix for its config to the 2^S pairs p0 ^ span(lu)
// of each class this evolve can reach.  p0 comes from the thread index with
// zeros inserted at the u and class pivots, the class pivots then set so that
// p0 lies in the class.  The chunk's group records sit in shared memory.
template <int S, int NC>
__global__ void __launch_bounds__(kMaxThreads, 1)
small_rot_kernel(double2 *__restrict__ psi, int n, uint64_t basis, const SmallGroup *__restrict__ groups,
                 const int32_t *__restrict__ meta, const double *__restrict__ theta,
                 const int32_t *__restrict__ chunks, int nchunks, uint32_t cls0, uint32_t cls1)
{
    constexpr int kShare = 1 << S;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t dim = 1u << n;
    const uint32_t nthr = blockDim.x;
    double2 *st = reinterpret_cast<double2 *>(smem_raw);  // state
    double2 *cs = st + dim;                               // (cos, sin) of the chunk's angles
    double2 *mt = cs + kSmallChunkRots;                   // [group][16 configs][kRow]
    SmallGroup *gs = reinterpret_cast<SmallGroup *>(mt + 16 * kRow * kSmallChunkGroups);  // the chunk's groups
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < dim; i += nthr)
        st[sslot(i)] = basis != ~0ull ? make_double2(i == basis ? 1.0 : 0.0, 0.0) : psi[i];
    for (int ch = 0; ch < nchunks; ++ch) {
        const int g0 = chunks[2 * ch], g1 = chunks[2 * ch + 1];
        const int rb = groups[g0].r0, re = groups[g1 - 1].r1;
        for (int r = rb + (int)tid; r < re; r += nthr) {
            double s, c;
            sincos(0.5 * theta[r], &s, &c);
            cs[r - rb] = make_double2(c, s);
        }
        {
            const int words = (g1 - g0) * (int)(sizeof(SmallGroup) / 4);
            const uint32_t *src = reinterpret_cast<const uint32_t *>(groups + g0);
            uint32_t *dst = reinterpret_cast<uint32_t *>(gs);
            for (int i = (int)tid; i < words; i += nthr) dst[i] = src[i];
        }
        __syncthreads();  // angles and groups ready; the previous chunk is done with mt
        for (int t = (int)tid; t < (g1 - g0) * 8; t += nthr) {
            const SmallGroup &G = gs[t / 8];
            const uint32_t cfg = (uint32_t)(t & 7);
            if (cfg >= (1u << G.dimb)) continue;
            double2 m00 = make_double2(1.0, 0.0), m01 = make_double2(0.0, 0.0);
            double2 m10 = make_double2(0.0, 0.0), m11 = make_double2(1.0, 0.0);
            for (int r = G.r0; r < G.r1; ++r) {
                const int mk = meta[r];
                const double2 csr = cs[r - rb];
                const double sig = (__popc((uint32_t)(mk >> 3) & cfg) & 1) ? -1.0 : 1.0;
                // off-diagonals: b = -i s i^ny sigma (lo <- hi gets (-1)^ny more)
                const double2 b = ipow((mk & 3) + 3, csr.y * sig);
                const double2 a = (mk & 4) ? make_double2(-b.x, -b.y) : b;
                const double c = csr.x;
                const double2 n00 = cfma(a, m10, make_double2(c * m00.x, c * m00.y));
                const double2 n01 = cfma(a, m11, make_double2(c * m01.x, c * m01.y));
                const double2 n10 = cfma(b, m00, make_double2(c * m10.x, c * m10.y));
                const double2 n11 = cfma(b, m01, make_double2(c * m11.x, c * m11.y));
                m00 = n00; m01 = n01; m10 = n10; m11 = n11;
            }
            double2 *row = mt + ((t / 8) * 16 + (int)cfg) * kRow;
            row[0] = m00; row[1] = m01; row[2] = m10; row[3] = m11;
            row += 8 * kRow;  // g = 1: D M D, D = diag(1, -1)
            row[0] = m00; row[1] = make_double2(-m01.x, -m01.y);
            row[2] = make_double2(-m10.x, -m10.y); row[3] = m11;
        }
        __syncthreads();
        for (int gi = 0; gi < g1 - g0; ++gi) {
            const SmallGroup &G = gs[gi];
            uint32_t q0 = tid;
#pragma unroll
            for (int i = 0; i < S + NC; ++i) {  // zeros at the (ascending) u and class pivots
                const uint32_t lm = (1u << G.zpos[i]) - 1u;
                q0 = ((q0 & ~lm) << 1) | (q0 & lm);
            }
            const uint32_t lowm = (1u << G.h) - 1u, xm = G.xm;
            for (uint32_t cl = cls0; cl < cls1; ++cl) {  // the classes this evolve can reach
                uint32_t p0 = q0;
#pragma unroll
                for (int k = 0; k < NC; ++k)
                    if (par(p0 & G.crow[k]) != par(G.comb[k] & cl)) p0 |= 1u << G.cpiv[k];
                const uint32_t cfg = par(p0 & G.pm[0]) | (par(p0 & G.pm[1]) << 1) | (par(p0 & G.pm[2]) << 2) |
                                     (par(p0 & G.pm[3]) << 3);
                const double2 *M = mt + (gi * 16 + (int)cfg) * kRow;
                const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
                const uint32_t lo0 = ((p0 & ~lowm) << 1) | (p0 & lowm);
                uint32_t lo[kShare];
#pragma unroll
                for (int a = 0; a < kShare; ++a) {
                    uint32_t v = lo0;
#pragma unroll
                    for (int i = 0; i < S; ++i)
                        if ((a >> i) & 1) v ^= G.lu[i];
                    lo[a] = v;
                }
                double2 x[kShare], y[kShare];
#pragma unroll
                for (int a = 0; a < kShare; ++a) {
                    x[a] = st[sslot(lo[a])];
                    y[a] = st[sslot(lo[a] ^ xm)];
                }
#pragma unroll
                for (int a = 0; a < kShare; ++a) {
                    st[sslot(lo[a])] = cfma(m01, y[a], cmul(m00, x[a]));
                    st[sslot(lo[a] ^ xm)] = cfma(m11, y[a], cmul(m10, x[a]));
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = tid; i < dim; i += nthr) psi[i] = st[sslot(i)];
}

template <int NC>
cudaError_t launch_nc(double2 *psi, int n, uint64_t basis, const SmallGroup *groups, const int32_t *meta,
                      const double *theta, const int32_t *chunks, int nchunks, uint32_t c0, uint32_t c1,
                      cudaStream_t st, size_t smem)
{
    static PerDeviceOnce once;
    if (cudaError_t e = once.run([&] {
            return cudaFuncSetAttribute(small_rot_kernel<2, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)small_smem_bytes(kSmallMaxQubits));
        }))
        return e;
    const int threads = std::max(32, std::min(kMaxThreads, ((1 << n) >> 1) >> (2 + NC)));
    small_rot_kernel<2, NC><<<1, threads, smem, st>>>(psi, n, basis, groups, meta, theta, chunks, nchunks, c0, c1);
    return cudaGetLastError();
}

}  // namespace

namespace {

// Parity-reduced states (statevector.ParityReduced): the full n-qubit state
// from the (n-1)-qubit half that holds one invariant class.  dst[j] =
// src[j without its top bit] when parity(j & w) = cls, else 0 (w = all
// ones on the low bits + the top bit).  One coalesced write per amplitude.
__global__ void __launch_bounds__(256) embed_parity_kernel(double2 *__restrict__ dst,
                                                           const double2 *__restrict__ src, uint64_t dim,
                                                           uint64_t wlow, int top, uint32_t cls)
{
    const uint64_t topbit = 1ull << top;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < dim;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t pj = (uint32_t)(__popcll(j & (wlow | topbit)) & 1);
        dst[j] = pj == cls ? src[j & ~topbit] : make_double2(0.0, 0.0);
    }
}

}  // namespace

cudaError_t launch_embed_parity(double2 *dst, const double2 *src, int n_dst, uint64_t wlow, uint32_t cls,
                                int sms, cudaStream_t st)
{
    const uint64_t dim = 1ull << n_dst;
    const uint64_t blocks = std::min<uint64_t>((dim + 255) / 256, (uint64_t)sms * 8);
    embed_parity_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, src, dim, wlow, n_dst - 1, cls);
    return cudaGetLastError();
}

size_t small_smem_bytes(int n)
{
    return ((size_t)16 << n) + 16 * (size_t)kSmallChunkRots + 16 * (size_t)kRow * 16 * kSmallChunkGroups +
           sizeof(SmallGroup) * kSmallChunkGroups;
}

cudaError_t launch_small(double2 *psi, int n, uint64_t basis, const SmallProgram &sp,
                         const SmallGroup *groups, const int32_t *meta, const double *theta,
                         const int32_t *chunks, cudaStream_t st)
{
    // from a basis state only its own class is ever non-zero
    uint32_t c0 = 0, c1 = 1u << sp.ncls;
    if (basis != ~0ull) {
        c0 = 0;
        for (int k = 0; k < sp.ncls; ++k) c0 |= (uint32_t)__builtin_parityll(basis & sp.w[k]) << k;
        c1 = c0 + 1;
    }
    const int nchunks = (int)(sp.chunks.size() / 2);
    const size_t smem = small_smem_bytes(n);
    switch (sp.ncls) {
        case 0: return launch_nc<0>(psi, n, basis, groups, meta, theta, chunks, nchunks, c0, c1, st, smem);
        case 1: return launch_nc<1>(psi, n, basis, groups, meta, theta, chunks, nchunks, c0, c1, st, smem);
        case 2: return launch_nc<2>(psi, n, basis, groups, meta, theta, chunks, nchunks, c0, c1, st, smem);
        default: return launch_nc<3>(psi, n, basis, groups, meta, theta, chunks, nchunks, c0, c1, st, smem);
    }
}

}  // namespace qsv
