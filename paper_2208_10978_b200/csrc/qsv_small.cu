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
// off-diagonal entry, so the fused product is D M D with D = diag(1, g): the
// 8 configs' matrices M are built, and g = -1 negates the off-diagonals at use
// (sign-bit XORs).  A pair's config is linear in its pair index p, so the pairs
// lo0 ^ span(lu0, lu1) for lu in the null space of the four parity masks all
// share lo0's config (SmallGroup.lu).  The matrices are built on the device
// from the raw angles (sincos) by builder warps, one run ahead of use.
//
// Warp runs: inside a run of consecutive groups every warp stays in one coset
// of an 8-dimensional subspace holding the run's flips and share vectors, so
// the groups of a run are separated by __syncwarp and only the run's end needs
// a CTA barrier (config 1: 21 barriers instead of 261).  The thread -> pair map
// is a host table (SmallProgram::tab) streamed a few groups ahead by cp.async.
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
// thread (4 pairs): config 1 (one class of 2,048 amplitudes, 256 threads)
// walks 261 groups; history in profiles/r02_ucc12_small.txt.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <array>
#include <cstdlib>

#include "qsv_internal.h"
#include "qsv_planner.h"

namespace qsv {

// Shared-memory budget (the state takes 2^n x 16 B <= 64 KiB).
constexpr int kSmallRunRots = 2048;   // angles of one run: 32 KiB of (cos, sin) + 8 KiB of meta
constexpr int kSmallRunGroups = 48;   // matrices of one run: 48 x 8 configs x 80 B = 30 KiB, double-buffered
                                      // (the group sign g is applied at use: D M D only negates the off-diagonals)
constexpr int kRing = 8;               // table ring slots (per-thread entries of upcoming groups)
constexpr int kAhead = 6;              // table entries in flight ahead of use
constexpr int kRow = 5;                // double2 per matrix row (4 used; 80 B spreads rows over banks)
constexpr uint32_t kSmallRunEnd = 1u << 31;         // xo[4 g + 3]: a CTA barrier follows group g
constexpr size_t kSmallMaxTable = (size_t)16 << 20;  // per-thread table entries (64 MiB)
namespace {

// Small-state expectation (n <= 12: the state is <= 64 KiB and stays in L1):
// one CTA of 256 threads per string (grid-stride over strings).  For a flip
// f != 0 the pairs (i, i ^ f) contribute complex-conjugate terms (P is
// Hermitian), so <P_t> = sum over the lows i (bit h of i = 0) of
// 2 Re(conj(psi_i) i^ny (-1)^{|(i^f) & m|} psi_{i^f}) -- half the elements;
// Z-only strings sum |psi_i|^2 signs over all i.  Each thread keeps two
// independent partial sums (short dependent chains), then a fixed-order
// block reduction (warp shuffles, 8 warp partials in order): deterministic.
// rec[t] = {flip, sign mask, ny mod 4}.  One launch replaces the sweep +
// column-reduction pairs of the general path.
constexpr int kExpT = 256;
__global__ void __launch_bounds__(kExpT) expect_small_kernel(const double2 *__restrict__ psi, uint32_t dim,
                                                             const uint4 *__restrict__ rec, int S,
                                                             double *__restrict__ out)
{
    __shared__ double red[kExpT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < S; t += gridDim.x) {
        const uint4 r = __ldg(rec + t);
        const uint32_t f = r.x, m = r.y, ny = r.z;
        double a0 = 0.0, a1 = 0.0;
        if (f != 0) {
            const int h = 31 - __clz(f);
            const uint32_t lowm = (1u << h) - 1u;
            const uint32_t npairs = dim >> 1;
            for (uint32_t p = threadIdx.x; p < npairs; p += 2 * kExpT) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t q = p + (uint32_t)u * kExpT;
                    if (q >= npairs) break;
                    const uint32_t i = ((q & ~lowm) << 1) | (q & lowm), j = i ^ f;
                    const double2 x = __ldg(psi + i), y = __ldg(psi + j);
                    // Re(i^ny conj(x) y): P = Re conj(x) y, Q = Im conj(x) y
                    double v = (ny & 1) ? fma(x.x, y.y, -x.y * y.x) : fma(x.x, y.x, x.y * y.y);
                    if (ny == 1 || ny == 2) v = -v;
                    if (__popc(j & m) & 1) v = -v;
                    if (u == 0) a0 += v; else a1 += v;
                }
            }
            a0 *= 2.0;
            a1 *= 2.0;
        } else {
            for (uint32_t i = threadIdx.x; i < dim; i += 2 * kExpT) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t k = i + (uint32_t)u * kExpT;
                    if (k >= dim) break;
                    const double2 x = __ldg(psi + k);
                    double v = fma(x.x, x.x, x.y * x.y);
                    if (__popc(k & m) & 1) v = -v;
                    if (u == 0) a0 += v; else a1 += v;
                }
            }
        }
        double acc = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kExpT / 32; ++w) v += red[w];
            out[t] = v;
        }
        __syncthreads();  // red is reused by the next string
    }
}

}  // namespace

cudaError_t launch_expect_small(const double2 *psi, int n, const uint32_t *rec, int S, double *out, int sms,
                                cudaStream_t st)
{
    if (S <= 0) return cudaSuccess;
    const int grid = std::max(1, std::min(S, 8 * sms));
    expect_small_kernel<<<grid, kExpT, 0, st>>>(psi, 1u << n, reinterpret_cast<const uint4 *>(rec), S, out);
    return cudaGetLastError();
}

size_t small_smem_bytes(int n);
static_assert(sizeof(SmallGroup) % 4 == 0, "group records are copied as words");

static inline uint32_t parity32(uint32_t v) { return (uint32_t)__builtin_popcount(v) & 1u; }

// Shared-memory slot of amplitude l: the low 3 bits (16-B granule within a
// 128-B row) are flipped by bit 3, so any three of the bits 0-3 -- the bits a
// quarter warp's 8 pairs vary once the pivot bit is skipped -- reach 8
// distinct granules.  Linear over GF(2): slot(a ^ b) = slot(a) ^ slot(b).
__host__ __device__ __forceinline__ uint32_t small_slot(uint32_t l) { return l ^ (((l >> 3) & 1u) * 7u); }

// The program's slot map: the low 3 bits (16-B granule in a 128-B row) are
// XOR-ed with three parities of the bits >= 3 (masks m[0..2]; small_slot is
// m = {8, 8, 8}).  Linear and an involution; chosen per program so that every
// group's lanes can reach 8 distinct granules per quarter warp.
__host__ __device__ __forceinline__ uint32_t slot3(uint32_t l, uint32_t m0, uint32_t m1, uint32_t m2)
{
#ifdef __CUDA_ARCH__
    const uint32_t g = (__popc(l & m0) & 1u) | ((__popc(l & m1) & 1u) << 1) | ((__popc(l & m2) & 1u) << 2);
#else
    const uint32_t g = (__builtin_popcount(l & m0) & 1u) | ((__builtin_popcount(l & m1) & 1u) << 1) |
                       ((__builtin_popcount(l & m2) & 1u) << 2);
#endif
    return l ^ g;
}

// A GF(2) subspace of small index vectors: basis kept by descending pivot
// (highest bit), so reduce() clears the pivots in order.
struct Gf2Span {
    uint32_t b[32] = {0};
    int d = 0;
    static int piv(uint32_t v) { return 31 - __builtin_clz(v); }
    uint32_t reduce(uint32_t v) const
    {
        for (int i = 0; i < d; ++i)
            if ((v >> piv(b[i])) & 1u) v ^= b[i];
        return v;
    }
    bool contains(uint32_t v) const { return reduce(v) == 0; }
    bool add(uint32_t v)
    {
        const uint32_t r = reduce(v);
        if (!r) return false;
        int i = d++;
        while (i > 0 && piv(b[i - 1]) < piv(r)) { b[i] = b[i - 1]; --i; }
        b[i] = r;
        return true;
    }
    std::vector<uint32_t> elements() const
    {
        std::vector<uint32_t> out(1u << d, 0);
        for (uint32_t m = 1; m < (1u << d); ++m) out[m] = out[m & (m - 1)] ^ b[__builtin_ctz(m)];
        return out;
    }
};

bool build_small_program(int n, const std::vector<Rot> &R, SmallProgram &sp)
{
    sp = SmallProgram();
    if (n < kSmallMinQubits || n > kSmallMaxQubits || R.empty()) return false;
    for (const Rot &r : R)
        if ((r.x | r.y) == 0) return false;  // diagonal strings: not handled here
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
    const int ng = (int)sp.groups.size();
    // Warp runs.  Per class the CTA holds 2^(n - ncls) amplitudes; every
    // group of a run is applied with each warp confined to one coset of an
    // 8-dimensional subspace V of the class (256 amplitudes: 32 lanes x 4
    // pairs) that contains the run's flips and each group's two share
    // vectors, so inside a run a warp only ever touches its own amplitudes
    // and the groups are separated by __syncwarp; one CTA barrier ends the
    // run.  Runs are grown greedily while V stays at <= 8 dimensions and the
    // run's matrices and angles fit their shared-memory buffers (the builder
    // warp prepares run r + 1 while the others apply run r).
    const int dimE = n - ncls;
    std::vector<uint32_t> E;  // the class direction space (functionals vanish)
    for (uint32_t v = 0; v < (1u << n); ++v) {
        bool in = true;
        for (int k = 0; k < ncls; ++k) in &= parity32(v & W[k]) == 0;
        if (in) E.push_back(v);
    }
    uint32_t swz[3] = {8u, 8u, 8u};  // the slot map's masks (see slot3), chosen below
    auto slot = [&](uint32_t v) { return slot3(v, swz[0], swz[1], swz[2]); };
    auto low3 = [&](uint32_t v) { return slot(v) & 7u; };
    // per group: amplitude-space parity masks (bit h free: share vectors have bit h = 0)
    auto in_null = [&](const SmallGroup &G, uint32_t v) {
        if ((v >> G.h) & 1u) return false;
        const uint32_t lowm = (1u << G.h) - 1u;
        for (int j = 0; j < 4; ++j) {
            const uint32_t am = (G.pm[j] & lowm) | ((G.pm[j] & ~lowm) << 1);
            if (parity32(v & am)) return false;
        }
        return true;
    };
    auto share_dim = [&](const Gf2Span &V, const SmallGroup &G) {
        Gf2Span S;
        for (uint32_t e : V.elements())
            if (in_null(G, e)) S.add(e);
        return S;
    };
    sp.nthr = 1 << ((n - 1) - share - ncls);
    const int nwarps = sp.nthr / 32;
    const size_t entries = sp.groups.size() * ((size_t)sp.nthr << ncls);
    if (entries > kSmallMaxTable) return false;
    sp.tab.assign(entries, 0);
    sp.xo.assign(4 * sp.groups.size(), 0);
    std::vector<int> warp_of(1u << n, -1);
    std::vector<Gf2Span> run_V;  // per run: its 8-dimensional subspace
    std::vector<uint32_t> cls_of(1u << n, 0);
    for (uint32_t i = 0; i < (1u << n); ++i)
        for (int k = 0; k < ncls; ++k) cls_of[i] |= parity32(i & W[k]) << k;
    {
        const int c1 = ng;
        int g = 0;
        while (g < c1) {
            if (sp.groups[g].r1 - sp.groups[g].r0 > kSmallRunRots) return false;  // one group's angles exceed the buffer
            Gf2Span V;
            int gg = g;
            for (; gg < c1; ++gg) {
                if (gg - g >= kSmallRunGroups || sp.groups[gg].r1 - sp.groups[g].r0 > kSmallRunRots) break;
                Gf2Span V1 = V;
                V1.add(sp.groups[gg].xm);
                bool ok = V1.d <= 8;
                for (int m = g; m <= gg && ok; ++m) {
                    const SmallGroup &G = sp.groups[m];
                    while (ok && share_dim(V1, G).d < share) {
                        // a vector of the group's null space (in E) not yet in V1,
                        // preferring one that adds a new low slot pattern
                        uint32_t best = 0;
                        int best_score = -1;
                        Gf2Span L;
                        for (uint32_t e : V1.elements()) L.add(low3(e));
                        for (uint32_t e : E) {
                            if (!e || !in_null(G, e) || V1.contains(e)) continue;
                            const int score = L.contains(low3(e)) ? 0 : 1;
                            if (score > best_score) { best = e; best_score = score; }
                            if (best_score == 1) break;
                        }
                        if (best_score < 0 || V1.d >= 8) { ok = false; break; }
                        V1.add(best);
                    }
                }
                if (!ok) break;
                V = V1;
            }
            if (gg == g) return false;  // one group alone: no two share vectors in its class
            // pad V to 8 dimensions inside E, widening its low slot patterns first
            while (V.d < 8) {
                Gf2Span L;
                for (uint32_t e : V.elements()) L.add(low3(e));
                uint32_t best = 0;
                int best_score = -1;
                for (uint32_t e : E) {
                    if (!e || V.contains(e)) continue;
                    const int score = L.contains(low3(e)) ? 0 : 1;
                    if (score > best_score) { best = e; best_score = score; }
                    if (best_score == 1) break;
                }
                if (best_score < 0) return false;
                V.add(best);
            }
            // share vectors: two independent ones of V in each group's null space
            for (int m = g; m < gg; ++m) {
                SmallGroup &G = sp.groups[m];
                const Gf2Span S = share_dim(V, G);
                if (S.d < 2) return false;
                G.lu[0] = S.b[0];
                G.lu[1] = S.b[1];
            }
            run_V.push_back(V);
            sp.runs.push_back(g);
            sp.runs.push_back(gg);
            g = gg;
        }
    }
    // The slot map: every group needs the low slot bits of its pair lows
    // (V minus bit h) to span all 8 granules, so a quarter warp's 8 lanes can
    // take distinct granules (conflict-free 128-bit accesses).  Keep the
    // default map when it already does; else the best of a seeded random
    // search over the masks.
    {
        std::vector<std::array<uint32_t, 7>> vh0(sp.groups.size());
        for (size_t r = 0; r < run_V.size(); ++r)
            for (int m = sp.runs[2 * r]; m < sp.runs[2 * r + 1]; ++m) {
                const Gf2Span &V = run_V[r];
                const int h = sp.groups[m].h;
                int star = -1, k = 0;
                for (int i = 0; i < V.d; ++i)
                    if ((V.b[i] >> h) & 1u) { star = i; break; }
                for (int i = 0; i < V.d; ++i) {
                    if (i == star) continue;
                    vh0[m][k++] = ((V.b[i] >> h) & 1u) ? V.b[i] ^ V.b[star] : V.b[i];
                }
            }
        auto score = [&](const uint32_t msk[3]) {
            int full = 0;
            for (size_t m = 0; m < vh0.size(); ++m) {
                Gf2Span L;
                for (uint32_t v : vh0[m]) L.add(slot3(v, msk[0], msk[1], msk[2]) & 7u);
                full += L.d == 3;
            }
            return full;
        };
        int best = score(swz);
        uint64_t rng = 0x9e3779b97f4a7c15ull;
        const uint32_t hi = ((1u << n) - 1u) & ~7u;
        // bounded one-time search (per structure): <= ~2e7 rank evaluations
        const int iters = (int)std::min<size_t>(4000, (size_t)20000000 / std::max<size_t>(1, 7 * vh0.size()));
        for (int it = 0; it < iters && best < (int)vh0.size(); ++it) {
            uint32_t cand[3];
            for (int j = 0; j < 3; ++j) {
                rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
                cand[j] = (uint32_t)rng & hi;
            }
            const int sc = score(cand);
            if (sc > best) {
                best = sc;
                for (int j = 0; j < 3; ++j) swz[j] = cand[j];
            }
        }
        for (int j = 0; j < 3; ++j) sp.swz[j] = swz[j];
    }
    for (size_t r = 0; r < run_V.size(); ++r) {
        const int g = sp.runs[2 * r], gg = sp.runs[2 * r + 1];
        const Gf2Span &V = run_V[r];
        {
            // warp = coset of V inside the class: enumerate the cosets from
            // each class's smallest index and a complement basis of V in E
            Gf2Span Cs = V;
            std::vector<uint32_t> comp;
            for (uint32_t e : E)
                if (Cs.add(e)) comp.push_back(e);
            if ((int)comp.size() != dimE - 8 || (1 << comp.size()) != nwarps) return false;
            const std::vector<uint32_t> Vel = V.elements();
            for (uint32_t cl = 0; cl < (1u << ncls); ++cl) {
                uint32_t b = 0;
                while (cls_of[b] != cl) ++b;
                for (int a = 0; a < nwarps; ++a) {
                    uint32_t r = b;
                    for (size_t k = 0; k < comp.size(); ++k)
                        if ((a >> k) & 1) r ^= comp[k];
                    for (uint32_t v : Vel) warp_of[r ^ v] = a;
                }
            }
            for (int m = g; m < gg; ++m) {
                SmallGroup &G = sp.groups[m];
                const uint32_t u0 = G.lu[0], u1 = G.lu[1];
                const uint32_t lowm = (1u << G.h) - 1u;
                sp.xo[4 * m + 0] = slot(u0) << 4;
                sp.xo[4 * m + 1] = slot(u1) << 4;
                sp.xo[4 * m + 2] = slot(u0 ^ u1) << 4;
                sp.xo[4 * m + 3] = (slot(G.xm) << 4) | (m == gg - 1 ? kSmallRunEnd : 0u);
                const uint32_t span4[4] = {0, u0, u1, u0 ^ u1};
                for (uint32_t cl = 0; cl < (1u << ncls); ++cl) {
                    std::vector<std::vector<uint32_t>> quads(nwarps);
                    for (uint32_t i = 0; i < (1u << n); ++i) {
                        if (cls_of[i] != cl || ((i >> G.h) & 1u)) continue;
                        if (i != std::min(std::min(i, i ^ u0), std::min(i ^ u1, i ^ u0 ^ u1))) continue;
                        quads[warp_of[i]].push_back(i);
                    }
                    uint32_t *row = sp.tab.data() + (((size_t)m << ncls) | cl) * (size_t)sp.nthr;
                    for (int w = 0; w < nwarps; ++w) {
                        std::vector<uint32_t> &Q = quads[w];
                        if (Q.size() != 32) return false;
                        // lanes in quarters of 8 with distinct low slot
                        // bits (conflict-free 128-bit accesses), greedily
                        std::vector<bool> taken(32, false);
                        for (int qt = 0; qt < 4; ++qt) {
                            uint32_t used = 0;
                            for (int j = 0; j < 8; ++j) {
                                int pick = -1, pick_rep = 0, pick_opts = 99;
                                for (int qi = 0; qi < 32; ++qi) {
                                    if (taken[qi]) continue;
                                    int opts = 0, rep = -1;
                                    for (int a = 0; a < 4; ++a)
                                        if (!((used >> low3(Q[qi] ^ span4[a])) & 1u)) {
                                            ++opts;
                                            if (rep < 0) rep = a;
                                        }
                                    if (opts && opts < pick_opts) { pick = qi; pick_rep = rep; pick_opts = opts; }
                                }
                                if (pick < 0) {  // no free pattern left: accept a conflict
                                    for (int qi = 0; qi < 32 && pick < 0; ++qi)
                                        if (!taken[qi]) pick = qi;
                                    pick_rep = 0;
                                }
                                taken[pick] = true;
                                const uint32_t lo0 = Q[pick] ^ span4[pick_rep];
                                used |= 1u << low3(lo0);
                                const uint32_t p0 = (lo0 & lowm) | ((lo0 >> 1) & ~lowm);
                                const uint32_t cfg = parity32(p0 & G.pm[0]) | (parity32(p0 & G.pm[1]) << 1) |
                                                     (parity32(p0 & G.pm[2]) << 2) | (parity32(p0 & G.pm[3]) << 3);
                                row[w * 32 + qt * 8 + j] = (slot(lo0) << 4) | (cfg << 16);
                            }
                        }
                    }
                }
            }
        }
    }
    sp.valid = true;
    return true;
}

SmallProgram::DevCopy::~DevCopy()
{
    if (!base) return;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return;  // runtime already torn down
    cudaSetDevice(device);
    cudaFree(base);
    cudaSetDevice(cur);
    cudaGetLastError();
}

namespace {

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
// -v when sg = 1 << 31 (sign bits of both parts), else v: integer XORs, no FP64 issue
__device__ __forceinline__ double2 flip_sign(double2 v, uint32_t sg)
{
    return make_double2(__hiloint2double(__double2hiint(v.x) ^ (int)sg, __double2loint(v.x)),
                        __hiloint2double(__double2hiint(v.y) ^ (int)sg, __double2loint(v.y)));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c)
{
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

constexpr int kMaxThreads = 512;
constexpr int kBuilders = 4;  // builder warps (A/B under ncu, config 1: 2 / 4 / 8 -> 151 / 141 / 149 us; with the slot map 4 / 6 / 8 -> 118 / 121 / 127 us)

// One CTA of nthr = (pairs in a class) / 4 compute threads plus kBuilders
// builder warps.  Runs alternate between two shared-memory buffers: while the compute
// warps apply run r (matrices and slot constants in buffer r & 1), the
// builder warps prepare run r + 1 in the other buffer -- angles and meta
// staged from global, sincos, the 8 configs' fused matrices per group -- and
// one CTA barrier per run hands the buffers over.  Per group every compute
// thread applies the group's matrix for its config to the 4 pairs
// lo0 ^ span(lu0, lu1) of each class this evolve can reach; the thread ->
// pair map is the host's table (SmallProgram::tab: first low slot | config
// << 16), streamed kAhead items ahead through a shared-memory ring; the other
// slots are that slot XOR the group's constants (small_slot is linear).
// Inside a run each warp stays in its own coset, so groups are separated by
// __syncwarp only.
template <int NC>
__global__ void __launch_bounds__(kMaxThreads + 32 * kBuilders, 1)
small_rot_kernel(double2 *__restrict__ psi, int n, uint64_t basis, const SmallGroup *__restrict__ groups,
                 const int32_t *__restrict__ meta, const double *__restrict__ theta,
                 const int32_t *__restrict__ runs, int nruns, const uint4 *__restrict__ xo,
                 const uint32_t *__restrict__ tab, uint32_t cls0, uint32_t cls1, uint32_t nthr, uint4 swz)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t dim = 1u << n;
    double2 *st = reinterpret_cast<double2 *>(smem_raw);                       // state
    double2 *mt = st + dim;                                                    // [2][group][8 configs][kRow]
    uint4 *xs = reinterpret_cast<uint4 *>(mt + 2 * 8 * kRow * kSmallRunGroups);  // [2][group] slot XORs
    uint32_t *ring = reinterpret_cast<uint32_t *>(xs + 2 * kSmallRunGroups);    // [kRing][nthr] table entries
    double2 *cs = reinterpret_cast<double2 *>(ring + kRing * kMaxThreads);     // builder: (cos, sin) of a run
    int32_t *ms = reinterpret_cast<int32_t *>(cs + kSmallRunRots);             // builder: meta of a run
    int4 *gr = reinterpret_cast<int4 *>(ms + kSmallRunRots);                   // builder: (r0, r1, dimb) per group
    unsigned char *sb = smem_raw;
    const uint32_t tid = threadIdx.x;
    const bool builder = tid >= nthr;

    // builder warps (kBuilders x 32 threads): matrices + slot constants of
    // run r into buffer r & 1.  All global loads of a run are issued before
    // their uses (group records into shared memory, angles two per thread per
    // step), then the 8 configs x groups matrix chains read shared memory only.
    const uint32_t bt = tid - nthr;  // builder thread index (builders only)
    auto bsync = [] { asm volatile("bar.sync 1, %0;" ::"n"(kBuilders * 32) : "memory"); };
    auto build = [&](int r) {
        const int g0 = __ldg(runs + 2 * r), g1 = __ldg(runs + 2 * r + 1);
        double2 *mb = mt + (r & 1) * 8 * kRow * kSmallRunGroups;
        for (int i = (int)bt; i < g1 - g0; i += kBuilders * 32) {
            const SmallGroup *G = groups + g0 + i;
            gr[i] = make_int4(__ldg(&G->r0), __ldg(&G->r1), __ldg(&G->dimb), 0);
            xs[(r & 1) * kSmallRunGroups + i] = __ldg(xo + g0 + i);
        }
        const int rb = __ldg(&groups[g0].r0), re = __ldg(&groups[g1 - 1].r1);
        constexpr int kB = kBuilders * 32;
        for (int k = rb + (int)bt; k < re; k += 2 * kB) {
            const bool two = k + kB < re;
            const double t0 = __ldg(theta + k), t1 = two ? __ldg(theta + k + kB) : 0.0;
            const int32_t q0 = __ldg(meta + k), q1 = two ? __ldg(meta + k + kB) : 0;
            double s0, c0, s1, c1;
            sincos(0.5 * t0, &s0, &c0);
            sincos(0.5 * t1, &s1, &c1);
            cs[k - rb] = make_double2(c0, s0);
            ms[k - rb] = q0;
            if (two) {
                cs[k + kB - rb] = make_double2(c1, s1);
                ms[k + kB - rb] = q1;
            }
        }
        bsync();
        for (int t = (int)bt; t < (g1 - g0) * 8; t += kB) {
            const int4 G = gr[t / 8];
            const uint32_t cfg = (uint32_t)(t & 7);
            if (cfg >= (1u << G.z)) continue;
            double2 m00 = make_double2(1.0, 0.0), m01 = make_double2(0.0, 0.0);
            double2 m10 = make_double2(0.0, 0.0), m11 = make_double2(1.0, 0.0);
            for (int k = G.x; k < G.y; ++k) {
                const int mk = ms[k - rb];
                const double2 csr = cs[k - rb];
                const double sig = (__popc((uint32_t)(mk >> 3) & cfg) & 1) ? -1.0 : 1.0;
                // off-diagonals: b = -i s i^ny sigma (lo <- hi gets (-1)^ny more)
                const double2 bq = ipow((mk & 3) + 3, csr.y * sig);
                const double2 aq = (mk & 4) ? make_double2(-bq.x, -bq.y) : bq;
                const double c = csr.x;
                const double2 n00 = cfma(aq, m10, make_double2(c * m00.x, c * m00.y));
                const double2 n01 = cfma(aq, m11, make_double2(c * m01.x, c * m01.y));
                const double2 n10 = cfma(bq, m00, make_double2(c * m10.x, c * m10.y));
                const double2 n11 = cfma(bq, m01, make_double2(c * m11.x, c * m11.y));
                m00 = n00; m01 = n01; m10 = n10; m11 = n11;
            }
            double2 *row = mb + t * kRow;  // [group][config]
            row[0] = m00; row[1] = m01; row[2] = m10; row[3] = m11;
        }
        bsync();  // cs / ms / gr are reused by the next build
    };

    // compute threads: the (group, class) items in order; each thread streams
    // its own table entries kAhead items ahead of use (cp.async, one commit
    // group per item; a thread reads only its own ring slots)
    const uint32_t ncl = cls1 - cls0;
    const uint32_t n_items = (uint32_t)runs[2 * nruns - 1] * ncl;
    const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(ring + (builder ? 0 : tid));
    uint32_t f_item = 0, f_g = 0, f_cl = cls0;  // next item to fetch and its (group, class)
    auto fetch = [&]() {
        if (f_item < n_items) {
            const uint32_t *src = tab + (((size_t)f_g << NC) | f_cl) * nthr + tid;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(ring_base + (f_item % kRing) * nthr * 4u),
                         "l"(src));
            if (++f_cl == cls1) {
                f_cl = cls0;
                ++f_g;
            }
        }
        ++f_item;
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (!builder)
        for (int k = 0; k < kAhead; ++k) fetch();
    for (uint32_t i = tid; i < dim; i += blockDim.x)
        st[slot3(i, swz.x, swz.y, swz.z)] = basis != ~0ull ? make_double2(i == basis ? 1.0 : 0.0, 0.0) : psi[i];
    if (builder) build(0);
    __syncthreads();
    uint32_t item = 0;
    for (int r = 0; r < nruns; ++r) {
        if (builder) {
            if (r + 1 < nruns) build(r + 1);
        } else {
            const int g0 = runs[2 * r], g1 = runs[2 * r + 1];
            const double2 *mb = mt + (r & 1) * 8 * kRow * kSmallRunGroups;
            const uint4 *xb = xs + (r & 1) * kSmallRunGroups;
            for (int gi = 0; gi < g1 - g0; ++gi) {
                const uint4 X = xb[gi];
                const uint32_t xh = X.w & 0xffffu;
                for (uint32_t c = 0; c < ncl; ++c) {  // the classes this evolve can reach
                    fetch();
                    asm volatile("cp.async.wait_group %0;\n" ::"n"(kAhead));
                    const uint32_t e = ring[(item % kRing) * nthr + tid];
                    ++item;
                    const double2 *M = mb + (gi * 8 + (int)((e >> 16) & 7u)) * kRow;
                    const uint32_t sg = (e >> 19) << 31;  // g = -1: D M D, D = diag(1, -1)
                    const double2 m00 = M[0], m11 = M[3];
                    const double2 m01 = flip_sign(M[1], sg), m10 = flip_sign(M[2], sg);
                    const uint32_t o0 = e & 0xffffu;
                    const uint32_t lo[4] = {o0, o0 ^ X.x, o0 ^ X.y, o0 ^ X.z};
                    double2 x[4], y[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        x[a] = *reinterpret_cast<const double2 *>(sb + lo[a]);
                        y[a] = *reinterpret_cast<const double2 *>(sb + (lo[a] ^ xh));
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        *reinterpret_cast<double2 *>(sb + lo[a]) = cfma(m01, y[a], cmul(m00, x[a]));
                        *reinterpret_cast<double2 *>(sb + (lo[a] ^ xh)) = cfma(m11, y[a], cmul(m10, x[a]));
                    }
                }
                // inside a run each warp owns its amplitudes: a warp barrier
                if (gi + 1 < g1 - g0) __syncwarp();
            }
        }
        __syncthreads();  // run r applied, run r + 1 built
    }
    for (uint32_t i = tid; i < dim; i += blockDim.x) psi[i] = st[slot3(i, swz.x, swz.y, swz.z)];
}

template <int NC>
cudaError_t launch_nc(double2 *psi, int n, uint64_t basis, const SmallProgram &sp, const SmallGroup *groups,
                      const int32_t *meta, const double *theta, const int32_t *runs, const uint4 *xo,
                      const uint32_t *tab, int nruns, uint32_t c0, uint32_t c1, cudaStream_t st, size_t smem)
{
    static PerDeviceOnce once;
    if (cudaError_t e = once.run([&] {
            return cudaFuncSetAttribute(small_rot_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)small_smem_bytes(kSmallMaxQubits));
        }))
        return e;
    small_rot_kernel<NC><<<1, sp.nthr + 32 * kBuilders, smem, st>>>(psi, n, basis, groups, meta, theta, runs, nruns, xo, tab,
                                                        c0, c1, (uint32_t)sp.nthr,
                                                        make_uint4(sp.swz[0], sp.swz[1], sp.swz[2], 0u));
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
    return ((size_t)16 << n) + 2 * 16 * (size_t)kRow * 8 * kSmallRunGroups + 2 * 16 * (size_t)kSmallRunGroups +
           4 * (size_t)kRing * kMaxThreads + 16 * (size_t)kSmallRunRots + 4 * (size_t)kSmallRunRots +
           16 * (size_t)kSmallRunGroups;
}

cudaError_t launch_small(double2 *psi, int n, uint64_t basis, const SmallProgram &sp,
                         const SmallGroup *groups, const int32_t *meta, const double *theta,
                         const int32_t *runs, const uint32_t *xo, const uint32_t *tab, cudaStream_t st)
{
    // from a basis state only its own class is ever non-zero
    uint32_t c0 = 0, c1 = 1u << sp.ncls;
    if (basis != ~0ull) {
        c0 = 0;
        for (int k = 0; k < sp.ncls; ++k) c0 |= (uint32_t)__builtin_parityll(basis & sp.w[k]) << k;
        c1 = c0 + 1;
    }
    const int nruns = (int)(sp.runs.size() / 2);
    const size_t smem = small_smem_bytes(n);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(xo);
#define QSV_SMALL_LAUNCH(NC) \
    launch_nc<NC>(psi, n, basis, sp, groups, meta, theta, runs, x4, tab, nruns, c0, c1, st, smem)
    switch (sp.ncls) {
        case 0: return QSV_SMALL_LAUNCH(0);
        case 1: return QSV_SMALL_LAUNCH(1);
        case 2: return QSV_SMALL_LAUNCH(2);
        default: return QSV_SMALL_LAUNCH(3);
    }
#undef QSV_SMALL_LAUNCH
}

}  // namespace qsv
