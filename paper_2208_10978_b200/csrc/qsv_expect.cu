// qsv_expect.cu -- K3 v2: batched Pauli-string expectation sweep (sm_100a).
//
// One launch = one read-only HBM sweep over the state.  Each CTA streams
// 2^m-amplitude tiles through shared memory and evaluates every string of the
// sweep whose flip mask lies inside the tile:
//
//  * flip groups (strings sharing f = x|y): the group's 2^(m-1) amplitude
//    pairs (l0, l0 ^ f) are cut into quarters of 512; one warp takes a
//    quarter, each lane the 16 pair indices lane + 32 r.  A lane forms
//    w = conj(psi_l0) psi_l1 for its 16 pairs, runs a 16-point Walsh-Hadamard
//    transform of Re w / Im w in registers, and every string of the group
//    then costs one shared-memory lookup + one warp reduction instead of a
//    pass over the pairs:
//       <P> over the quarter = scale * sum_lanes (+-) WHT16[s' & 15]
//    with s' the string's sign mask in pair-index coordinates.
//  * Z-only strings: a full in-SMEM WHT of |psi|^2 over the tile, then one
//    lookup per string.
//
// Derivation (reference P, _cykernels.pyx:84-102):  for the pair
// (l0, l1 = l0 ^ f),  <P> contribution = ph sg(l1) (w + eps conj w),
// eps = (-1)^{|y|}, ph = i^{|y|}; sg(l1) = sg(l0) (-1)^{|y|}.  Hence
// |y| even: 2 ph' sg(l0) Re w;  |y| odd: -2 i^{|y|+1} sg(l0) Im w.
// Partial sums go to per-(CTA, string) slots reduced in a fixed order, so
// results are deterministic.
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "qsv_internal.h"

namespace qsv {

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kPer = (1 << kMaxTileBits) / kT;  // amplitudes per thread in load / WHT (16)
constexpr int kSlots = 4;                        // quarters of a full tile's pairs

__device__ __forceinline__ uint32_t ins0(uint32_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1u << b) - 1u));
}

__device__ __forceinline__ uint64_t tbase(uint64_t tile, int lane, int ncomp, int comp_lane)
{
    uint64_t bit = (lane < ncomp && ((tile >> lane) & 1ull)) ? (1ull << comp_lane) : 0ull;
    uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)bit);
    uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(bit >> 32));
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc)
{
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ double wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void wht16(double (&v)[16])
{
#pragma unroll
    for (int b = 1; b < 16; b <<= 1) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            if (r & b) continue;
            const double u = v[r], w = v[r | b];
            v[r] = u + w;
            v[r | b] = u - w;
        }
    }
}

// Strings [t_a, t_b) of one group against the lane's WHT16 vector in scratch.
// The lane's pairs are p = pbase + 32 r (r = 0..15): the WHT runs over pair
// bits 5..8, the lane's own bits enter as a sign.
__device__ __forceinline__ void eval_terms(const double *scr, int lane, uint32_t pbase,
                                           uint64_t base, const TermRec *terms, int t_a, int t_b,
                                           double *acc, int ndiag, int slot)
{
    for (int t = t_a; t < t_b; ++t) {
        const uint32_t sp = __ldg(&terms[t].s_loc);
        const uint64_t s_hi = __ldg(&terms[t].s_hi);
        const uint32_t sg = (__popc(pbase & sp & ~(15u << 5)) + __popcll(base & s_hi)) & 1u;
        const double v = scr[((sp >> 5) & 15u) * 32 + lane];
        const double sum = wsum(sg ? -v : v);
        if (lane == 0) acc[(t - ndiag) * kSlots + slot] += __ldg(&terms[t].scale) * sum;
    }
}

// Position of pair index p (11 bits) inside a 2048-double half of the
// transform scratch: low 4 bits XOR-swizzled by bits 4-7, so every access
// pattern of tile_wht is conflict-free (two wavefronts per warp).
__device__ __forceinline__ int wpos(uint32_t p) { return (int)(p ^ ((p >> 4) & 15u)); }

// Walsh-Hadamard transform of 4096 values held as v[k] = value at index
// threadIdx.x + 256 k.  Index bits 8.. (8 + kbits) run in registers first:
// kbits = 3 keeps bit 11 apart (two independent 2048-point transforms, e.g.
// Re w | Im w), kbits = 4 transforms all 12 bits.  Bits 0-3 and 4-7 then run
// in registers after two transposes through S (4096 doubles, swizzled
// halves).  On return S holds the transform: index i at
// S[(i >> 11) * 2048 + wpos(i & 2047)].
__device__ __forceinline__ void tile_wht(double (&v)[16], int kbits, double *S)
{
    const int t = threadIdx.x;
#pragma unroll
    for (int b = 1; b < 16; b <<= 1) {
        if (b >= (1 << kbits)) break;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            if (r & b) continue;
            const double u = v[r], w = v[r | b];
            v[r] = u + w;
            v[r | b] = u - w;
        }
    }
    __syncthreads();  // S free (previous lookups done)
#pragma unroll
    for (int k = 0; k < 16; ++k) S[(k >> 3) * 2048 + wpos((uint32_t)(t + 256 * (k & 7)))] = v[k];
    __syncthreads();
    double *H = S + (t >> 7) * 2048;
    const uint32_t tp = t & 127;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = H[wpos((tp << 4) | r)];
    wht16(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) H[wpos((tp << 4) | r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = H[wpos((tp & 15u) | (r << 4) | ((tp >> 4) << 8))];
    wht16(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) H[wpos((tp & 15u) | (r << 4) | ((tp >> 4) << 8))] = v[r];
    __syncthreads();
}

__global__ void __launch_bounds__(kT, 1)
expect_sweep2_kernel(const double2 *__restrict__ psi, const TileDims g,
                     const uint64_t *__restrict__ g_offhi, const int32_t *__restrict__ g_comp,
                     const GroupRec *__restrict__ groups, int ngroups,
                     const TermRec *__restrict__ terms, int nterms, int ndiag, int gsplit,
                     int wide, double *__restrict__ partial)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = g.m, c = g.c;
    const int tsize = 1 << m;
    const int npairs = tsize >> 1;
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);    // 2 x tsize (double-buffered)
    double *scr = reinterpret_cast<double *>(bufs + 2 * tsize);  // [kW][16][32]
    double *acc = scr + kW * 16 * 32;  // flip: [nflip][kSlots] (wide sweeps: [nflip]), then diag
    const int nflip = nterms - ndiag;
    const int slots = wide ? 1 : kSlots;
    double *accd = acc + nflip * slots;
    uint64_t *offhi = reinterpret_cast<uint64_t *>(accd + ndiag);
    for (int i = threadIdx.x; i < (1 << (m - c)); i += kT) offhi[i] = __ldg(g_offhi + i);
    for (int i = threadIdx.x; i < nflip * slots + ndiag; i += kT) acc[i] = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int comp_lane = __ldg(g_comp + lane);
    const uint32_t cmask = (1u << c) - 1u;
    const int qsize = npairs < 512 ? npairs : 512;  // pairs per item
    const int items_per_group = npairs / qsize;
    double *wscr = scr + warp * 16 * 32;
    __syncthreads();
    // small states (fewer tiles than CTAs): gsplit CTAs share a tile, each
    // taking every gsplit-th (group, quarter) item; the last one does the
    // Z-only strings
    const uint64_t ntiles = 1ull << g.ncomp;
    const int split = blockIdx.x % gsplit;
    const uint64_t tstride = gridDim.x / gsplit;
    uint64_t tile = blockIdx.x / gsplit;
    if (tile >= ntiles) return;
    uint64_t base = tbase(tile, lane, g.ncomp, comp_lane);
    {
        const double2 *src = psi + base;
#pragma unroll 4
        for (int l = threadIdx.x; l < tsize; l += kT) cp_async16(bufs + l, src + (l & cmask) + offhi[l >> c]);
        cp_async_commit();
    }
    for (int it = 0; tile < ntiles; ++it, tile += tstride) {
        double2 *sm = bufs + (it & 1) * tsize;
        const uint64_t next = tile + tstride;
        if (next < ntiles) {  // prefetch the next tile into the other buffer
            const double2 *src = psi + tbase(next, lane, g.ncomp, comp_lane);
            double2 *dstb = bufs + ((it + 1) & 1) * tsize;
#pragma unroll 4
            for (int l = threadIdx.x; l < tsize; l += kT) cp_async16(dstb + l, src + (l & cmask) + offhi[l >> c]);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        // ---- flip groups: items (group, quarter) round-robin over warps ----
        for (int item = warp + kW * split; !wide && item < ngroups * items_per_group;
             item += kW * gsplit) {
            const int gi = item / items_per_group, slot = item % items_per_group;
            const uint32_t f = __ldg(&groups[gi].f_loc);
            const int h = __ldg(&groups[gi].h);
            const int t0 = __ldg(&groups[gi].t0), tim = __ldg(&groups[gi].t_im),
                      t1 = __ldg(&groups[gi].t1);
            const uint32_t pbase = slot * qsize + lane;  // lanes on consecutive pairs
            double vr[16], vi[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const uint32_t p = pbase + 32 * r;
                double re = 0.0, im = 0.0;
                if (p < (uint32_t)npairs) {
                    const uint32_t l0 = ins0(p, h), l1 = l0 ^ f;
                    const double2 x = sm[l0], y = sm[l1];
                    re = fma(x.x, y.x, x.y * y.y);
                    im = fma(x.x, y.y, -x.y * y.x);
                }
                vr[r] = re;
                vi[r] = im;
            }
            if (tim > t0) {
                wht16(vr);
#pragma unroll
                for (int r = 0; r < 16; ++r) wscr[r * 32 + lane] = vr[r];
                __syncwarp();
                eval_terms(wscr, lane, pbase, base, terms, t0, tim, acc, ndiag, slot);
                __syncwarp();
            }
            if (t1 > tim) {
                wht16(vi);
#pragma unroll
                for (int r = 0; r < 16; ++r) wscr[r * 32 + lane] = vi[r];
                __syncwarp();
                eval_terms(wscr, lane, pbase, base, terms, tim, t1, acc, ndiag, slot);
                __syncwarp();
            }
        }
        // ---- wide groups (12-bit tiles): transform of the pair products ----
        for (int gi = split; wide && gi < ngroups; gi += gsplit) {
            const uint32_t f = __ldg(&groups[gi].f_loc);
            const int h = __ldg(&groups[gi].h);
            const int t0 = __ldg(&groups[gi].t0), tim = __ldg(&groups[gi].t_im),
                      t1 = __ldg(&groups[gi].t1);
            double v[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t l0 = ins0(threadIdx.x + 256 * k, h), l1 = l0 ^ f;
                const double2 x = sm[l0], y = sm[l1];
                v[k] = fma(x.x, y.x, x.y * y.y);
                v[8 + k] = fma(x.x, y.y, -x.y * y.x);
            }
            tile_wht(v, 3, scr);
            for (int t = t0 + threadIdx.x; t < t1; t += kT) {
                const uint32_t sp = __ldg(&terms[t].s_loc);
                const double val = scr[(t >= tim ? 2048 : 0) + wpos(sp)];
                const uint32_t sg = __popcll(base & __ldg(&terms[t].s_hi)) & 1u;
                acc[t - ndiag] += __ldg(&terms[t].scale) * (sg ? -val : val);
            }
        }
        // ---- Z-only strings: WHT of |psi|^2 over the tile ----
        if (ndiag > 0 && split == gsplit - 1 && m == kMaxTileBits) {
            double v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double2 a = sm[threadIdx.x + 256 * k];
                v[k] = fma(a.x, a.x, a.y * a.y);
            }
            tile_wht(v, 4, scr);
            for (int t = threadIdx.x; t < ndiag; t += kT) {
                const uint32_t sp = __ldg(&terms[t].s_loc);
                const double val = scr[(sp >> 11) * 2048 + wpos(sp & 2047u)];
                const uint32_t tp = __popcll(base & __ldg(&terms[t].s_hi)) & 1u;
                accd[t] += tp ? -val : val;
            }
        } else if (ndiag > 0 && split == gsplit - 1) {
            double p[kPer];
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int l = threadIdx.x + k * kT;
                if (l < tsize) {
                    const double2 a = sm[l];
                    p[k] = fma(a.x, a.x, a.y * a.y);
                }
            }
            __syncthreads();
            double *pw = reinterpret_cast<double *>(sm);
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int l = threadIdx.x + k * kT;
                if (l < tsize) pw[l] = p[k];
            }
            __syncthreads();
            for (int b = 0; b < m; ++b) {
                for (int i = threadIdx.x; i < npairs; i += kT) {
                    const uint32_t l0 = ins0(i, b), l1 = l0 | (1u << b);
                    const double u = pw[l0], v = pw[l1];
                    pw[l0] = u + v;
                    pw[l1] = u - v;
                }
                __syncthreads();
            }
            for (int t = threadIdx.x; t < ndiag; t += kT) {
                const double v = pw[__ldg(&terms[t].s_loc)];
                const uint32_t tp = __popcll(base & __ldg(&terms[t].s_hi)) & 1u;
                accd[t] += tp ? -v : v;
            }
        }
        __syncthreads();
        if (next < ntiles) base = tbase(next, lane, g.ncomp, comp_lane);
    }
    cp_async_wait<0>();
    // per-CTA partial sums, fixed slot order
    for (int t = threadIdx.x; t < nterms; t += kT) {
        double v;
        if (t < ndiag) {
            v = accd[t];
        } else {
            v = 0.0;
            for (int s = 0; s < slots; ++s) v += acc[(t - ndiag) * slots + s];
        }
        partial[(size_t)blockIdx.x * nterms + t] = v;
    }
}

size_t sweep2_smem(const TileDims &g, int nterms, int ndiag, bool wide)
{
    return ((size_t)32 << g.m) + (size_t)8 * kW * 16 * 32 +
           (size_t)8 * ((nterms - ndiag) * (wide ? 1 : kSlots) + ndiag) + ((size_t)8 << (g.m - g.c));
}

}  // namespace

// Grid of one sweep: tiles over CTAs (persistent, per_sm CTAs per SM); when
// there are fewer tiles than CTA slots, *gsplit CTAs share each tile's items.
int expect_sweep_grid(const TileDims &g, int nterms, int ndiag, int ngroups, bool wide, int *gsplit)
{
    int dev = 0;
    cudaGetDevice(&dev);
    static PerDeviceOnce once;
    // a failure here surfaces as the launch error of expect_sweep2_kernel
    (void)once.run([] {
        return cudaFuncSetAttribute(expect_sweep2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    227 * 1024);
    });
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expect_sweep2_kernel, kT,
                                                      sweep2_smem(g, nterms, ndiag, wide)) != cudaSuccess)
        per_sm = 1;
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << g.ncomp;
    const uint64_t cap = (uint64_t)num_sms(dev) * per_sm;
    int split = 1;
    if (ntiles < cap) {
        const int npairs = 1 << (g.m - 1);
        const int items = ngroups * (npairs / (npairs < 512 ? npairs : 512));
        // one item per warp; wide sweeps: one group per CTA
        const uint64_t want = wide ? (uint64_t)ngroups : (uint64_t)(items + kW - 1) / kW;
        split = (int)std::max<uint64_t>(1, std::min<uint64_t>(cap / ntiles, want));
    }
    if (gsplit) *gsplit = split;
    return ntiles < cap ? (int)(ntiles * split) : (int)cap;
}

cudaError_t launch_expect_sweep(const double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                                const int32_t *d_comp, const GroupRec *d_groups, int ngroups,
                                const TermRec *d_terms, int nterms, int ndiag, bool wide,
                                double *d_partial, int *grid_out, cudaStream_t st)
{
    int split = 1;
    const int grid = expect_sweep_grid(g, nterms, ndiag, ngroups, wide, &split);
    *grid_out = grid;
    expect_sweep2_kernel<<<grid, kT, sweep2_smem(g, nterms, ndiag, wide), st>>>(
        psi, g, d_offhi, d_comp, d_groups, ngroups, d_terms, nterms, ndiag, split, wide ? 1 : 0,
        d_partial);
    return cudaGetLastError();
}

}  // namespace qsv
