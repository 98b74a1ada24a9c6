// qsv_internal.h -- shared definitions between the sm_100a kernels, the C++
// pass planner and the C-ABI (include/qsv.h).
//
// Data layout in HBM: one state = 2^n complex128 amplitudes stored as
// double2 {re, im} in basis-index order; index bit k is qubit k
// (reference: statevector.py:1-6, dump_state layout statevector.py:214-216).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

namespace qsv {

// Shared-memory tile swizzle (16-B slot of tile index l), used by the planner
// (register-block maps), the interpreted tile kernels and -- restated as source
// text -- the NVRTC kernels (qsv_jit.cpp).  GF(2)-linear: slot bits 0..2 =
// (l ^ F) & 7 with F = fold of l's higher 3-bit chunks, bits 3..5 = F, bits
// 6.. = l's.  The banks are those of the plain fold; the row permutation puts
// each 64 / 128-B segment where the TMA 64B / 128B swizzle expects it.
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t tile_swz(uint32_t l)
{
    const uint32_t f = ((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u;
    return (l & ~63u) | (f << 3) | ((l ^ f) & 7u);
}

// One-time setup per device (kernel attributes such as the dynamic shared
// memory cap are per device context): run(f) calls f once for the current
// device, thread-safely, and again on a device that has not seen it yet.
class PerDeviceOnce {
    std::mutex mu_;
    bool done_[64] = {};

public:
    template <class F>
    cudaError_t run(F f)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu_);
        if (dev >= 0 && dev < 64 && done_[dev]) return cudaSuccess;
        const cudaError_t e = f();
        if (e == cudaSuccess && dev >= 0 && dev < 64) done_[dev] = true;
        return e;
    }
};

// Largest tile (in qubits) a CTA keeps resident in shared memory: 2^12
// amplitudes x 16 B = 64 KiB, so three CTAs fit one SM's 228 KiB.
constexpr int kMaxTileBits = 12;
// Low physical bits that every tile always contains: 2^5 amplitudes = 512 B
// contiguous segments, so every warp-wide 16 B load is fully coalesced.
constexpr int kMinContig = 5;
constexpr int kMaxQubits = 40;
// Register bits of a tile-kernel block: each thread holds 2^kBlockBits
// amplitudes (8 -> 512 threads per 4096-amplitude tile, 16 warps per SM).
#ifndef QSV_BLOCK_BITS
#define QSV_BLOCK_BITS 4
#endif
constexpr int kBlockBits = QSV_BLOCK_BITS;

// ---- fused tile-pass program -------------------------------------------
enum OpType : int32_t {
    OP_U1 = 1,     // dense 2x2 on local bit a; params[p..p+8)
    OP_U2 = 2,     // dense 4x4, rows = 2*bit(a) + bit(b); params[p..p+32)
    OP_CX = 3,     // CNOT control a, target b (permutation, no flops)
    OP_SWAP = 4,   // SWAP a, b
    OP_X = 5,      // Pauli X on a
    OP_DIAG1 = 6,  // diag(d0, d1) on a; params[p..p+4)
    OP_ROTG = 7,   // rotations exp(-i t/2 P) sharing local flip mask f (highest bit h), rots[r0..r1)
    OP_ROTD = 8,   // diagonal (Z-only) rotations, rots[r0..r1)
    OP_GMAT = 9,   // fused same-flip group: per pair one 2x2 from params[p..], selected by
                   // (common sign parity, flip-bit pattern); rots[r0] holds the common masks
    OP_U1C = 10,   // dense 2x2 on a selected by bit b: params[p..p+8) if bit b = 0, [p+8..p+16)
                   // if 1 (a U3 that absorbed a deferred controlled phase, qsv_planner.cpp CzDefer)
};

struct OpRec {  // 32 B
    int32_t type;
    int32_t a, b, h;  // h: highest flip bit (ROTG) / matrix class (U1: 0 general, 1 m00 real, 2 real, 3 m00+m10 real)
    int32_t r0, r1, p;
    uint32_t f;
};

struct RotRec {     // 32 B
    uint64_t s_hi;  // sign bits outside the tile (per-tile constant parity)
    uint32_t s_loc; // sign bits inside the tile, in local bit order
    int32_t q;      // low 2 bits: kappa = i^q ; bit 2: |y| odd
    double c, s;    // cos(theta/2), sin(theta/2)
};

// A block of the tile kernel.  The SMEM tile is addressed through a
// GF(2)-affine map slot(L) = swz(A L ^ t) of the logical tile index L, so
// permutation gates (CNOT, SWAP, X) cost nothing on the device: the planner
// folds them into (A, t).  cols[] hold swizzled map columns:
//   kind 0 (register block, <= kBlockBits logical bits B): cols[0..11-kBlockBits]
//          = columns of the non-B bits in ascending order (= thread-index
//          bits), cols[12-kBlockBits..11] = columns of B (block-local bits);
//          ops[op0..op1) use block-local bit indices.
//   kind 1 (wide-flip rotation group on SMEM): cols[b] = column of tile bit b.
struct BlockRec {  // 48 B
    int32_t kind;
    int32_t op0, op1;
    uint16_t cols[12];
    uint16_t tswz;
    uint16_t pad0;  // bit 0: warp-local entry (the transition into this block needs only __syncwarp)
    int32_t pad[2];
};

// Tile geometry of one pass (host side): local bit i <-> physical bit pos[i]; pos[i] = i
// for i < c (contiguous low block).  The tile index enumerates the n - m
// complement bits comp[] in ascending order.
struct TileGeom {
    int32_t n, m, c, ncomp;
    int32_t pos[kMaxTileBits];
    int32_t comp[kMaxQubits];
};

// What the kernels see of a TileGeom (the position tables travel as device
// arrays: offhi[2^(m-c)] and comp[32]).
struct TileDims {
    int32_t n, m, c, ncomp;
};

// ---- expectation sweep --------------------------------------------------
struct GroupRec {   // a flip group of an expectation sweep (32 B)
    uint32_t f_loc;
    int32_t h;
    int32_t t0, t_im, t1;  // terms [t0, t_im) use Re w, [t_im, t1) use Im w
    int32_t pad[3];        // pad[0] bit 0: wide group (tile-wide transform path)
};

struct TermRec {    // 24 B
    uint64_t s_hi;
    uint32_t s_loc;
    int32_t use_im;
    double scale;
};

}  // namespace qsv

// ---- state handle -------------------------------------------------------
struct qsv_state {
    int n = 0;
    int device = 0;
    uint64_t dim = 0;
    double2 *amps = nullptr;
    cudaStream_t stream = nullptr;  // the device's library stream unless qsv_set_stream
    // asynchronous download (qsv_download_async) in flight on the copy stream
    cudaEvent_t dl_done = nullptr;
    bool dl_pending = false;
};

namespace qsv {

void set_error(const std::string &msg);
int fail(const std::string &msg);

// kernels (qsv_kernels.cu)
int num_sms(int device);
cudaError_t launch_tile_pass(double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                             const int32_t *d_comp, const OpRec *d_ops, int nops,
                             const RotRec *d_rots, const double *d_params, cudaStream_t st);
cudaError_t launch_tile_blocks(double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                               const int32_t *d_geo, const BlockRec *d_blocks, int nblocks,
                               const OpRec *d_ops, int nops, const RotRec *d_rots, int nrots,
                               const double *d_params, int nparams, bool lite, cudaStream_t st);
cudaError_t launch_expect_sweep(const double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                                const int32_t *d_comp, const GroupRec *d_groups, int ngroups,
                                const TermRec *d_terms, int nterms, int ndiag, bool wide,
                                double *d_partial, int *grid_out, cudaStream_t st);
int elementwise_grid(uint64_t dim, int device);
int adjoint_smem_max_qubits();
size_t adjoint_scratch_doubles(int n, int64_t R, int device);
cudaError_t launch_rotation_adjoint(double2 *phi, double2 *lam, int n, int64_t R, const uint64_t *X,
                                    const uint64_t *Y, const uint64_t *Z, const uint64_t *hX,
                                    const uint64_t *hY, const uint64_t *hZ, const double2 *cs,
                                    double *d_scratch, double *d_grad, cudaStream_t st);
cudaError_t launch_reduce_columns(const double *partial, int rows, int cols, const int32_t *d_map,
                                  double *out, cudaStream_t st);
cudaError_t launch_set_basis(double2 *psi, uint64_t dim, uint64_t index, cudaStream_t st);
struct GmatJob {     // one OP_GMAT table filled on the device
    uint64_t dst;     // byte offset of the table from the blob base
    int32_t r0, r1;   // rotations of the group (cs / q / yF index)
    int32_t F, H, w;  // block-local flip, its highest bit, popcount
    int32_t yf;       // offset of the group's yF bytes
};
cudaError_t launch_gmat_fill(char *base, const GmatJob *d_jobs, int njobs, const double2 *d_cs,
                             const int32_t *d_q, const uint8_t *d_yF, cudaStream_t st);
cudaError_t launch_apply_operator_small(const double2 *src, double2 *dst, uint64_t dim,
                                        const uint64_t *d_fs, const double2 *d_coefs, int S,
                                        cudaStream_t st);
cudaError_t launch_apply_pauli(const double2 *src, double2 *dst, uint64_t dim, uint64_t x,
                               uint64_t y, uint64_t z, double cre, double cim, int accumulate,
                               cudaStream_t st);
cudaError_t launch_dot(const double2 *a, const double2 *b, uint64_t dim, double *d_partial,
                       double *d_out2, int mode, cudaStream_t st);
cudaError_t launch_rot_global(double2 *psi, int n, uint64_t flip, const RotRec *d_rots, int nrot,
                              cudaStream_t st);
cudaError_t launch_expect_global(const double2 *psi, int n, const GroupRec *d_groups,
                                 const uint64_t *d_gflip, int ngroups, const TermRec *d_terms,
                                 int nterms, double *d_partial, int *grid_out, cudaStream_t st);
int expect_global_grid(int n);
int expect_sweep_grid(const TileDims &g, int nterms, int ndiag, int ngroups, bool wide,
                      int *gsplit = nullptr);
// run-time specialised tile passes (qsv_jit.cpp)
bool jit_enabled(int n_qubits, int uses = 0);
const char *jit_unavailable_reason();
bool jit_source(const TileGeom &g, const BlockRec *blocks, int nblocks, const OpRec *ops,
                const RotRec *rots, int nparams, std::string &src);
int jit_prepare(int device, const std::vector<const std::string *> &srcs, std::string &err);
bool jit_launch(int device, const std::string &src, double2 *psi, const TileDims &g,
                const uint64_t *d_offhi, const int32_t *d_geo, const double *d_params, int nparams,
                int grid, cudaStream_t st);
// Loaded module of a prepared source (nullptr if unavailable); stable for the
// process lifetime, so a cached program launches without re-hashing sources.
const void *jit_module(int device, const std::string &src);
// basis != ~0: the pass reads |basis> instead of psi (first pass of an evolve
// from a basis state: no HBM read, no separate set_basis write)
bool jit_launch_module(const void *mod, double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                       const int32_t *d_geo, const double *d_params, int nparams, int grid,
                       cudaStream_t st, uint64_t basis = ~0ull);
size_t sample_scratch_bytes(uint64_t dim);
cudaError_t launch_sample_parity(const double2 *psi, uint64_t dim, int64_t shots, uint64_t k0,
                                 uint64_t k1, uint64_t support, void *scratch, size_t scratch_bytes,
                                 int64_t *d_outcomes, unsigned long long *h_odd, cudaStream_t st);
struct SweepPlan;
bool jit_sweep_source(const SweepPlan &sp, std::string &src);
bool jit_sweep_launch(int device, const std::string &src, const double2 *psi, const TileDims &g,
                      const uint64_t *d_offhi, const int32_t *d_geo, double *d_partial, int grid,
                      cudaStream_t st);
cudaError_t launch_dense(double2 *psi, int n, int k, const int *qubits, const double2 *d_m, int sms,
                         cudaStream_t st);
struct SmallGroup;    // qsv_planner.h
struct SmallProgram;  // qsv_planner.h
// Small-state rotation program: one CTA, state in shared memory (qsv_small.cu).
cudaError_t launch_small(double2 *psi, int n, uint64_t basis, const SmallProgram &sp, const SmallGroup *groups,
                         const int32_t *meta, const double *theta, const int32_t *runs, const uint32_t *xo,
                         const uint32_t *tab, cudaStream_t st);
// dst (n_dst qubits) = the parity class cls embedded from its (n_dst-1)-qubit half
// <P_t> of a state of <= 12 qubits, one warp per string (rec: 4 x u32 per string)
cudaError_t launch_expect_small(const double2 *psi, int n, const uint32_t *rec, int S, double *out, int sms,
                                cudaStream_t st);
cudaError_t launch_embed_parity(double2 *dst, const double2 *src, int n_dst, uint64_t wlow, uint32_t cls,
                                int sms, cudaStream_t st);
// a[i] <-> b[i] (i < n) over peer memory: the relayout exchange of qsv_dist.cpp
cudaError_t launch_swap_chunks(double2 *a, double2 *b, uint64_t n, int sms, cudaStream_t st);
cudaError_t launch_axpby(double2 *y, const double2 *x, uint64_t dim, double are, double aim,
                         double bre, double bim, cudaStream_t st);

}  // namespace qsv
