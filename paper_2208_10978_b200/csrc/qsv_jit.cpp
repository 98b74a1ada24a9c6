// qsv_jit.cpp -- run-time specialised tile passes (NVRTC -> sm_100a cubin).
//
// The interpreted tile kernel (qsv_tile_block.cu) decodes each pass's block
// program at run time: a switch per op, matrices re-read from shared memory,
// and -- because the register array a[16] must sit in the same registers at
// every loop back-edge -- register moves after every in-place 2x2 update.
// ncu on the config-2 brickwork shows the FP64 pipe only ~38 % busy with
// ~1.5 non-FP64 instructions issued per FP64 one.  A dense-gate pass is pure
// data-independent straight-line code once the planner has fixed its
// structure, so this module generates that code: every block's gather /
// scatter offsets become immediates, every op a template instantiation whose
// matrix entries are __constant__ operands of the DFMA/DMUL instructions (no
// loads, no registers), and the whole block is one basic block the compiler
// schedules freely.  Structure-identical passes share a module (cache keyed by
// the generated source); the angle-dependent matrices are copied into the
// module's __constant__ bank before each launch (stream-ordered DtoD copy).
//
// The tile skeleton is the two-group ring pipeline of tile_ring_kernel:
// 512 threads = 2 groups x 8 warps, 3 x 64 KiB SMEM stages, LDGSTS loads with
// mbarrier completion, named-barrier block syncs, streaming stores.
//
// NVRTC and the driver API are dlopen'ed on first use, so libqsv.so still
// loads (and its planner entry points work) on machines without a GPU driver.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "qsv_internal.h"
#include "qsv_planner.h"

namespace qsv {

namespace {

// ---- minimal driver / NVRTC API surface ----------------------------------
typedef int CUresult;
typedef void *CUmodule;
typedef void *CUfunction;
typedef unsigned long long CUdeviceptr;
typedef int nvrtcResult;
typedef void *nvrtcProgram;

struct Api {
    bool tried = false, ok = false;
    std::string why;
    // nvrtc
    nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                                 const char *const *) = nullptr;
    nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
    // driver
    CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*ModuleGetGlobal)(CUdeviceptr *, size_t *, CUmodule, const char *) = nullptr;
    CUresult (*FuncSetAttribute)(CUfunction, int, int) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             unsigned, cudaStream_t, void **, void **) = nullptr;
    CUresult (*MemcpyDtoDAsync)(CUdeviceptr, CUdeviceptr, size_t, cudaStream_t) = nullptr;
    // optional: TMA tile loads (QSV_PASS_TMA); absent -> LDGSTS staging
    CUresult (*TensorMapEncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                     const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                     const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
};
Api g_api;

template <typename F>
bool sym(void *h, const char *name, F &out)
{
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

bool load_api()
{
    if (g_api.tried) return g_api.ok;
    g_api.tried = true;
    void *nv = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!nv) nv = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
    void *cu = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!nv || !cu) {
        g_api.why = !nv ? "libnvrtc not found" : "libcuda.so.1 not found";
        return false;
    }
    bool ok = sym(nv, "nvrtcCreateProgram", g_api.CreateProgram) &&
              sym(nv, "nvrtcCompileProgram", g_api.CompileProgram) &&
              sym(nv, "nvrtcGetCUBINSize", g_api.GetCUBINSize) && sym(nv, "nvrtcGetCUBIN", g_api.GetCUBIN) &&
              sym(nv, "nvrtcGetProgramLogSize", g_api.GetProgramLogSize) &&
              sym(nv, "nvrtcGetProgramLog", g_api.GetProgramLog) &&
              sym(nv, "nvrtcDestroyProgram", g_api.DestroyProgram) &&
              sym(cu, "cuModuleLoadData", g_api.ModuleLoadData) &&
              sym(cu, "cuModuleGetFunction", g_api.ModuleGetFunction) &&
              sym(cu, "cuModuleGetGlobal_v2", g_api.ModuleGetGlobal) &&
              sym(cu, "cuFuncSetAttribute", g_api.FuncSetAttribute) &&
              sym(cu, "cuLaunchKernel", g_api.LaunchKernel) &&
              sym(cu, "cuMemcpyDtoDAsync_v2", g_api.MemcpyDtoDAsync);
    if (ok) sym(cu, "cuTensorMapEncodeTiled", g_api.TensorMapEncodeTiled);
    if (!ok) g_api.why = "missing NVRTC / driver symbols";
    g_api.ok = ok;
    return ok;
}

// ---- device-side skeleton (compiled by NVRTC) ------------------------------
const char *kSkeleton = R"QSV(
typedef unsigned long long u64;
typedef unsigned int u32;
#define KT 256
#define KSTAGES 3
#define TSIZE 4096
__constant__ double C[QSV_NPARAMS];

__device__ __forceinline__ double2 cmul(double ar, double ai, double2 x)
{
    return make_double2(fma(ar, x.x, -ai * x.y), fma(ar, x.y, ai * x.x));
}

// dense 2x2 on register bit J; K = 0 general, 1 m00 real, 2 all real,
// 3 m00 and m10 real, 4 m00 = 1, 6 m00 = m11 = 1
template <int J, int K, int P>
__device__ __forceinline__ void u1(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r & (1 << J)) continue;
        const double2 x = a[r], y = a[r | (1 << J)];
        double2 o0, o1;
        if (K == 2) {
            o0.x = fma(C[P], x.x, C[P + 2] * y.x);
            o0.y = fma(C[P], x.y, C[P + 2] * y.y);
            o1.x = fma(C[P + 4], x.x, C[P + 6] * y.x);
            o1.y = fma(C[P + 4], x.y, C[P + 6] * y.y);
        } else if (K == 4) {  // m00 = 1 (U3 divided by cos(theta/2), qsv_planner.cpp U3Norm)
            o0.x = fma(C[P + 2], y.x, fma(-C[P + 3], y.y, x.x));
            o0.y = fma(C[P + 2], y.y, fma(C[P + 3], y.x, x.y));
            o1.x = fma(C[P + 4], x.x, fma(-C[P + 5], x.y, fma(C[P + 6], y.x, -C[P + 7] * y.y)));
            o1.y = fma(C[P + 4], x.y, fma(C[P + 5], x.x, fma(C[P + 6], y.y, C[P + 7] * y.x)));
        } else if (K == 6) {  // m00 = m11 = 1: the shear of a phase-deferred U3 (U3Norm)
            o0.x = fma(C[P + 2], y.x, fma(-C[P + 3], y.y, x.x));
            o0.y = fma(C[P + 2], y.y, fma(C[P + 3], y.x, x.y));
            o1.x = fma(C[P + 4], x.x, fma(-C[P + 5], x.y, y.x));
            o1.y = fma(C[P + 4], x.y, fma(C[P + 5], x.x, y.y));
        } else if (K == 3) {  // m00 and m10 real (phase-deferred U3)
            o0.x = fma(C[P], x.x, fma(C[P + 2], y.x, -C[P + 3] * y.y));
            o0.y = fma(C[P], x.y, fma(C[P + 2], y.y, C[P + 3] * y.x));
            o1.x = fma(C[P + 4], x.x, fma(C[P + 6], y.x, -C[P + 7] * y.y));
            o1.y = fma(C[P + 4], x.y, fma(C[P + 6], y.y, C[P + 7] * y.x));
        } else {
            if (K == 1) {
                o0.x = fma(C[P], x.x, fma(C[P + 2], y.x, -C[P + 3] * y.y));
                o0.y = fma(C[P], x.y, fma(C[P + 2], y.y, C[P + 3] * y.x));
            } else {
                o0.x = fma(C[P], x.x, fma(-C[P + 1], x.y, fma(C[P + 2], y.x, -C[P + 3] * y.y)));
                o0.y = fma(C[P], x.y, fma(C[P + 1], x.x, fma(C[P + 2], y.y, C[P + 3] * y.x)));
            }
            o1.x = fma(C[P + 4], x.x, fma(-C[P + 5], x.y, fma(C[P + 6], y.x, -C[P + 7] * y.y)));
            o1.y = fma(C[P + 4], x.y, fma(C[P + 5], x.x, fma(C[P + 6], y.y, C[P + 7] * y.x)));
        }
        a[r] = o0;
        a[r | (1 << J)] = o1;
    }
}

// u1 selected by register bit JB: matrix P if bit JB = 0, P + 8 if 1 (OP_U1C);
// K = 1 (m00 real) or 4 (m00 = 1), as u1
template <int J, int JB, int K, int P>
__device__ __forceinline__ void u1c(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r & (1 << J)) continue;
        const int Q = P + 8 * ((r >> JB) & 1);
        const double2 x = a[r], y = a[r | (1 << J)];
        double2 o0, o1;
        if (K == 4) {
            o0.x = fma(C[Q + 2], y.x, fma(-C[Q + 3], y.y, x.x));
            o0.y = fma(C[Q + 2], y.y, fma(C[Q + 3], y.x, x.y));
        } else if (K == 1) {
            o0.x = fma(C[Q], x.x, fma(C[Q + 2], y.x, -C[Q + 3] * y.y));
            o0.y = fma(C[Q], x.y, fma(C[Q + 2], y.y, C[Q + 3] * y.x));
        } else {
            o0.x = fma(C[Q], x.x, fma(-C[Q + 1], x.y, fma(C[Q + 2], y.x, -C[Q + 3] * y.y)));
            o0.y = fma(C[Q], x.y, fma(C[Q + 1], x.x, fma(C[Q + 2], y.y, C[Q + 3] * y.x)));
        }
        o1.x = fma(C[Q + 4], x.x, fma(-C[Q + 5], x.y, fma(C[Q + 6], y.x, -C[Q + 7] * y.y)));
        o1.y = fma(C[Q + 4], x.y, fma(C[Q + 5], x.x, fma(C[Q + 6], y.y, C[Q + 7] * y.x)));
        a[r] = o0;
        a[r | (1 << J)] = o1;
    }
}

// dense 4x4 on register bits (JA = MSB of the row index, JB)
template <int JA, int JB, int P>
__device__ __forceinline__ void u2(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r & ((1 << JA) | (1 << JB))) continue;
        const int i0 = r, i1 = r | (1 << JB), i2 = r | (1 << JA), i3 = r | (1 << JA) | (1 << JB);
        const double2 x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
        double2 o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int R = P + 8 * k;
            o[k].x = fma(C[R], x0.x, fma(-C[R + 1], x0.y, fma(C[R + 2], x1.x, fma(-C[R + 3], x1.y,
                     fma(C[R + 4], x2.x, fma(-C[R + 5], x2.y, fma(C[R + 6], x3.x, -C[R + 7] * x3.y)))))));
            o[k].y = fma(C[R], x0.y, fma(C[R + 1], x0.x, fma(C[R + 2], x1.y, fma(C[R + 3], x1.x,
                     fma(C[R + 4], x2.y, fma(C[R + 5], x2.x, fma(C[R + 6], x3.y, C[R + 7] * x3.x)))))));
        }
        a[i0] = o[0];
        a[i1] = o[1];
        a[i2] = o[2];
        a[i3] = o[3];
    }
}

// diag(d0, d1) on register bit J
template <int J, int P>
__device__ __forceinline__ void dg(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r)
        a[r] = (r & (1 << J)) ? cmul(C[P + 2], C[P + 3], a[r]) : cmul(C[P], C[P + 1], a[r]);
}

// diag(d0, d1) on a thread-index bit
template <int P>
__device__ __forceinline__ void dgt(double2 (&a)[16], bool bit)
{
    const double dr = bit ? C[P + 2] : C[P], di = bit ? C[P + 3] : C[P + 1];
#pragma unroll
    for (int r = 0; r < 16; ++r) a[r] = cmul(dr, di, a[r]);
}

// fused same-flip rotation group on block-local flip F (highest bit H): per
// pair one 2x2 from the cp = 0 half of the table, selected by the flip
// pattern of r ^ F; the other parity uses Z M Z (negated off-diagonals),
// applied as sign flips of y and of the second output.
__host__ __device__ constexpr int hbit(int v) { return v >= 8 ? 3 : v >= 4 ? 2 : v >= 2 ? 1 : 0; }
__host__ __device__ constexpr int par4(int v) { return (v ^ (v >> 1) ^ (v >> 2) ^ (v >> 3)) & 1; }
template <int F>
__device__ __forceinline__ constexpr int gm_cfg(int r1)
{
    int out = 0, k = 0;
    const int H = hbit(F);
    for (int b = 0; b < 4; ++b)
        if (((F >> b) & 1) && b != H) {
            out |= ((r1 >> b) & 1) << k;
            ++k;
        }
    return out;
}
__device__ __forceinline__ double negif(double v, u32 s)
{
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)s << 63));
}
template <int F, int P, int ZB>
__device__ __forceinline__ void gm(double2 (&a)[16], u32 par0)
{
    constexpr int H = hbit(F);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r & (1 << H)) continue;
        const int r1 = r ^ F;
        const u32 cp = par0 ^ (u32)par4(r1 & ZB);
        const int M = P + 8 * gm_cfg<F>(r1);
        const double2 x = a[r], yy = a[r1];
        const double2 y = make_double2(negif(yy.x, cp), negif(yy.y, cp));
        double2 o0, o1;
        o0.x = fma(C[M], x.x, fma(-C[M + 1], x.y, fma(C[M + 2], y.x, -C[M + 3] * y.y)));
        o0.y = fma(C[M], x.y, fma(C[M + 1], x.x, fma(C[M + 2], y.y, C[M + 3] * y.x)));
        o1.x = fma(C[M + 4], x.x, fma(-C[M + 5], x.y, fma(C[M + 6], y.x, -C[M + 7] * y.y)));
        o1.y = fma(C[M + 4], x.y, fma(C[M + 5], x.x, fma(C[M + 6], y.y, C[M + 7] * y.x)));
        a[r] = o0;
        a[r1] = make_double2(negif(o1.x, cp), negif(o1.y, cp));
    }
}

#ifdef QSV_GMD
// gm with the table offset P and the block sign mask ZB at run time: one code
// body per flip pattern F, shared by every group with that pattern (the
// compact form of small-state passes, whose straight-line code would be
// executed once and stream through the instruction cache).  The matrices are
// read from the pass's parameter copy in shared memory (QS: stage 2 of the
// ring, which a pass over <= 2 tiles per CTA never fills) as 16-B broadcast
// loads -- four per pair instead of eight run-time-indexed constant loads.
template <int F>
__device__ __forceinline__ void gm_rt(double2 (&a)[16], u32 par0, int P, u32 ZB, const double2 *QS)
{
    constexpr int H = hbit(F);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r & (1 << H)) continue;
        const int r1 = r ^ F;
        const u32 cp = par0 ^ (u32)(__popc((u32)r1 & ZB) & 1);
        const double2 *M = QS + ((P + 8 * gm_cfg<F>(r1)) >> 1);
        const double2 m01 = M[0], m23 = M[1], m45 = M[2], m67 = M[3];
        const double2 x = a[r], yy = a[r1];
        const double2 y = make_double2(negif(yy.x, cp), negif(yy.y, cp));
        double2 o0, o1;
        o0.x = fma(m01.x, x.x, fma(-m01.y, x.y, fma(m23.x, y.x, -m23.y * y.y)));
        o0.y = fma(m01.x, x.y, fma(m01.y, x.x, fma(m23.x, y.y, m23.y * y.x)));
        o1.x = fma(m45.x, x.x, fma(-m45.y, x.y, fma(m67.x, y.x, -m67.y * y.y)));
        o1.y = fma(m45.x, x.y, fma(m45.y, x.x, fma(m67.x, y.y, m67.y * y.x)));
        a[r] = o0;
        a[r1] = make_double2(negif(o1.x, cp), negif(o1.y, cp));
    }
}
#endif
#ifdef QSV_GMD
// a run of fused rotation groups [k0, k1) of the descriptor table
__device__ __forceinline__ void gm_run(double2 (&a)[16], u32 tid, u64 base, int k0, int k1)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const double2 *QS = reinterpret_cast<const double2 *>(smem_raw + 1024) + 2 * TSIZE;
#pragma unroll 1
    for (int k = k0; k < k1; ++k) {
        const u32 pk = GMD_PK[k];
        const u32 par0 = (u32)((__popcll(base & GMD_SHI[k]) + __popc(tid & (pk >> 8))) & 1);
        const int P = GMD_P[k];
        const u32 zb = (pk >> 4) & 15u;
        switch (pk & 15u) {
            case 1: gm_rt<1>(a, par0, P, zb, QS); break;
            case 2: gm_rt<2>(a, par0, P, zb, QS); break;
            case 3: gm_rt<3>(a, par0, P, zb, QS); break;
            case 4: gm_rt<4>(a, par0, P, zb, QS); break;
            case 5: gm_rt<5>(a, par0, P, zb, QS); break;
            case 6: gm_rt<6>(a, par0, P, zb, QS); break;
            case 7: gm_rt<7>(a, par0, P, zb, QS); break;
            case 8: gm_rt<8>(a, par0, P, zb, QS); break;
            case 9: gm_rt<9>(a, par0, P, zb, QS); break;
            case 10: gm_rt<10>(a, par0, P, zb, QS); break;
            case 11: gm_rt<11>(a, par0, P, zb, QS); break;
            case 12: gm_rt<12>(a, par0, P, zb, QS); break;
            case 13: gm_rt<13>(a, par0, P, zb, QS); break;
            case 14: gm_rt<14>(a, par0, P, zb, QS); break;
            default: gm_rt<15>(a, par0, P, zb, QS); break;
        }
    }
}
#endif

// in-register permutations: pure relabelings in straight-line code
template <int A, int B>
__device__ __forceinline__ void pcx(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if ((r & (1 << A)) && !(r & (1 << B))) { const double2 t = a[r]; a[r] = a[r | (1 << B)]; a[r | (1 << B)] = t; }
}
template <int A, int B>
__device__ __forceinline__ void pswap(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if ((r & (1 << A)) && !(r & (1 << B))) {
            const int q = r ^ (1 << A) ^ (1 << B);
            const double2 t = a[r]; a[r] = a[q]; a[q] = t;
        }
}
template <int J>
__device__ __forceinline__ void px(double2 (&a)[16])
{
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (!(r & (1 << J))) { const double2 t = a[r]; a[r] = a[r | (1 << J)]; a[r | (1 << J)] = t; }
}

// GF(2)-linear tile swizzle (16-B slots): the low 3 bits (bank group) are the
// granule index XOR the fold F of all higher 3-bit chunks; bits 3..5 become F
// itself.  So a 2^c-amplitude segment (c = 2, 3) lands in one 64 / 128-B row
// whose chunks are XOR-ed with that row's address bits 7..8 / 7..9 -- exactly
// the TMA SWIZZLE_64B / 128B pattern -- while the bank of every slot is the
// same as with the plain fold (conflict analysis unchanged).
__device__ __forceinline__ u32 swz(u32 l)
{
    const u32 f = ((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u;
    return (l & ~63u) | (f << 3) | ((l ^ f) & 7u);
}
__device__ __forceinline__ u32 tb(u32 tid, int i, u32 col) { return (0u - ((tid >> i) & 1u)) & col; }
__device__ __forceinline__ void gsync(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }

__device__ __forceinline__ u64 tbase(u64 tile, int lane, int ncomp, int comp_lane)
{
    u64 bit = (lane < ncomp && ((tile >> lane) & 1ull)) ? (1ull << comp_lane) : 0ull;
    u32 lo = __reduce_or_sync(0xffffffffu, (u32)bit);
    u32 hi = __reduce_or_sync(0xffffffffu, (u32)(bit >> 32));
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u32 saddr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void *d, const void *s)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void mbar_init(u64 *b, int n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *b, u32 parity)
{
    asm volatile("{\n\t.reg .pred p;\nQJ_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra QJ_WAIT_%=;\n\t}" ::"r"(saddr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(u64 *b)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ int ring_bar(int it) { return it % KSTAGES + KSTAGES * ((it / KSTAGES) & 1); }
__device__ __forceinline__ void mbar_arrive_tx(u64 *b, u32 bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
struct __align__(64) TmapParam { u64 v[16]; };
// one 2^c-amplitude segment (row y of the 2-D view psi[2^(n-c)][2^(c+1) doubles])
// -> the 64 / 128-B shared row at dst, chunks XOR-swizzled by the hardware
__device__ __forceinline__ void tma_row(void *dst, const TmapParam *tm, int y, u64 *bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(saddr(dst)), "l"((u64)tm), "r"(0), "r"(y), "r"(saddr(bar)) : "memory");
}

__device__ __forceinline__ void apply_tile(double2 *sm, u32 tid, int bar, u64 base);

#ifdef QSV_GMD
#define QSV_PASS_THREADS KT  // compact passes: one tile group (<= 255 registers)
#else
#define QSV_PASS_THREADS (2 * KT)
#endif
extern "C" __global__ void __launch_bounds__(QSV_PASS_THREADS, 1)
qsv_pass(double2 *__restrict__ psi, int ncomp, int c, const u64 *__restrict__ g_offhi,
         const int *__restrict__ g_geo, u64 basis, const __grid_constant__ TmapParam tmap, int tma)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    u64 *full = reinterpret_cast<u64 *>(smem_raw);
    u32 *st_k = reinterpret_cast<u32 *>(full + 2 * KSTAGES);
    u64 *offk = reinterpret_cast<u64 *>(smem_raw + 256);  // per-k global offsets (see below)
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw + 1024);  // 1024-B aligned stages (TMA swizzle)
    u64 *offhi = reinterpret_cast<u64 *>(bufs + KSTAGES * TSIZE);
    const int nhi = 1 << (12 - c);
    const u32 tid_all = threadIdx.x;
    for (int i = tid_all; i < nhi; i += QSV_PASS_THREADS) offhi[i] = __ldg(g_offhi + i);
    if (tid_all < TSIZE / KT) {
        const u32 l = tid_all * KT;
        offk[tid_all] = (l & ((1u << c) - 1u)) + __ldg(g_offhi + (l >> c));
    }
    if (tid_all < 16) {
        u32 v = 0;
        for (int j = 0; j < 4; ++j)
            if ((tid_all >> j) & 1u) v ^= (u32)__ldg(g_geo + 40 + j);
        st_k[tid_all] = v;
    }
    if (tid_all == 0) {
        for (int s = 0; s < 2 * KSTAGES; ++s) mbar_init(full + s, KT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
#ifdef QSV_GMD
    {  // the pass parameters into ring stage 2 (gm_rt's broadcast loads)
        double *qs = reinterpret_cast<double *>(bufs + 2 * TSIZE);
        for (int i = tid_all; i < QSV_NPARAMS; i += QSV_PASS_THREADS) qs[i] = C[i];
    }
#endif
    __syncthreads();
    const u64 ntiles = 1ull << ncomp;
    if ((u64)blockIdx.x >= ntiles) return;
    const int T = (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1;
#ifdef QSV_GMD
    if (T > 1) __trap();  // one tile per CTA (compact passes cover <= 8 tiles)
#endif
    const int grp = (int)(tid_all / KT);
    const u32 tid = tid_all % KT;
    const int bar = 1 + grp;
    const int lane = tid & 31;
    const int comp_lane = __ldg(g_geo + lane);
    const u32 cmask = (1u << c) - 1u;
    u32 st_base = (u32)__ldg(g_geo + 44);
    for (int i = 0; i < 8; ++i)
        if ((tid >> i) & 1u) st_base ^= (u32)__ldg(g_geo + 32 + i);
    // loop-invariant parts of the tile addresses: slot l = tid + KT k is
    // tid ^ KT k (tid < KT), and swz and the global offset (l & cmask) +
    // offhi[l >> c] are both linear over disjoint index bits, so per k only a
    // constant slot mask and one broadcast table entry offk[k] remain
    const u32 swz_t = swz(tid);
    const u64 goff_t = (u64)(tid & cmask) + offhi[tid >> c];
    auto load = [&](int it) {
        const u64 tile = blockIdx.x + (u64)it * gridDim.x;
        const u64 b = tbase(tile, lane, ncomp, comp_lane);
        double2 *buf = bufs + (it % KSTAGES) * TSIZE;
        if (basis != ~0ull) {  // the pass starts from |basis>: synthesise, no HBM read
#pragma unroll
            for (int k = 0; k < TSIZE / KT; ++k) {
                const u64 gi = b + goff_t + offk[k];
                buf[swz_t ^ swz((u32)(k * KT))] = make_double2(gi == basis ? 1.0 : 0.0, 0.0);
            }
            mbar_arrive(full + ring_bar(it));
            return;
        }
        if (tma) {  // TMA: the thread's share of the tile's segments, one row each
            const int nseg = TSIZE >> c;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // stage reuse (WAR)
            mbar_arrive_tx(full + ring_bar(it), (u32)(nseg / KT) * (16u << c));
            for (int h = tid; h < nseg; h += KT)
                tma_row(buf + (swz((u32)h << c) & ~cmask), &tmap, (int)((b + offhi[h]) >> c),
                        full + ring_bar(it));
            return;
        }
        const double2 *src = psi + b + goff_t;
#pragma unroll
        for (int k = 0; k < TSIZE / KT; ++k)
            cp_async16(buf + (swz_t ^ swz((u32)(k * KT))), src + offk[k]);
        cp_async_mbar_arrive(full + ring_bar(it));
    };
    if (grp == 0) {
        load(0);
        if (T > 2) load(2);
    } else if (T > 1) {
        load(1);
    }
    for (int it = grp; it < T; it += 2) {
        const int st = it % KSTAGES;
        const u64 tile = blockIdx.x + (u64)it * gridDim.x;
        const u64 base = tbase(tile, lane, ncomp, comp_lane);
        mbar_wait(full + ring_bar(it), (u32)((it / (2 * KSTAGES)) & 1));
        double2 *sm = bufs + st * TSIZE;
        apply_tile(sm, tid, bar, base);
        double2 *dst = psi + base + goff_t;
#pragma unroll
        for (int k = 0; k < TSIZE / KT; ++k) __stcs(dst + offk[k], sm[st_base ^ st_k[k]]);
        if (it + KSTAGES < T) {
            gsync(bar);
            load(it + KSTAGES);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}
)QSV";


// ---- expectation sweep skeleton (read-only ring; per-lane term accumulators) ----
const char *kSweepSkeleton = R"QSV(
typedef unsigned long long u64;
typedef unsigned int u32;
// SW_GROUPS tile groups of KT threads per CTA (2 x 256: each group sweeps
// its own tiles; 1 x 512: the whole CTA sweeps one tile, two more loading);
// a thread's pairs are p = pl + KT j, j < SW_NJ = 2048 / KT
#ifndef SW_GROUPS
#define SW_GROUPS 2
#endif
#define KT (512 / SW_GROUPS)
#define SW_NJ (2048 / KT)
#define KSTAGES 3
#define TSIZE 4096
// GF(2)-linear tile swizzle (16-B slots): the low 3 bits (bank group) are the
// granule index XOR the fold F of all higher 3-bit chunks; bits 3..5 become F
// itself.  So a 2^c-amplitude segment (c = 2, 3) lands in one 64 / 128-B row
// whose chunks are XOR-ed with that row's address bits 7..8 / 7..9 -- exactly
// the TMA SWIZZLE_64B / 128B pattern -- while the bank of every slot is the
// same as with the plain fold (conflict analysis unchanged).
__device__ __forceinline__ u32 swz(u32 l)
{
    const u32 f = ((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u;
    return (l & ~63u) | (f << 3) | ((l ^ f) & 7u);
}
__device__ __forceinline__ u32 ins0(u32 i, int b) { return ((i >> b) << (b + 1)) | (i & ((1u << b) - 1u)); }
__device__ __forceinline__ double wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double sgn(u32 lane, u32 sl, u64 base, u64 sh)
{
    return ((__popc(lane & sl) + __popcll(base & sh)) & 1) ? -1.0 : 1.0;
}
// Pair products w = conj(psi_l0) psi_l0^F for the thread's 8 pairs
// p = pl + 256 j (pl = lane + 32 warp; pair index = l0 with bit H removed),
// then an 8-point Walsh-Hadamard transform over j: W[m] = sum_j (-1)^{|j & m|} w_j,
// so a string whose sign mask has pair bits 8..10 = m reads W[m].  All eight
// warps of a tile group run the same group code on disjoint pairs (one
// instruction stream -> no I-cache pressure).
template <bool RE, bool IM, int H>
__device__ __forceinline__ void wht8(const double2 *sm, u32 pl, u32 sF, double (&Wr)[8], double (&Wi)[8])
{
    const u32 b0 = swz(ins0(pl, H));
#pragma unroll
    for (int j = 0; j < SW_NJ; ++j) {
        const u32 a0 = b0 ^ swz(ins0((u32)KT * j, H));
        const double2 x = sm[a0], y = sm[a0 ^ sF];
        if (RE) Wr[j] = fma(x.x, y.x, x.y * y.y);
        if (IM) Wi[j] = fma(x.x, y.y, -x.y * y.x);
    }
#pragma unroll
    for (int b = 1; b < SW_NJ; b <<= 1) {
#pragma unroll
        for (int r = 0; r < SW_NJ; ++r) {
            if (r & b) continue;
            if (RE) { const double u = Wr[r], v = Wr[r | b]; Wr[r] = u + v; Wr[r | b] = u - v; }
            if (IM) { const double u = Wi[r], v = Wi[r | b]; Wi[r] = u + v; Wi[r | b] = u - v; }
        }
    }
}
// l0-side amplitudes of the thread's 8 pairs for highest flip bit H (shared
// by every group of the sweep with that H)
template <int H>
__device__ __forceinline__ u32 load_x(const double2 *sm, u32 pl, double2 (&X)[8])
{
    const u32 b0 = swz(ins0(pl, H));
#pragma unroll
    for (int j = 0; j < SW_NJ; ++j) X[j] = sm[b0 ^ swz(ins0((u32)KT * j, H))];
    return b0;
}
// WRE / WIM: transform that component (else its strings sum the 8 products
// directly with their sign pattern: cheaper for <= 3 strings per component)
template <bool RE, bool IM, bool WRE, bool WIM, int H>
__device__ __forceinline__ void wht8x(const double2 *sm, u32 b0, const double2 (&X)[8], u32 sF,
                                      double (&Wr)[8], double (&Wi)[8])
{
#pragma unroll
    for (int j = 0; j < SW_NJ; ++j) {
        const double2 x = X[j], y = sm[b0 ^ swz(ins0((u32)KT * j, H)) ^ sF];
        if (RE) Wr[j] = fma(x.x, y.x, x.y * y.y);
        if (IM) Wi[j] = fma(x.x, y.y, -x.y * y.x);
    }
#pragma unroll
    for (int b = 1; b < SW_NJ; b <<= 1) {
#pragma unroll
        for (int r = 0; r < SW_NJ; ++r) {
            if (r & b) continue;
            if (RE && WRE) { const double u = Wr[r], v = Wr[r | b]; Wr[r] = u + v; Wr[r | b] = u - v; }
            if (IM && WIM) { const double u = Wi[r], v = Wi[r | b]; Wi[r] = u + v; Wi[r | b] = u - v; }
        }
    }
}
__device__ __forceinline__ void gsync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(KT) : "memory"); }
__device__ __forceinline__ u64 tbase(u64 tile, int lane, int ncomp, int comp_lane)
{
    u64 bit = (lane < ncomp && ((tile >> lane) & 1ull)) ? (1ull << comp_lane) : 0ull;
    u32 lo = __reduce_or_sync(0xffffffffu, (u32)bit);
    u32 hi = __reduce_or_sync(0xffffffffu, (u32)(bit >> 32));
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u32 saddr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void *d, const void *s)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void mbar_init(u64 *b, int n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *b, u32 parity)
{
    asm volatile("{\n\t.reg .pred p;\nQS_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra QS_WAIT_%=;\n\t}" ::"r"(saddr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(u64 *b)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ int ring_bar(int it) { return it % KSTAGES + KSTAGES * ((it / KSTAGES) & 1); }

// generated: every flip group of the sweep on one tile (acc[] persists across tiles)
__device__ __forceinline__ void sweep_tile(const double2 *sm, u32 pl, u64 base, double (&acc)[MAXT]);

extern "C" __global__ void __launch_bounds__(512, 1)
qsv_sweep(const double2 *__restrict__ psi, int ncomp, int c, const u64 *__restrict__ g_offhi,
          const int *__restrict__ g_geo, double *__restrict__ partial)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    u64 *full = reinterpret_cast<u64 *>(smem_raw);
    u64 *offk = reinterpret_cast<u64 *>(smem_raw + 128);  // per-k global offsets (see qsv_pass)
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw + 256);
    u64 *offhi = reinterpret_cast<u64 *>(bufs + KSTAGES * TSIZE);
    const int nhi = 1 << (12 - c);
    const u32 tid_all = threadIdx.x;
    for (int i = tid_all; i < nhi; i += 512) offhi[i] = __ldg(g_offhi + i);
    if (tid_all < TSIZE / KT) {
        const u32 l = tid_all * KT;
        offk[tid_all] = (l & ((1u << c) - 1u)) + __ldg(g_offhi + (l >> c));
    }
    if (tid_all == 0) {
        for (int s = 0; s < 2 * KSTAGES; ++s) mbar_init(full + s, KT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const u64 ntiles = 1ull << ncomp;
    const int grp = (int)(tid_all / KT);
    const u32 tid = tid_all % KT;
    const int bar = 1 + grp;
    const u32 lane = tid & 31;
    const int warp = (int)(tid >> 5);
    double acc[MAXT];
#pragma unroll
    for (int i = 0; i < MAXT; ++i) acc[i] = 0.0;
    if ((u64)blockIdx.x < ntiles) {
        const int T = (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1;
        const int comp_lane = __ldg(g_geo + lane);
        const u32 cmask = (1u << c) - 1u;
        // loop-invariant address parts (see qsv_pass): l = tid ^ KT k
        const u32 swz_t = swz(tid);
        const u64 goff_t = (u64)(tid & cmask) + offhi[tid >> c];
        auto load = [&](int it) {
            const u64 tile = blockIdx.x + (u64)it * gridDim.x;
            const u64 b = tbase(tile, lane, ncomp, comp_lane);
            double2 *buf = bufs + (it % KSTAGES) * TSIZE;
            const double2 *src = psi + b + goff_t;
#pragma unroll
            for (int k = 0; k < TSIZE / KT; ++k)
                cp_async16(buf + (swz_t ^ swz((u32)(k * KT))), src + offk[k]);
            cp_async_mbar_arrive(full + ring_bar(it));
        };
        if (SW_GROUPS == 1) {
            for (int it = 0; it < KSTAGES && it < T; ++it) load(it);
        } else if (grp == 0) {
            load(0);
            if (T > 2) load(2);
        } else if (T > 1) {
            load(1);
        }
        for (int it = grp; it < T; it += SW_GROUPS) {
            const u64 tile = blockIdx.x + (u64)it * gridDim.x;
            const u64 base = tbase(tile, lane, ncomp, comp_lane);
            mbar_wait(full + ring_bar(it), (u32)((it / (2 * KSTAGES)) & 1));
            sweep_tile(bufs + (it % KSTAGES) * TSIZE, tid, base, acc);
            if (it + KSTAGES < T) {
                gsync(bar);
                load(it + KSTAGES);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    // one row per (CTA, warp): reduce_columns sums rows in a fixed order
#ifdef SWEEP_COLS_ON
    // per-warp string sets: the row has one column per string of the sweep
    double *row = partial + (size_t)(blockIdx.x * 16 + grp * 8 + warp) * NTERMS;
    for (int i = lane; i < NTERMS; i += 32) row[i] = 0.0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
        const double v = wsum(acc[i]);
        const int col = SWEEP_COLS[warp * MAXT + i];
        if (lane == 0 && col >= 0) row[col] = v;
    }
#else
    double *row = partial + (size_t)(blockIdx.x * 16 + grp * (KT / 32) + warp) * MAXT;
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
        const double v = wsum(acc[i]);
        if (lane == 0) row[i] = v;
    }
#endif
}
)QSV";

inline uint32_t h_swz(uint32_t l) { return tile_swz(l); }
inline uint32_t h_ins0(uint32_t i, int b) { return ((i >> b) << (b + 1)) | (i & ((1u << b) - 1u)); }

struct Module {
    bool sweep = false;
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    CUdeviceptr cparams = 0;
    size_t cbytes = 0;
    unsigned threads = 512;  // 256 for compact passes (one tile group)
    bool failed = false;
    std::vector<char> cubin;
    std::string log;
};

// device -> source -> module
std::unordered_map<std::string, Module> g_mods[64];

// Optional on-disk cubin cache (QSV_JIT_CACHE=dir, default ~/.cache/qsv_jit,
// "0" disables): a pure compile-time saving, keyed by a 64-bit FNV-1a hash of
// the generated source plus its length; a hit is only used when the cached
// file also carries the exact source it was compiled from.
std::string cache_path(const std::string &src)
{
    const char *env = getenv("QSV_JIT_CACHE");
    std::string dir;
    if (env) {
        if (env[0] == '0' && env[1] == 0) return "";
        dir = env;
    } else if (const char *home = getenv("HOME")) {
        dir = std::string(home) + "/.cache/qsv_jit";
    } else {
        return "";
    }
    uint64_t h = 1469598103934665603ull;
    for (unsigned char ch : src) {
        h ^= ch;
        h *= 1099511628211ull;
    }
    char name[64];
    snprintf(name, sizeof(name), "/%016llx_%zu.bin", (unsigned long long)h, src.size());
    return dir + name;
}

bool cache_load(const std::string &path, const std::string &src, std::vector<char> &cubin)
{
    if (path.empty()) return false;
    FILE *f = fopen(path.c_str(), "rb");
    if (!f) return false;
    uint64_t ls = 0, lc = 0;
    bool ok = fread(&ls, 8, 1, f) == 1 && ls == src.size();
    std::string stored;
    if (ok) {
        stored.resize(ls);
        ok = fread(&stored[0], 1, ls, f) == ls && stored == src && fread(&lc, 8, 1, f) == 1 && lc > 0;
    }
    if (ok) {
        cubin.resize(lc);
        ok = fread(cubin.data(), 1, lc, f) == lc;
    }
    fclose(f);
    return ok;
}

void cache_store(const std::string &path, const std::string &src, const std::vector<char> &cubin)
{
    if (path.empty()) return;
    const std::string dir = path.substr(0, path.rfind('/'));
    std::string cmd_dir;
    for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
        if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)getpid());
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    const uint64_t ls = src.size(), lc = cubin.size();
    bool ok = fwrite(&ls, 8, 1, f) == 1 && fwrite(src.data(), 1, ls, f) == ls && fwrite(&lc, 8, 1, f) == 1 &&
              fwrite(cubin.data(), 1, lc, f) == lc;
    ok = (fclose(f) == 0) && ok;
    if (ok) rename(tmp.c_str(), path.c_str());
    else remove(tmp.c_str());
}

bool compile(const std::string &src, Module &m)
{
    const std::string cpath = cache_path(src);
    if (cache_load(cpath, src, m.cubin)) return true;
    nvrtcProgram prog = nullptr;
    if (g_api.CreateProgram(&prog, src.c_str(), "qsv_pass.cu", 0, nullptr, nullptr) != 0) {
        m.log = "nvrtcCreateProgram failed";
        return false;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                          "--fmad=true"};
    const int rc = g_api.CompileProgram(prog, 4, opts);
    size_t ls = 0;
    g_api.GetProgramLogSize(prog, &ls);
    if (ls > 1) {
        m.log.resize(ls);
        g_api.GetProgramLog(prog, &m.log[0]);
    }
    bool ok = rc == 0;
    if (ok) {
        size_t n = 0;
        ok = g_api.GetCUBINSize(prog, &n) == 0 && n > 0;
        if (ok) {
            m.cubin.resize(n);
            ok = g_api.GetCUBIN(prog, m.cubin.data()) == 0;
        }
    }
    g_api.DestroyProgram(&prog);
    if (ok) cache_store(cpath, src, m.cubin);
    return ok;
}

// Specialise every pass from QSV_JIT_MIN_QUBITS (default 22) qubits up; below
// that only hot programs: a cached circuit structure run QSV_JIT_HOT_USES
// (default 3; 0 = never) times -- e.g. the fixed ansatz of a VQE loop, whose
// one-off NVRTC compile is then amortised over every later evaluation.
bool jit_wanted(int n, int uses)
{
    const char *e = getenv("QSV_JIT");
    if (e && e[0] == '0') return false;
    const char *mq = getenv("QSV_JIT_MIN_QUBITS");
    const int min_q = mq ? atoi(mq) : 22;
    if (n >= min_q) return true;
    const char *hu = getenv("QSV_JIT_HOT_USES");
    const int hot = hu ? atoi(hu) : 3;
    return hot > 0 && uses >= hot && n >= kMaxTileBits;
}

}  // namespace

bool jit_source(const TileGeom &g, const BlockRec *blocks, int nblocks, const OpRec *ops,
                const RotRec *rots, int nparams, std::string &src)
{
    if (g.m != kMaxTileBits || kBlockBits != 4 || nparams > 8192) return false;
    constexpr int TB = kMaxTileBits - kBlockBits;  // 8 thread-index bits
    std::string body;
    body.reserve(4096 + 160 * nblocks);
    char buf[256];
    // Compact form (QSV_COMPACT_GMAT=1) for passes over few tiles made only of
    // fused rotation groups: a data-driven block loop with ONE copy of the
    // group code (gm_run, table offsets at run time) instead of straight-line
    // code that runs once per warp.  A/B on config 1 (B200,
    // profiles/r02_ucc12_compact_ab.txt): the instruction-fetch stalls go
    // (ncu "no_instructions" 68 % -> 2 %) but the run-time-indexed constant
    // loads (LDC, MIO-throttled) and 1.6x the instructions take their place:
    // the same ~0.22 ms per pass under ncu, slower live -- straight-line code
    // stays the default.
    int n_gmat = 0;
    for (int bi = 0; bi < nblocks; ++bi)
        for (int k = blocks[bi].op0; k < blocks[bi].op1; ++k) n_gmat += ops[k].type == OP_GMAT;
    bool all_gmat = nblocks > 0;
    for (int bi = 0; bi < nblocks && all_gmat; ++bi) {
        if (blocks[bi].kind != 0) all_gmat = false;
        for (int k = blocks[bi].op0; k < blocks[bi].op1 && all_gmat; ++k)
            all_gmat = ops[k].type == OP_GMAT && (ops[k].p & 1) == 0;  // 16-B aligned matrices
    }
    const char *env_cg = getenv("QSV_COMPACT_GMAT");
    const bool compact = all_gmat && env_cg && env_cg[0] == '1' && g.ncomp <= 3 && n_gmat >= 16;
    std::vector<unsigned long long> gmd_shi;
    std::vector<unsigned> gmd_pk;
    std::vector<int> gmd_p;
    if (compact) {
        // data-driven block loop: ONE copy of the block code (loads, the
        // GMAT dispatch, stores) walks a constant table of blocks and groups
        std::vector<unsigned> bd;
        for (int bi = 0; bi < nblocks; ++bi) {
            const BlockRec &B = blocks[bi];
            bd.push_back((unsigned)B.tswz);
            for (int i = 0; i < 12; ++i) bd.push_back((unsigned)B.cols[i]);
            bd.push_back((unsigned)gmd_pk.size());
            for (int k = B.op0; k < B.op1; ++k) {
                const RotRec &rc = rots[ops[k].r0];
                const unsigned zb = ((unsigned)rc.q >> 8) & 15u, zt = (unsigned)rc.q >> 12;
                gmd_shi.push_back((unsigned long long)rc.s_hi);
                gmd_pk.push_back((ops[k].f & 15u) | (zb << 4) | (zt << 8));
                gmd_p.push_back(ops[k].p);
            }
            bd.push_back((unsigned)gmd_pk.size());
            bd.push_back(bi + 1 < nblocks && (blocks[bi + 1].pad0 & 1) ? 1u : 0u);
        }
        // global (L1-cached) tables: the 64 KiB constant bank holds the pass parameters
        std::string tab = "__device__ const unsigned BD[" + std::to_string(bd.size()) + "] = {";
        for (size_t i = 0; i < bd.size(); ++i) tab += (i ? "," : "") + std::to_string(bd[i]) + "u";
        tab += "};\n";
        char big[2048];
        snprintf(big, sizeof(big),
                 "#pragma unroll 1\n  for (int bi = 0; bi < %d; ++bi) {\n"
                 "    const unsigned *B = BD + 16 * bi;\n"
                 "    u32 sb = B[0];\n"
                 "#pragma unroll\n    for (int i = 0; i < %d; ++i) sb ^= tb(tid, i, B[1 + i]);\n"
                 "    const u32 e1 = B[1 + %d], e2 = B[2 + %d], e4 = B[3 + %d], e8 = B[4 + %d];\n"
                 "    double2 a[16];\n"
                 "#pragma unroll\n    for (int r = 0; r < 16; ++r)\n"
                 "      a[r] = sm[sb ^ ((r & 1) ? e1 : 0u) ^ ((r & 2) ? e2 : 0u) ^ ((r & 4) ? e4 : 0u) ^ ((r & 8) ? e8 : 0u)];\n"
                 "    gm_run(a, tid, base, (int)B[13], (int)B[14]);\n"
                 "#pragma unroll\n    for (int r = 0; r < 16; ++r)\n"
                 "      sm[sb ^ ((r & 1) ? e1 : 0u) ^ ((r & 2) ? e2 : 0u) ^ ((r & 4) ? e4 : 0u) ^ ((r & 8) ? e8 : 0u)] = a[r];\n"
                 "    if (B[15]) __syncwarp(); else gsync(bar);\n  }\n",
                 nblocks, TB, TB, TB, TB, TB);
        body = tab + "@@BODY@@" + big;
        nblocks = 0;  // the straight-line emission below is skipped
    }
    for (int bi = 0; bi < nblocks; ++bi) {
        const BlockRec &B = blocks[bi];
        if (B.kind != 0) return false;
        for (int k = B.op0; k < B.op1; ++k) {
            const int t = ops[k].type;
            if (t != OP_U1 && t != OP_U1C && t != OP_U2 && t != OP_DIAG1 && t != OP_GMAT && t != OP_CX &&
                t != OP_SWAP && t != OP_X)
                return false;
        }
        snprintf(buf, sizeof(buf), "  {\n    const u32 sb = %uu", (unsigned)B.tswz);
        body += buf;
        for (int i = 0; i < TB; ++i) {
            snprintf(buf, sizeof(buf), " ^ tb(tid, %d, %uu)", i, (unsigned)B.cols[i]);
            body += buf;
        }
        body += ";\n    double2 a[16];\n";
        unsigned E[16];
        for (int r = 0; r < 16; ++r) {
            unsigned o = 0;
            for (int j = 0; j < 4; ++j)
                if ((r >> j) & 1) o ^= B.cols[TB + j];
            E[r] = o;
            snprintf(buf, sizeof(buf), "    a[%d] = sm[sb ^ %uu];\n", r, o);
            body += buf;
        }
        for (int k = B.op0; k < B.op1; ++k) {
            const OpRec &op = ops[k];
            if (op.type == OP_U1) {
                const int cls = ((op.h >= 0 && op.h <= 4) || op.h == 6) ? op.h : 0;
                snprintf(buf, sizeof(buf), "    u1<%d, %d, %d>(a);\n", op.a, cls, op.p);
            } else if (op.type == OP_U1C) {
                const int cls = (op.h == 1 || op.h == 4) ? op.h : 0;
                snprintf(buf, sizeof(buf), "    u1c<%d, %d, %d, %d>(a);\n", op.a, op.b, cls, op.p);
            } else if (op.type == OP_U2) {
                snprintf(buf, sizeof(buf), "    u2<%d, %d, %d>(a);\n", op.a, op.b, op.p);
            } else if (op.type == OP_CX) {
                snprintf(buf, sizeof(buf), "    pcx<%d, %d>(a);\n", op.a, op.b);
            } else if (op.type == OP_SWAP) {
                snprintf(buf, sizeof(buf), "    pswap<%d, %d>(a);\n", op.a, op.b);
            } else if (op.type == OP_X) {
                snprintf(buf, sizeof(buf), "    px<%d>(a);\n", op.a);
            } else if (op.type == OP_GMAT) {
                // common sign masks of the group (qsv_planner.cpp block_pass)
                const RotRec &rc = rots[op.r0];
                const unsigned zb = ((unsigned)rc.q >> 8) & 15u, zt = (unsigned)rc.q >> 12;
                snprintf(buf, sizeof(buf),
                         "    gm<%u, %d, %u>(a, (u32)((__popcll(base & %lluull) + __popc(tid & %uu)) & 1));\n",
                         op.f, op.p, zb, (unsigned long long)rc.s_hi, zt);
            } else if (op.a >= 0) {
                snprintf(buf, sizeof(buf), "    dg<%d, %d>(a);\n", op.a, op.p);
            } else {
                snprintf(buf, sizeof(buf), "    dgt<%d>(a, (tid >> %d) & 1u);\n", op.p, op.b);
            }
            body += buf;
        }
        for (int r = 0; r < 16; ++r) {
            snprintf(buf, sizeof(buf), "    sm[sb ^ %uu] = a[%d];\n", E[r], r);
            body += buf;
        }
        // group barrier, or only __syncwarp when the next block keeps this
        // warp's W-coset of slots (BlockRec.pad0 bit 0, qsv_planner.cpp)
        if (bi + 1 < nblocks && (blocks[bi + 1].pad0 & 1)) body += "  }\n  __syncwarp();\n";
        else body += "  }\n  gsync(bar);\n";
    }
    snprintf(buf, sizeof(buf), "#define QSV_NPARAMS %d\n", std::max(1, nparams));
    src = buf;
    if (!gmd_pk.empty()) {
        const size_t nd = gmd_pk.size();
        src += "#define QSV_GMD 1\n__device__ const unsigned long long GMD_SHI[" + std::to_string(nd) + "] = {";
        for (size_t i = 0; i < nd; ++i) src += (i ? "," : "") + std::to_string(gmd_shi[i]) + "ull";
        src += "};\n__device__ const unsigned GMD_PK[" + std::to_string(nd) + "] = {";
        for (size_t i = 0; i < nd; ++i) src += (i ? "," : "") + std::to_string(gmd_pk[i]) + "u";
        src += "};\n__device__ const int GMD_P[" + std::to_string(nd) + "] = {";
        for (size_t i = 0; i < nd; ++i) src += (i ? "," : "") + std::to_string(gmd_p[i]);
        src += "};\n";
    }
    std::string tile_body = body;
    const size_t at = body.find("@@BODY@@");
    if (at != std::string::npos) {  // compact: block table before the skeleton, loop inside
        src += body.substr(0, at);
        tile_body = body.substr(at + 8);
    }
    src += kSkeleton;
    src += "__device__ __forceinline__ void apply_tile(double2 *sm, u32 tid, int bar, u64 base)\n{\n";
    src += tile_body;
    src += "}\n";
    return true;
}


// Specialised expectation sweep: flip groups only (Z-only strings stay on the
// interpreted sweep, whose in-tile Walsh-Hadamard transform serves thousands
// of them at once).  Groups go to the 8 warps of a tile group by
// longest-processing-time on cost = pairs x (2 + 2 + terms); each warp keeps
// one per-lane accumulator per string across all of its tiles, so the warp
// reduction happens once per kernel instead of once per (tile, string).
// Pair-bit sweep code for the flip groups gl (in that order): per H run one
// load of the l0-side amplitudes, per group (or share class) the l1-side
// loads, products, 8-point transform / direct sums; string t accumulates
// into acc[slot[t]].  Uses `pl` (0..255, the thread's pair base) and `base`.
static void emit_pairbit(const SweepPlan &sp, const std::vector<size_t> &gl, const std::vector<int> &slot,
                         std::string &fn, int nj = 8)
{
    // nj = pairs per thread (8: groups of 256 threads, 4: one group of 512);
    // pair index p = pl + nt j with pl < nt = 2048 / nj
    const unsigned nt = 2048u / (unsigned)nj;
    const int lnt = nj == 8 ? 8 : 9, lnj = nj == 8 ? 3 : 2;
    char buf[512];
    int prev_h = -1;
    // a component with <= kDirect strings skips its 8-point transform
    // (24 adds) and sums each string's 8 products directly (7 adds)
    const int kDirect = nj == 8 ? 3 : 2;
    auto direct = [&](const GroupRec &G) {
        return G.t_im - G.t0 <= kDirect && G.t1 - G.t_im <= kDirect;
    };
    // tile positions of pair bits 8..10 for highest flip bit H (ins0 skips H)
    auto rpos = [&](int H, int k) { return (lnt + k) + ((lnt + k) >= H ? 1 : 0); };
    const char *env_share = getenv("QSV_SWEEP_SHARE");
    const bool share = !(env_share && env_share[0] == '0');
    const char *env_fs = getenv("QSV_SWEEP_FUSE1");  // 0: product + add even for single strings
    const bool fuse_single = !(env_fs && env_fs[0] == '0');
    auto sign_expr = [&](const TermRec &tr) {
        snprintf(buf, sizeof(buf), "((__popc(pl & %uu) + __popcll(base & %lluull)) & 1) ? %.17g : %.17g",
                 tr.s_loc & (nt - 1u), (unsigned long long)tr.s_hi, -tr.scale, tr.scale);
        return std::string(buf);
    };
    size_t gi = 0;
    while (gi < gl.size()) {
        const GroupRec &G = sp.groups[gl[gi]];
        if (G.h != prev_h) {  // new run of groups with this highest flip bit
            if (prev_h >= 0) fn += "  }\n";
            snprintf(buf, sizeof(buf), "  { double2 X[8];\n    const u32 b0 = load_x<%d>(sm, pl, X);\n", G.h);
            fn += buf;
            prev_h = G.h;
        }
        if (share && direct(G)) {
            // groups whose flips differ from G's only in the pair-bit positions
            // 8..10 read a permutation of G's l1-side amplitudes: ONE load of
            // y_j serves them all (member k uses pair j ^ d_k)
            uint32_t R = 0;
            for (int k = 0; k < lnj; ++k) R |= 1u << rpos(G.h, k);
            std::vector<std::pair<size_t, unsigned>> cls{{gl[gi], 0u}};
            size_t k = gi + 1;
            while (k < gl.size() && sp.groups[gl[k]].h == G.h && direct(sp.groups[gl[k]]) &&
                   ((sp.groups[gl[k]].f_loc ^ G.f_loc) & ~R) == 0) {
                const uint32_t D = sp.groups[gl[k]].f_loc ^ G.f_loc;
                unsigned d = 0;
                for (int q = 0; q < lnj; ++q) d |= ((D >> rpos(G.h, q)) & 1u) << q;
                cls.push_back({gl[k], d});
                ++k;
            }
            fn += "  {\n";
            for (const auto &m : cls)
                for (int t = sp.groups[m.first].t0; t < sp.groups[m.first].t1; ++t) {
                    snprintf(buf, sizeof(buf), "    double s%d = 0.0;\n", t);
                    fn += buf;
                }
            for (unsigned J = 0; J < (unsigned)nj; ++J) {
                snprintf(buf, sizeof(buf),
                         "    { const double2 y = sm[b0 ^ swz(ins0(%uu, %d)) ^ %uu];\n", nt * J, G.h,
                         h_swz(G.f_loc));
                fn += buf;
                for (size_t q = 0; q < cls.size(); ++q) {
                    const GroupRec &M = sp.groups[cls[q].first];
                    const unsigned jj = J ^ cls[q].second;
                    // a component with ONE string accumulates its product
                    // straight into the string's sum (2 DFMA, negation free)
                    // instead of product (DMUL + DFMA) + add
                    const bool fuse_re = fuse_single && M.t_im - M.t0 == 1;
                    const bool fuse_im = fuse_single && M.t1 - M.t_im == 1;
                    if (M.t_im > M.t0 && !fuse_re) {
                        snprintf(buf, sizeof(buf), "      const double r%zu = fma(X[%u].x, y.x, X[%u].y * y.y);\n",
                                 q, jj, jj);
                        fn += buf;
                    }
                    if (M.t1 > M.t_im && !fuse_im) {
                        snprintf(buf, sizeof(buf), "      const double i%zu = fma(X[%u].x, y.y, -X[%u].y * y.x);\n",
                                 q, jj, jj);
                        fn += buf;
                    }
                    for (int t = M.t0; t < M.t1; ++t) {
                        const TermRec &tr = sp.terms[t];
                        const unsigned msk = (tr.s_loc >> lnt) & (unsigned)(nj - 1);
                        const bool neg = __builtin_popcount(jj & msk) & 1;
                        if (tr.use_im ? fuse_im : fuse_re) {
                            if (tr.use_im)  // Im(conj x y) = x.re y.im - x.im y.re
                                snprintf(buf, sizeof(buf), "      s%d = fma(%sX[%u].x, y.y, fma(%sX[%u].y, y.x, s%d));\n",
                                         t, neg ? "-" : "", jj, neg ? "" : "-", jj, t);
                            else  // Re(conj x y) = x.re y.re + x.im y.im
                                snprintf(buf, sizeof(buf), "      s%d = fma(%sX[%u].x, y.x, fma(%sX[%u].y, y.y, s%d));\n",
                                         t, neg ? "-" : "", jj, neg ? "-" : "", jj, t);
                        } else {
                            snprintf(buf, sizeof(buf), "      s%d %s= %c%zu;\n", t, neg ? "-" : "+",
                                     tr.use_im ? 'i' : 'r', q);
                        }
                        fn += buf;
                    }
                }
                fn += "    }\n";
            }
            for (const auto &m : cls)
                for (int t = sp.groups[m.first].t0; t < sp.groups[m.first].t1; ++t) {
                    snprintf(buf, sizeof(buf), "    acc[%d] = fma(", slot[t]);
                    fn += buf;
                    fn += sign_expr(sp.terms[t]);
                    snprintf(buf, sizeof(buf), ", s%d, acc[%d]);\n", t, slot[t]);
                    fn += buf;
                }
            fn += "  }\n";
            gi = k;
            continue;
        }
        const bool need_re = G.t_im > G.t0, need_im = G.t1 > G.t_im;
        const bool w_re = G.t_im - G.t0 > kDirect, w_im = G.t1 - G.t_im > kDirect;
        snprintf(buf, sizeof(buf),
                 "  { double Wr[8], Wi[8];\n    wht8x<%s, %s, %s, %s, %d>(sm, b0, X, %uu, Wr, Wi);\n",
                 need_re ? "true" : "false", need_im ? "true" : "false", w_re ? "true" : "false",
                 w_im ? "true" : "false", G.h, h_swz(G.f_loc));
        fn += buf;
        for (int t = G.t0; t < G.t1; ++t) {
            const TermRec &tr = sp.terms[t];
            const char *W = tr.use_im ? "Wi" : "Wr";
            const unsigned msk = (tr.s_loc >> lnt) & (unsigned)(nj - 1);
            std::string val;
            if (tr.use_im ? w_im : w_re) {
                snprintf(buf, sizeof(buf), "%s[%u]", W, msk);
                val = buf;
            } else {  // W[m] of the transform = sum_j (-1)^{|j & m|} w_j
                val = "(";
                for (unsigned j = 0; j < (unsigned)nj; ++j) {
                    snprintf(buf, sizeof(buf), "%s%s[%u]", j == 0 ? "" : (__builtin_popcount(j & msk) & 1) ? " - " : " + ", W, j);
                    val += buf;
                }
                val += ")";
            }
            // scale folded in: the term's sweep total is scale * sum_p sign(p) w_p
            snprintf(buf, sizeof(buf), "    acc[%d] = fma(", slot[t]);
            fn += buf;
            fn += sign_expr(tr);
            fn += ", " + val;
            snprintf(buf, sizeof(buf), ", acc[%d]);\n", slot[t]);
            fn += buf;
        }
        fn += "  }\n";
        ++gi;
    }
    if (prev_h >= 0) fn += "  }\n";
}

// Pair-bit share classes in group order: maximal runs of direct groups with
// the same highest flip bit whose flips differ only in pair-bit positions
// (emit_pairbit loads their l1 side once); other groups are units of their own.
static std::vector<std::vector<size_t>> pairbit_units(const SweepPlan &sp)
{
    const int kDirect = 3;
    auto direct = [&](const GroupRec &G) { return G.t_im - G.t0 <= kDirect && G.t1 - G.t_im <= kDirect; };
    auto rpos = [](int H, int k) { return (8 + k) + ((8 + k) >= H ? 1 : 0); };
    std::vector<std::vector<size_t>> units;
    size_t gi = 0;
    while (gi < sp.groups.size()) {
        const GroupRec &G = sp.groups[gi];
        std::vector<size_t> u{gi};
        size_t k = gi + 1;
        if (direct(G)) {
            uint32_t R = 0;
            for (int q = 0; q < 3; ++q) R |= 1u << rpos(G.h, q);
            while (k < sp.groups.size() && sp.groups[k].h == G.h && direct(sp.groups[k]) &&
                   ((sp.groups[k].f_loc ^ G.f_loc) & ~R) == 0)
                u.push_back(k++);
        }
        units.push_back(u);
        gi = k;
    }
    return units;
}

// Per-warp specialised sweep: the sweep's flip groups are split over the 8
// warps of a tile group (share classes kept whole, longest-processing-time on
// their strings), each warp running ITS groups over all 2048 pairs of the
// tile (8 rounds of 32 lanes) with its own <= 24 per-lane accumulators.  A
// sweep therefore holds up to 8 x 24 strings instead of 24, so a config-3
// expectation needs about half the HBM sweeps (the tile-capacity bound).
bool jit_sweep_source_warps(const SweepPlan &sp, std::string &src)
{
    const int kWarps = 8, kCap = 24;
    const int nterms = (int)sp.terms.size();
    std::vector<std::vector<size_t>> units = pairbit_units(sp);
    auto ustr = [&](const std::vector<size_t> &u) {
        int n = 0;
        for (size_t g : u) n += sp.groups[g].t1 - sp.groups[g].t0;
        return n;
    };
    // split classes that cannot fit a warp
    std::vector<std::vector<size_t>> uu;
    for (auto &u : units) {
        if (ustr(u) <= kCap) {
            uu.push_back(u);
        } else {
            for (size_t g : u) uu.push_back({g});
        }
    }
    std::vector<std::vector<size_t>> wu;
    std::vector<int> load;
    // longest-processing-time over the warps; if the share classes do not
    // pack, pack single groups (the planner checked that those fit)
    auto pack = [&]() {
        std::vector<size_t> ord(uu.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
        std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return ustr(uu[a]) > ustr(uu[b]); });
        wu.assign(kWarps, {});
        load.assign(kWarps, 0);
        for (size_t i : ord) {
            const int n = ustr(uu[i]);
            int best = -1;
            for (int w = 0; w < kWarps; ++w)
                if (load[w] + n <= kCap && (best < 0 || load[w] < load[best])) best = w;
            if (best < 0) return false;
            wu[best].push_back(i);
            load[best] += n;
        }
        return true;
    };
    if (!pack()) {
        uu.clear();
        for (size_t g = 0; g < sp.groups.size(); ++g) uu.push_back({g});
        if (!pack()) return false;
    }
    int maxt = 1;
    for (int w = 0; w < kWarps; ++w) maxt = std::max(maxt, load[w]);
    std::vector<int> slot(nterms, -1), cols(kWarps * maxt, -1);
    std::string fn = "__device__ __forceinline__ void sweep_tile(const double2 *sm, u32 tid, u64 base, double (&acc)[MAXT])\n{\n"
                     "  const u32 lane = tid & 31u;\n  switch (tid >> 5) {\n";
    char buf[256];
    for (int w = 0; w < kWarps; ++w) {
        if (wu[w].empty()) continue;
        // the warp's groups in sweep order (keeps H runs adjacent)
        std::vector<size_t> units_w = wu[w];
        std::sort(units_w.begin(), units_w.end(), [&](size_t a, size_t b) { return uu[a][0] < uu[b][0]; });
        std::vector<size_t> gl;
        int k = 0;
        for (size_t ui : units_w)
            for (size_t g : uu[ui]) {
                gl.push_back(g);
                for (int t = sp.groups[g].t0; t < sp.groups[g].t1; ++t) {
                    slot[t] = k;
                    cols[w * maxt + k] = t;
                    ++k;
                }
            }
        snprintf(buf, sizeof(buf), "  case %d: {\n#pragma unroll 1\n  for (u32 q = 0; q < 8u; ++q) {\n  const u32 pl = lane + 32u * q;\n", w);
        fn += buf;
        emit_pairbit(sp, gl, slot, fn);
        fn += "  } } break;\n";
    }
    fn += "  default: break;\n  }\n}\n";
    std::string head;
    snprintf(buf, sizeof(buf), "#define MAXT %d\n#define NTERMS %d\n#define SWEEP_COLS_ON 1\n", maxt, nterms);
    head = buf;
    head += "__constant__ int SWEEP_COLS[" + std::to_string(kWarps * maxt) + "] = {";
    for (size_t i = 0; i < cols.size(); ++i) head += (i ? "," : "") + std::to_string(cols[i]);
    head += "};\n";
    src = head;
    src += kSweepSkeleton;
    src += fn;
    return true;
}

// Register-coset sweep.  The specialised sweep above is bound by shared-memory
// bandwidth (LSU shared wavefronts at 73-84 % of peak, profiles/r02_sweep_ncu.txt):
// every flip group re-reads 32 KiB of partner amplitudes per tile.  Here the
// groups of a sweep are packed into PHASES whose flips span a subspace V of
// the tile bits with dim V <= 4; in a phase each of the 256 threads of a tile
// group loads ONE coset w + V (16 amplitudes, 64 KiB per tile in total) into
// registers and forms the pair products of EVERY group of the phase from
// registers (a flip F in V pairs coset elements c and c ^ F).  V's basis is
// kept in reduced echelon form with pivots = highest bits, so F's highest bit
// is a pivot and the pair representative (that bit clear) is a static coset
// coordinate; the coset bases w range over the complement W = {pivot bits
// 0}, whose basis is ordered so that swz(w) mod 8 differs across each
// quarter-warp (conflict-free 16-B loads).  Per string the sign of pair c is
// (-1)^{|w & s|} (thread) x (-1)^{|vec(c) & s|} (static, a character of the
// 3 non-pivot-H coordinates -> an 8-point Walsh-Hadamard index).
bool jit_sweep_source_coset(const SweepPlan &sp, std::string &src)
{
    const int nterms = (int)sp.terms.size();
    if (nterms > 48) return false;
    struct Phase {
        uint32_t b[4] = {0, 0, 0, 0};
        int piv[4] = {-1, -1, -1, -1};
        int dim = 0;
        std::vector<size_t> groups;
        uint32_t reduce(uint32_t v) const
        {
            for (int i = 0; i < dim; ++i)
                if ((v >> piv[i]) & 1u) v ^= b[i];
            return v;
        }
        void insert(uint32_t v)
        {
            v = reduce(v);
            if (!v) return;
            const int p = 31 - __builtin_clz(v);
            for (int i = 0; i < dim; ++i)
                if ((b[i] >> p) & 1u) b[i] ^= v;
            b[dim] = v;
            piv[dim] = p;
            ++dim;
        }
        uint32_t vec(unsigned c) const
        {
            uint32_t v = 0;
            for (int i = 0; i < 4; ++i)
                if ((c >> i) & 1u) v ^= b[i];
            return v;
        }
        unsigned coord(uint32_t v) const
        {
            unsigned c = 0;
            for (int i = 0; i < 4; ++i)
                if ((v >> piv[i]) & 1u) c |= 1u << i;
            return c;
        }
    };
    // greedy phases: heaviest groups first; a group joins the current phase
    // if its flip is already spanned or the span can still grow
    std::vector<size_t> order(sp.groups.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return sp.groups[a].t1 - sp.groups[a].t0 > sp.groups[b].t1 - sp.groups[b].t0;
    });
    std::vector<Phase> phases;
    std::vector<bool> used(sp.groups.size(), false);
    for (size_t oi = 0; oi < order.size(); ++oi) {
        if (used[order[oi]]) continue;
        Phase ph;
        ph.insert(sp.groups[order[oi]].f_loc);
        ph.groups.push_back(order[oi]);
        used[order[oi]] = true;
        for (;;) {
            // every group the span already holds is free: take them all
            for (size_t oj = oi + 1; oj < order.size(); ++oj) {
                const size_t g = order[oj];
                if (!used[g] && ph.reduce(sp.groups[g].f_loc) == 0) {
                    ph.groups.push_back(g);
                    used[g] = true;
                }
            }
            if (ph.dim >= 4) break;
            // grow the span by the next heaviest group
            size_t pick = order.size();
            for (size_t oj = oi + 1; oj < order.size(); ++oj)
                if (!used[order[oj]]) {
                    pick = oj;
                    break;
                }
            if (pick == order.size()) break;
            ph.insert(sp.groups[order[pick]].f_loc);
            ph.groups.push_back(order[pick]);
            used[order[pick]] = true;
        }
        for (int q = 0; ph.dim < 4 && q < kMaxTileBits; ++q) ph.insert(1u << q);  // pad to 4 dims
        // pivots ascending in basis order (cosmetic; coordinates follow)
        phases.push_back(ph);
    }
    char buf[512];
    std::string fn = "__device__ __forceinline__ void sweep_tile(const double2 *sm, u32 pl, u64 base, double (&acc)[MAXT])\n{\n";
    const int kDirect = 3;
    for (const Phase &ph : phases) {
        // complement basis: non-pivot unit vectors; the first three chosen so
        // that swz(.) mod 8 is independent (quarter-warp conflict freedom)
        std::vector<uint32_t> unit;
        for (int q = 0; q < kMaxTileBits; ++q) {
            bool pv = false;
            for (int i = 0; i < 4; ++i) pv |= ph.piv[i] == q;
            if (!pv) unit.push_back(1u << q);
        }
        std::vector<uint32_t> U;
        {
            bool found = false;
            for (size_t a = 0; a < unit.size() && !found; ++a)
                for (size_t b2 = 0; b2 < unit.size() && !found; ++b2)
                    for (size_t c2 = 0; c2 < unit.size() && !found; ++c2) {
                        if (a == b2 || a == c2 || b2 == c2) continue;
                        const uint32_t x0 = h_swz(unit[a]) & 7u, x1 = h_swz(unit[b2]) & 7u,
                                       x2 = h_swz(unit[c2]) & 7u;
                        if (x0 && x1 && x2 && x0 != x1 && (x0 ^ x1) != x2 && x2 != x0 && x2 != x1) {
                            U = {unit[a], unit[b2], unit[c2]};
                            for (size_t d = 0; d < unit.size(); ++d)
                                if (d != a && d != b2 && d != c2) U.push_back(unit[d]);
                            found = true;
                        }
                    }
            if (!found) U = unit;
        }
        fn += "  {\n    u32 w = 0u, sw = 0u;\n";
        for (int i = 0; i < 8; ++i) {
            snprintf(buf, sizeof(buf), "    if ((pl >> %d) & 1u) { w ^= %uu; sw ^= %uu; }\n", i, U[i],
                     h_swz(U[i]));
            fn += buf;
        }
        fn += "    double2 A[16];\n";
        for (unsigned cc = 0; cc < 16; ++cc) {
            snprintf(buf, sizeof(buf), "    A[%u] = sm[sw ^ %uu];\n", cc, h_swz(ph.vec(cc)));
            fn += buf;
        }
        for (size_t g : ph.groups) {
            const GroupRec &G = sp.groups[g];
            const unsigned cF = ph.coord(G.f_loc);
            int mH = -1;
            for (int i = 0; i < 4; ++i)
                if (ph.piv[i] == G.h) mH = i;
            if (mH < 0 || !((cF >> mH) & 1u)) return false;  // cannot happen (echelon form)
            int other[3], no = 0;
            for (int i = 0; i < 4; ++i)
                if (i != mH) other[no++] = i;
            const bool need_re = G.t_im > G.t0, need_im = G.t1 > G.t_im;
            const bool w_re = G.t_im - G.t0 > kDirect, w_im = G.t1 - G.t_im > kDirect;
            fn += "    { double Wr[8], Wi[8];\n";
            for (unsigned k = 0; k < 8; ++k) {
                unsigned cc = 0;
                for (int j = 0; j < 3; ++j)
                    if ((k >> j) & 1u) cc |= 1u << other[j];
                const unsigned cy = cc ^ cF;
                if (need_re) {
                    snprintf(buf, sizeof(buf), "      Wr[%u] = fma(A[%u].x, A[%u].x, A[%u].y * A[%u].y);\n", k, cc, cy,
                             cc, cy);
                    fn += buf;
                }
                if (need_im) {
                    snprintf(buf, sizeof(buf), "      Wi[%u] = fma(A[%u].x, A[%u].y, -A[%u].y * A[%u].x);\n", k, cc,
                             cy, cc, cy);
                    fn += buf;
                }
            }
            auto emit_wht = [&](const char *W) {
                for (int bb = 1; bb < 8; bb <<= 1)
                    for (int r = 0; r < 8; ++r) {
                        if (r & bb) continue;
                        snprintf(buf, sizeof(buf), "      { const double u = %s[%d], v = %s[%d]; %s[%d] = u + v; %s[%d] = u - v; }\n",
                                 W, r, W, r | bb, W, r, W, r | bb);
                        fn += buf;
                    }
            };
            if (need_re && w_re) emit_wht("Wr");
            if (need_im && w_im) emit_wht("Wi");
            for (int t = G.t0; t < G.t1; ++t) {
                const TermRec &tr = sp.terms[t];
                const uint32_t sl = h_ins0(tr.s_loc, G.h);  // tile-local sign mask, bit H clear
                unsigned ms = 0;
                for (int j = 0; j < 3; ++j)
                    if (__builtin_popcount(ph.b[other[j]] & sl) & 1) ms |= 1u << j;
                const char *W = tr.use_im ? "Wi" : "Wr";
                std::string val;
                if (tr.use_im ? w_im : w_re) {
                    snprintf(buf, sizeof(buf), "%s[%u]", W, ms);
                    val = buf;
                } else {
                    val = "(";
                    for (unsigned j = 0; j < 8; ++j) {
                        snprintf(buf, sizeof(buf), "%s%s[%u]",
                                 j == 0 ? "" : (__builtin_popcount(j & ms) & 1) ? " - " : " + ", W, j);
                        val += buf;
                    }
                    val += ")";
                }
                snprintf(buf, sizeof(buf),
                         "      acc[%d] = fma(((__popc(w & %uu) + __popcll(base & %lluull)) & 1) ? %.17g : %.17g, %s, acc[%d]);\n",
                         t, sl, (unsigned long long)tr.s_hi, -tr.scale, tr.scale, val.c_str(), t);
                fn += buf;
            }
            fn += "    }\n";
        }
        fn += "  }\n";
    }
    fn += "}\n";
    snprintf(buf, sizeof(buf), "#define MAXT %d\n", nterms);
    src = buf;
    src += kSweepSkeleton;
    src += fn;
    return true;
}

bool jit_sweep_source(const SweepPlan &sp, std::string &src)
{
    if (sp.global || sp.geom.m != kMaxTileBits || sp.ndiag != 0 || sp.groups.empty()) return false;
    if (sp.groups.front().pad[0] & 1) return false;  // wide groups: interpreted transform path
    {
        // QSV_SWEEP_COSET=1: register-coset sweep.  A/B on config 3 (B200,
        // profiles/r02_expect30_coset_launches.csv): shared-memory wavefronts
        // 73-84 % -> 52 % of peak, but the same 0.76-0.77 s per expectation --
        // once SMEM is relieved the sweep is latency-bound (16 warps/SM at 128
        // registers, FP64 pipe ~36 %), so the pair-bit sweep (fewer spills)
        // stays the default.
        const char *env_cs = getenv("QSV_SWEEP_COSET");
        if (env_cs && env_cs[0] == '1' && jit_sweep_source_coset(sp, src)) return true;
    }
    if (sp.groups.front().pad[0] & 1) return false;  // wide groups: interpreted transform path
    const int nterms = (int)sp.terms.size();
    {
        // QSV_SWEEP_WARPS=1: per-warp group lists (A/B on config 3: 75 sweeps
        // instead of 162 but 1.43 s instead of 0.81 s -- the eight warp code
        // paths thrash the instruction cache and unbalance the warps; see
        // profiles/r02_expect30_warps_launches.csv)
        const char *env_w = getenv("QSV_SWEEP_WARPS");
        if (env_w && env_w[0] == '1' && jit_sweep_source_warps(sp, src)) return true;
    }
    if (nterms > 48) return false;
    // QSV_SWEEP_ONETILE=1: one 512-thread group per CTA sweeps one tile while
    // the next two load (4 pairs per thread), instead of two 256-thread
    // groups on alternate tiles with one tile in flight
    const char *env_ot = getenv("QSV_SWEEP_ONETILE");
    const bool onetile = env_ot && env_ot[0] == '1';
    std::string fn = "__device__ __forceinline__ void sweep_tile(const double2 *sm, u32 pl, u64 base, double (&acc)[MAXT])\n{\n";
    std::vector<size_t> gl(sp.groups.size());
    for (size_t i = 0; i < gl.size(); ++i) gl[i] = i;
    std::vector<int> slot(nterms);
    for (int t = 0; t < nterms; ++t) slot[t] = t;
    emit_pairbit(sp, gl, slot, fn, onetile ? 4 : 8);
    fn += "}\n";
    char buf[96];
    snprintf(buf, sizeof(buf), "#define MAXT %d\n#define SW_GROUPS %d\n", nterms, onetile ? 1 : 2);
    src = buf;
    src += kSweepSkeleton;
    src += fn;
    return true;
}

bool jit_enabled(int n, int uses) { return jit_wanted(n, uses) && load_api(); }

const char *jit_unavailable_reason() { return g_api.why.c_str(); }

// Compile every not-yet-cached source in parallel (NVRTC is thread-safe),
// then load the cubins into the current context.
int jit_prepare(int device, const std::vector<const std::string *> &srcs, std::string &err)
{
    if (!load_api()) {
        err = g_api.why;
        return 1;
    }
    auto &mods = g_mods[device];
    std::vector<std::pair<const std::string *, Module *>> todo;
    for (const std::string *s : srcs) {
        auto it = mods.find(*s);
        if (it != mods.end()) continue;
        Module &m = mods[*s];
        m.sweep = s->find("qsv_sweep(") != std::string::npos;
        todo.push_back({s, &m});
    }
    if (todo.empty()) return 0;
    if (const char *dump = getenv("QSV_JIT_DUMP")) {  // debug: write the generated sources
        for (size_t i = 0; i < todo.size(); ++i) {
            char path[512];
            snprintf(path, sizeof(path), "%s/qsv_jit_%zu_%zu.cu", dump, mods.size(), i);
            if (FILE *f = fopen(path, "w")) {
                fputs(todo[i].first->c_str(), f);
                fclose(f);
            }
        }
    }
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    size_t next = 0;
    std::vector<char> ok(todo.size(), 0);
    auto worker = [&](unsigned w) {
        for (size_t i = w; i < todo.size(); i += hw) ok[i] = compile(*todo[i].first, *todo[i].second);
    };
    (void)next;
    for (unsigned w = 0; w < hw && w < todo.size(); ++w) pool.emplace_back(worker, w);
    for (auto &t : pool) t.join();
    for (size_t i = 0; i < todo.size(); ++i) {
        Module &m = *todo[i].second;
        if (!ok[i]) {
            m.failed = true;
            err = "NVRTC: " + m.log.substr(0, 2000);
            continue;
        }
        if (g_api.ModuleLoadData(&m.mod, m.cubin.data()) != 0 ||
            g_api.ModuleGetFunction(&m.fn, m.mod, m.sweep ? "qsv_sweep" : "qsv_pass") != 0 ||
            (!m.sweep && g_api.ModuleGetGlobal(&m.cparams, &m.cbytes, m.mod, "C") != 0)) {
            m.failed = true;
            err = "cuModuleLoadData / GetFunction failed";
            continue;
        }
        // the largest launch of either kind: a pass (1 KiB header for the
        // 1024-B aligned TMA stages) over c = 1 tiles (2^11 offsets)
        const int smem = 1024 + 3 * (16 << kMaxTileBits) + 8 * (1 << (kMaxTileBits - 1));
        g_api.FuncSetAttribute(m.fn, 8 /* CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES */, smem);
        if (!m.sweep && todo[i].first->find("#define QSV_GMD") != std::string::npos) m.threads = 256;
        m.cubin.clear();
        m.cubin.shrink_to_fit();
    }
    return 0;
}

// Launch a prepared pass; returns false if its module is unavailable.
bool jit_launch(int device, const std::string &src, double2 *psi, const TileDims &g,
                const uint64_t *d_offhi, const int32_t *d_geo, const double *d_params, int nparams,
                int grid, cudaStream_t st)
{
    return jit_launch_module(jit_module(device, src), psi, g, d_offhi, d_geo, d_params, nparams,
                             grid, st, ~0ull);
}

const void *jit_module(int device, const std::string &src)
{
    auto &mods = g_mods[device];
    auto it = mods.find(src);
    if (it == mods.end() || it->second.failed || !it->second.fn) return nullptr;
    return &it->second;
}

// TMA staging of the pass tiles (QSV_PASS_TMA=1; A/B against LDGSTS, which
// stays the default): the state as a 2-D tensor [2^(n-3) segments][16
// doubles], one box = one 128-B segment landing in its tile row with the
// hardware SWIZZLE_128B (= the tile swizzle's row layout, qsv_internal.h
// tile_swz).  Measured on B200 (profiles/r02_tma_ab.txt): config 2 76.8 ms vs
// 70.1 ms with LDGSTS, 30 q UCC on 128-B tiles 4.46 s vs 4.33 s -- 512 TMA
// ops of 128 B per 64 KiB tile cost more than the 16 LDGSTS per thread they
// replace.  64-B segments (c = 2) cannot use it: a swizzled TMA destination
// must be 128-B aligned (the c = 2 run faulted with a misaligned address).
bool pass_tma_map(double2 *psi, const TileDims &g, CUtensorMap *out)
{
    static const char *env = getenv("QSV_PASS_TMA");
    if (!(env && env[0] == '1') || !g_api.TensorMapEncodeTiled) return false;
    if (g.m != kMaxTileBits || g.c != 3) return false;
    const int n = g.ncomp + g.m;
    if (n - g.c > 31) return false;  // row coordinates are signed 32-bit
    cuuint64_t dims[2] = {(cuuint64_t)(2u << g.c), (cuuint64_t)1 << (n - g.c)};
    cuuint64_t strides[1] = {(cuuint64_t)16 << g.c};
    cuuint32_t box[2] = {(cuuint32_t)(2u << g.c), 1};
    cuuint32_t estr[2] = {1, 1};
    return g_api.TensorMapEncodeTiled(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)psi, dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      g.c == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == 0;
}

bool jit_launch_module(const void *mod, double2 *psi, const TileDims &g, const uint64_t *d_offhi,
                       const int32_t *d_geo, const double *d_params, int nparams, int grid,
                       cudaStream_t st, uint64_t basis)
{
    if (!mod) return false;
    const Module &m = *static_cast<const Module *>(mod);
    if (nparams > 0)
        if (g_api.MemcpyDtoDAsync(m.cparams, (CUdeviceptr)d_params, (size_t)nparams * 8, st) != 0)
            return false;
    int ncomp = g.ncomp, c = g.c;
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    int tma = pass_tma_map(psi, g, &tmap) ? 1 : 0;
    void *args[] = {&psi, &ncomp, &c, (void *)&d_offhi, (void *)&d_geo, &basis, &tmap, &tma};
    const unsigned smem = 1024 + 3 * (16u << kMaxTileBits) + 8u * (1u << (kMaxTileBits - g.c));
    return g_api.LaunchKernel(m.fn, (unsigned)grid, 1, 1, m.threads, 1, 1, smem, st, args, nullptr) == 0;
}


// Launch a prepared expectation sweep; partial gets 16 * grid rows of nterms.
bool jit_sweep_launch(int device, const std::string &src, const double2 *psi, const TileDims &g,
                      const uint64_t *d_offhi, const int32_t *d_geo, double *d_partial, int grid,
                      cudaStream_t st)
{
    auto &mods = g_mods[device];
    auto it = mods.find(src);
    if (it == mods.end() || it->second.failed || !it->second.fn) return false;
    Module &m = it->second;
    int ncomp = g.ncomp, c = g.c;
    void *args[] = {(void *)&psi, &ncomp, &c, (void *)&d_offhi, (void *)&d_geo, (void *)&d_partial};
    const unsigned smem = 256 + 3 * (16u << kMaxTileBits) + 8u * (1u << (kMaxTileBits - g.c));
    return g_api.LaunchKernel(m.fn, (unsigned)grid, 1, 1, 512, 1, 1, smem, st, args, nullptr) == 0;
}

}  // namespace qsv
