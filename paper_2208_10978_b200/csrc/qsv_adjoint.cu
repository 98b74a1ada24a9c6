// qsv_adjoint.cu -- reverse-mode (adjoint) gradient of a product of Pauli
// rotations, all on the device (statevector.py:153-211).
//
// For U = U_R ... U_1 with U_r = exp(-i theta_r/2 P_r) and E = <psi|H|psi>,
// |psi> = U|psi0>:
//     dE/dtheta_r = 2 Re <lam_r| (-i/2) P_r |phi_r> = Im <lam_r| P_r |phi_r>,
// phi_r = U_r...U_1 psi0 (the state after rotation r) and
// lam_r = U_{r+1}^dag ... U_R^dag H|psi>.  Walking r = R-1 .. 0 both vectors
// are un-rotated in place: phi <- U_r^dag phi, lam <- U_r^dag lam, with
// U_r^dag = exp(+i theta_r/2 P_r) = cos I + i sin P_r.
//
// P convention (kernels.apply_pauli, _cykernels.pyx:76-102):
//     (P a)_j = i^{|y|} (-1)^{popc((j ^ f) & (y | z))} a_{j ^ f},   f = x | y.
//
// Small states (2^n <= 4096, both vectors in shared memory): ONE CTA runs
// the whole backward sweep -- per rotation one block reduction and one
// in-SMEM update, no launches, no host round trips.  Larger states: two
// launches per rotation (partial inner products into a [block][rotation]
// array, then the fused update of both vectors); one deterministic column
// reduction at the end.  Either way the host reads the gradient once.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qsv_internal.h"

namespace qsv {

namespace {

__device__ __forceinline__ double2 mul_ipow(double2 v, int k)  // v * i^k
{
    switch (k & 3) {
        case 0: return v;
        case 1: return make_double2(-v.y, v.x);
        case 2: return make_double2(-v.x, -v.y);
        default: return make_double2(v.y, -v.x);
    }
}

__device__ __forceinline__ uint64_t ins0_64(uint64_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1ull << b) - 1ull));
}

// Im conj(l) * w
__device__ __forceinline__ double im_cdot(double2 l, double2 w) { return l.x * w.y - l.y * w.x; }

// a <- cos a + i sin (P a) on the pair (j0, j1 = j0 ^ f), f != 0
__device__ __forceinline__ void unrotate_pair(double2 &a0, double2 &a1, uint64_t j0, uint64_t j1,
                                              uint64_t s, int ny, double c, double sn)
{
    // (P a)_{j0} = i^ny sg(j1) a1 ; (P a)_{j1} = i^ny sg(j0) a0 ; then times i sn
    double2 p0 = mul_ipow(a1, ny + 1), p1 = mul_ipow(a0, ny + 1);
    if (__popcll(j1 & s) & 1) p0 = make_double2(-p0.x, -p0.y);
    if (__popcll(j0 & s) & 1) p1 = make_double2(-p1.x, -p1.y);
    const double2 n0 = make_double2(fma(sn, p0.x, c * a0.x), fma(sn, p0.y, c * a0.y));
    const double2 n1 = make_double2(fma(sn, p1.x, c * a1.x), fma(sn, p1.y, c * a1.y));
    a0 = n0;
    a1 = n1;
}

// a_j <- (cos + i sin i^ny sg(j)) a_j  (diagonal string, f == 0)
__device__ __forceinline__ double2 unrotate_diag(double2 a, uint64_t j, uint64_t s, int ny, double c,
                                                 double sn)
{
    double2 p = mul_ipow(a, ny + 1);
    if (__popcll(j & s) & 1) p = make_double2(-p.x, -p.y);
    return make_double2(fma(sn, p.x, c * a.x), fma(sn, p.y, c * a.y));
}

constexpr int kSmemT = 1024;

__global__ void __launch_bounds__(kSmemT, 1)
adjoint_smem_kernel(double2 *__restrict__ phi_g, double2 *__restrict__ lam_g, int n, int R,
                    const uint64_t *__restrict__ X, const uint64_t *__restrict__ Y,
                    const uint64_t *__restrict__ Z, const double2 *__restrict__ cs,
                    double *__restrict__ grad)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t dim = 1u << n;
    double2 *phi = reinterpret_cast<double2 *>(smem_raw);
    double2 *lam = phi + dim;
    __shared__ double red[kSmemT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t j = tid; j < dim; j += kSmemT) {
        phi[j] = phi_g[j];
        lam[j] = lam_g[j];
    }
    __syncthreads();
    for (int r = R - 1; r >= 0; --r) {
        const uint64_t x = __ldg(X + r), y = __ldg(Y + r), z = __ldg(Z + r);
        const uint32_t f = (uint32_t)(x | y);
        const uint64_t s = y | z;
        const int ny = __popcll(y) & 3;
        // Im <lam| P |phi>
        double acc = 0.0;
        for (uint32_t j = tid; j < dim; j += kSmemT) {
            const uint32_t i = j ^ f;
            double2 w = mul_ipow(phi[i], ny);
            if (__popcll((uint64_t)i & s) & 1) w = make_double2(-w.x, -w.y);
            acc += im_cdot(lam[j], w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
        __syncthreads();  // every read of phi / lam for this rotation is done
        if (warp == 0) {
            double v = lane < kSmemT / 32 ? red[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) grad[r] = v;
        }
        const double2 csr = __ldg(cs + r);  // cos, sin of theta_r / 2 (host libm)
        const double c = csr.x, sn = csr.y;
        if (f != 0) {
            const int h = 31 - __clz(f);
            for (uint32_t p = tid; p < dim / 2; p += kSmemT) {
                const uint32_t j0 = (uint32_t)ins0_64(p, h), j1 = j0 ^ f;
                double2 a0 = phi[j0], a1 = phi[j1];
                unrotate_pair(a0, a1, j0, j1, s, ny, c, sn);
                phi[j0] = a0;
                phi[j1] = a1;
                double2 b0 = lam[j0], b1 = lam[j1];
                unrotate_pair(b0, b1, j0, j1, s, ny, c, sn);
                lam[j0] = b0;
                lam[j1] = b1;
            }
        } else {
            for (uint32_t j = tid; j < dim; j += kSmemT) {
                phi[j] = unrotate_diag(phi[j], j, s, ny, c, sn);
                lam[j] = unrotate_diag(lam[j], j, s, ny, c, sn);
            }
        }
        __syncthreads();
    }
    for (uint32_t j = tid; j < dim; j += kSmemT) {
        phi_g[j] = phi[j];
        lam_g[j] = lam[j];
    }
}

constexpr int kT = 256;

// partial[b * R + r] = block b's share of Im <lam| P_r |phi>
__global__ void __launch_bounds__(kT) adjoint_dot_kernel(const double2 *__restrict__ phi,
                                                         const double2 *__restrict__ lam,
                                                         uint64_t dim, uint64_t f, uint64_t s, int ny,
                                                         int r, int R, double *__restrict__ partial)
{
    __shared__ double red[kT / 32];
    double acc = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * kT;
    for (uint64_t j = (uint64_t)blockIdx.x * kT + threadIdx.x; j < dim; j += stride) {
        const uint64_t i = j ^ f;
        double2 w = mul_ipow(phi[i], ny);
        if (__popcll(i & s) & 1) w = make_double2(-w.x, -w.y);
        acc += im_cdot(lam[j], w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < kT / 32; ++w) v += red[w];
        partial[(size_t)blockIdx.x * R + r] = v;
    }
}

__global__ void __launch_bounds__(kT) adjoint_unrotate_kernel(double2 *__restrict__ phi,
                                                              double2 *__restrict__ lam, uint64_t dim,
                                                              uint64_t f, uint64_t s, int ny,
                                                              const double2 *__restrict__ cs, int r)
{
    const double2 csr = __ldg(cs + r);
    const double c = csr.x, sn = csr.y;
    const uint64_t stride = (uint64_t)gridDim.x * kT;
    if (f != 0) {
        const int h = 63 - __clzll(f);
        for (uint64_t p = (uint64_t)blockIdx.x * kT + threadIdx.x; p < dim / 2; p += stride) {
            const uint64_t j0 = ins0_64(p, h), j1 = j0 ^ f;
            double2 a0 = phi[j0], a1 = phi[j1];
            unrotate_pair(a0, a1, j0, j1, s, ny, c, sn);
            phi[j0] = a0;
            phi[j1] = a1;
            double2 b0 = lam[j0], b1 = lam[j1];
            unrotate_pair(b0, b1, j0, j1, s, ny, c, sn);
            lam[j0] = b0;
            lam[j1] = b1;
        }
    } else {
        for (uint64_t j = (uint64_t)blockIdx.x * kT + threadIdx.x; j < dim; j += stride) {
            phi[j] = unrotate_diag(phi[j], j, s, ny, c, sn);
            lam[j] = unrotate_diag(lam[j], j, s, ny, c, sn);
        }
    }
}

}  // namespace

int adjoint_smem_max_qubits() { return 12; }

size_t adjoint_scratch_doubles(int n, int64_t R, int device)
{
    if (n <= adjoint_smem_max_qubits()) return (size_t)R;
    return (size_t)elementwise_grid(1ull << n, device) * (size_t)R + (size_t)R;
}

// X/Y/Z/cs (cos, sin of theta/2): device arrays of R rotations in forward order; d_scratch of
// adjoint_scratch_doubles(); the gradient lands in d_grad[R].
cudaError_t launch_rotation_adjoint(double2 *phi, double2 *lam, int n, int64_t R, const uint64_t *X,
                                    const uint64_t *Y, const uint64_t *Z, const uint64_t *hX,
                                    const uint64_t *hY, const uint64_t *hZ, const double2 *cs,
                                    double *d_scratch, double *d_grad, cudaStream_t st)
{
    if (R <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t dim = 1ull << n;
    if (n <= adjoint_smem_max_qubits()) {
        const size_t smem = 32 * (size_t)dim;
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(adjoint_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 32 << 12);
            configured = true;
        }
        adjoint_smem_kernel<<<1, kSmemT, smem, st>>>(phi, lam, n, (int)R, X, Y, Z, cs, d_grad);
        return cudaGetLastError();
    }
    const int G = elementwise_grid(dim, dev);
    for (int64_t r = R - 1; r >= 0; --r) {
        const uint64_t f = hX[r] | hY[r], s = hY[r] | hZ[r];
        const int ny = __builtin_popcountll(hY[r]) & 3;
        adjoint_dot_kernel<<<G, kT, 0, st>>>(phi, lam, dim, f, s, ny, (int)r, (int)R, d_scratch);
        adjoint_unrotate_kernel<<<G, kT, 0, st>>>(phi, lam, dim, f, s, ny, cs, (int)r);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_columns(d_scratch, G, (int)R, nullptr, d_grad, st);
}

}  // namespace qsv
