// dsmem_probe.cu -- the two costs that decide whether the config-1 small-state
// kernel (one 12-qubit state, 64 KiB, in one SM's shared memory) should be
// split over a thread-block cluster: the bandwidth of shared-memory reads
// from a peer CTA (DSMEM) vs local shared memory, and the latency of a
// cluster barrier vs a CTA barrier.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
constexpr int kWords = 4096;  // 32 KiB of double2 (16-B) words per CTA (static shared-memory limit)
constexpr int kIters = 64;

// every thread reads 16-B words of the local (peer = 0) or the partner CTA's
// (peer = 1) shared memory, coalesced, kIters sweeps of the 32 KiB
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads)
    read_kernel(int peer, double *out, long long *cycles)
{
    __shared__ double2 buf[kWords / 2];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < kWords / 2; i += kThreads) buf[i] = make_double2(i, -i);
    cl.sync();
    const double2 *src = peer ? cl.map_shared_rank(buf, cl.block_rank() ^ 1) : buf;
    double acc = 0.0;
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it)
        for (int i = threadIdx.x; i < kWords / 2; i += kThreads) {
            const double2 v = src[i ^ (it & 1)];
            acc += v.x + v.y;
        }
    __syncthreads();
    const long long t1 = clock64();
    cl.sync();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 12345.0) out[0] = acc;  // keep the loads
}

// n barriers back to back: CTA barrier (cluster = 0) or cluster barrier (1)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads)
    barrier_kernel(int cluster, int n, long long *cycles)
{
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (cluster)
            cl.sync();
        else
            __syncthreads();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main()
{
    double *d_out;
    long long *d_cyc, h_cyc[2];
    cudaMalloc(&d_out, 8);
    cudaMalloc(&d_cyc, 16);
    double bpc[2];
    for (int peer = 0; peer < 2; ++peer) {
        read_kernel<<<2, kThreads>>>(peer, d_out, d_cyc);  // warm-up
        read_kernel<<<2, kThreads>>>(peer, d_out, d_cyc);
        cudaMemcpy(h_cyc, d_cyc, 16, cudaMemcpyDeviceToHost);
        const double bytes = (double)kIters * (kWords / 2) * 16.0;
        bpc[peer] = bytes / (double)h_cyc[0];
    }
    const int n = 4096;
    double lat[2];
    for (int cl = 0; cl < 2; ++cl) {
        barrier_kernel<<<2, kThreads>>>(cl, n, d_cyc);
        barrier_kernel<<<2, kThreads>>>(cl, n, d_cyc);
        cudaMemcpy(h_cyc, d_cyc, 16, cudaMemcpyDeviceToHost);
        lat[cl] = (double)h_cyc[0] / n;
    }
    const cudaError_t e = cudaGetLastError();
    printf("{\"local_smem_bytes_per_clk\": %.1f, \"dsmem_bytes_per_clk\": %.1f, "
           "\"cta_barrier_clk\": %.1f, \"cluster_barrier_clk\": %.1f, \"threads\": %d, \"error\": \"%s\"}\n",
           bpc[0], bpc[1], lat[0], lat[1], kThreads, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
