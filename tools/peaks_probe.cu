// Measured FP64 / popc issue peaks of this B200 (SURVEY.md §6 asks for them:
// MEASURED_PEAKS.json only has HBM and bf16).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks_probe.cu
//   /tmp/peaks > profiles/r02_peaks.json
// Each kernel runs one persistent wave (148 SMs x resident CTAs), every thread
// carrying 8 independent dependency chains so the pipe, not latency, binds.
// Timed with CUDA events after warm-up; best of 5.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int CHAINS = 8;

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double c[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) c[k] = fma(c[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k];
  if (s == 1.2345) out[blockIdx.x] = s;  // keep the chains alive
}

// popc + xor + and: the per-(amplitude, string) parity of the expectation sweeps
__global__ void popc_kernel(unsigned *out, int iters, unsigned m) {
  unsigned c[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k] = threadIdx.x * 2654435761u + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) c[k] = __popc(c[k] & m) + c[k];
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s ^= c[k];
  if (s == 0x12345u) out[blockIdx.x] = s;
}

// DADD (the expectation's accumulate)
__global__ void dadd_kernel(double *out, int iters, double a) {
  double c[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) c[k] = c[k] + a;
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k];
  if (s == 1.2345) out[blockIdx.x] = s;
}

template <class F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double *dout;
  unsigned *uout;
  CK(cudaMalloc(&dout, 1 << 20));
  CK(cudaMalloc(&uout, 1 << 20));
  const int threads = 256, per_sm = 8;  // 64 warps / SM
  const int blocks = sms * per_sm;
  const int iters = 4096;
  const double ops = double(blocks) * threads * iters * 16 * CHAINS;

  float ms_fma = best_ms([&] { dfma_kernel<<<blocks, threads>>>(dout, iters, 0.999999, 1e-7); });
  float ms_add = best_ms([&] { dadd_kernel<<<blocks, threads>>>(dout, iters, 1e-7); });
  float ms_pop = best_ms([&] { popc_kernel<<<blocks, threads>>>(uout, iters, 0x5a5a5a5au); });
  CK(cudaGetLastError());
  double dfma_s = ops / (ms_fma * 1e-3), dadd_s = ops / (ms_add * 1e-3);
  // popc chain = LOP3 (and) + POPC + IADD: report the popc-parity triples per second
  double pop_s = ops / (ms_pop * 1e-3);
  double clk = clk_khz * 1e3;
  printf("{\"sms\": %d, \"sm_clock_attr_mhz\": %.0f, "
         "\"dfma_per_s\": %.6e, \"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_attr_clock\": %.2f, "
         "\"dadd_per_s\": %.6e, \"popc_and_add_per_s\": %.6e, "
         "\"ms\": {\"dfma\": %.3f, \"dadd\": %.3f, \"popc\": %.3f}, "
         "\"how\": \"%d CTAs x %d threads, %d independent chains/thread, %d x 16 dependent steps, best of 5 CUDA-event timings\"}\n",
         sms, clk / 1e6, dfma_s, 2 * dfma_s / 1e12, dfma_s / clk / sms, dadd_s, pop_s,
         ms_fma, ms_add, ms_pop, blocks, threads, CHAINS, iters);
  return 0;
}
