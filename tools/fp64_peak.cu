// tools/fp64_peak.cu — builder-measured FP64 throughput of this B200 (the roofline denominator for the
// FP64-bound kernels; MEASURED_PEAKS.json carries HBM and bf16 only).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak > profiles/fp64_peak.json
//
// Every thread runs 16 independent DFMA (resp. DADD, DMUL) chains, so the measurement is pipe throughput, not
// latency; grids of 148 SMs x 8 CTAs x 256 threads. Timed with CUDA events after a warm-up launch; the best
// of 5 runs. Reported as instructions/clk/SM (at the measured SM clock) and TFLOP/s (DFMA = 2 flops).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_fp64(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) x[i] = __fma_rn(x[i], a, b);
      if (OP == 1) x[i] = __dadd_rn(x[i], b);
      if (OP == 2) x[i] = __dmul_rn(x[i], a);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[threadIdx.x] = s;  // never true; keeps the chains alive
}

__global__ void k_clock(long long* out, int spin) {
  const long long t0 = clock64();
  double x = 1.0;
  for (int i = 0; i < spin; ++i) x = __fma_rn(x, 0.999999, 1e-9);
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (x == 1234.5) out[1] = 1;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount, threads = 256, ctas = sms * 8, iters = 4096;
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // SM clock under load: clock64 ticks of a long spin over its event-timed duration
  long long* ck;
  cudaMalloc(&ck, 2 * sizeof(long long));
  k_clock<<<1, 32>>>(ck, 1 << 20);
  cudaEventRecord(e0);
  k_clock<<<1, 32>>>(ck, 1 << 22);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_clk = 0;
  cudaEventElapsedTime(&ms_clk, e0, e1);
  long long ticks = 0;
  cudaMemcpy(&ticks, ck, sizeof(ticks), cudaMemcpyDeviceToHost);
  const double mhz = ticks / (ms_clk * 1e3);
  const char* names[3] = {"dfma", "dadd", "dmul"};
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"sm_mhz_measured\": %.0f, \"source\": \"tools/fp64_peak.cu (builder-measured)\"",
              p.name, sms, mhz);
  for (int op = 0; op < 3; ++op) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      if (op == 0) k_fp64<0><<<ctas, threads>>>(out, iters, 0.999999, 1e-7);
      if (op == 1) k_fp64<1><<<ctas, threads>>>(out, iters, 0.999999, 1e-7);
      if (op == 2) k_fp64<2><<<ctas, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    const double inst = static_cast<double>(ctas) * threads * iters * 16;
    const double per_s = inst / (best * 1e-3);
    std::printf(", \"%s_inst_per_s\": %.4e, \"%s_per_clk_per_sm\": %.2f", names[op], per_s, names[op],
                per_s / (sms * mhz * 1e6));
    if (op == 0) std::printf(", \"fp64_tflops\": %.2f", 2.0 * per_s / 1e12);
  }
  std::printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
