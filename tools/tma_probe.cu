// tools/tma_probe.cu — standalone check of the HWF_TMA_TILES staging (k_pixel): a 48x24 u8 box of a [planes][h][w]
// u8 tensor via one cp.async.bulk.tensor.3d completing on an mbarrier, tensor map as a __grid_constant__ parameter,
// compared with the same bytes read directly (zeros out of bounds).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu && tools/tma_probe
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#ifndef BOXW
#define BOXW 48
#endif
constexpr int kBoxW = BOXW, kBoxH = 24;
struct TmaArg {
  CUtensorMap map;
  int valid;
};
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int VAR>
__global__ void k_probe(const __grid_constant__ TmaArg tm, const CUtensorMap* gmap, int bx, int by, int plane, uint8_t* out) {
  const uint64_t desc = gmap ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&tm.map);
  __shared__ __align__(128) uint8_t box[kBoxH][kBoxW];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sh_addr(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (VAR == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sh_addr(&bar)), "r"(kBoxW * kBoxH) : "memory");
    if (VAR == 3)
      asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sh_addr(&box[0][0])), "l"(desc), "r"(bx), "r"(by), "r"(plane), "r"(sh_addr(&bar))
        : "memory");
  }
  uint32_t done = 0, phase = 0;
  do {
    if (VAR == 0)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(sh_addr(&bar)) : "memory");
    else
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(sh_addr(&bar)), "r"(phase) : "memory");
  } while (!done);
  for (int i = threadIdx.x; i < kBoxW * kBoxH; i += blockDim.x) out[i] = box[i / kBoxW][i % kBoxW];
}

int main(int argc, char** argv) {
  const int w = 640, h = 480, planes = 8;
  std::vector<uint8_t> host(static_cast<size_t>(w) * h * planes);
  for (size_t i = 0; i < host.size(); ++i) host[i] = static_cast<uint8_t>((i * 2654435761u) >> 24);
  uint8_t *d, *dout;
  cudaMalloc(&d, host.size() + 32);
  cudaMalloc(&dout, kBoxW * kBoxH);
  uint8_t* base = d + 16;
  cudaMemcpy(base, host.data(), host.size(), cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  TmaArg tm{};
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(planes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(w) * h};
  const cuuint32_t box[3] = {kBoxW, kBoxH, 1}, estr[3] = {1, 1, 1};
  const int rc = encode ? encode(&tm.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (argc > 3 && atoi(argv[3]) == 0) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                        : -1;
  tm.valid = rc == 0;
  std::printf("encode=%p rc=%d query=%d\n", reinterpret_cast<void*>(encode), rc, static_cast<int>(q));
  CUtensorMap* gmap = nullptr;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  cudaMemcpy(gmap, &tm.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  std::printf("descriptor in %s memory\n", mode ? "global" : "param");
  int bad_total = 0;
  const int cases[4][3] = {{96, 50, 3}, {-16, -5, 0}, {608, 470, 7}, {0, 0, 1}};
  for (auto& c : cases) {
    const int var = argc > 2 ? atoi(argv[2]) : 0;
    if (var == 0) k_probe<0><<<1, 128>>>(tm, mode ? gmap : nullptr, c[0], c[1], c[2], dout);
    if (var == 1) k_probe<1><<<1, 128>>>(tm, mode ? gmap : nullptr, c[0], c[1], c[2], dout);
    if (var == 2) k_probe<2><<<1, 128>>>(tm, mode ? gmap : nullptr, c[0], c[1], c[2], dout);
    if (var == 3) k_probe<3><<<1, 128>>>(tm, mode ? gmap : nullptr, c[0], c[1], c[2], dout);
    const cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint8_t> got(kBoxW * kBoxH);
    cudaMemcpy(got.data(), dout, got.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < kBoxH; ++y)
      for (int x = 0; x < kBoxW; ++x) {
        const int gx = c[0] + x, gy = c[1] + y;
        const uint8_t want = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? host[(static_cast<size_t>(c[2]) * h + gy) * w + gx] : 0;
        bad += got[y * kBoxW + x] != want;
      }
    std::printf("box (%d,%d,%d): %s, %d mismatches\n", c[0], c[1], c[2], cudaGetErrorString(e), bad);
    bad_total += bad + (e != cudaSuccess);
    if (e != cudaSuccess) break;
  }
  std::printf("%s\n", bad_total ? "FAIL" : "OK");
  return bad_total ? 1 : 0;
}
