// Probe: does a TMA tensor map accept a 0-byte global stride (to replicate
// pixels, i.e. a 2x nearest upsample inside the load)?
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void load_kernel(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3,
                            int c4, uint16_t* out, int nbytes) {
  __shared__ __align__(1024) uint8_t buf[32768];
  __shared__ __align__(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf), bb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(nbytes));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sb),
        "l"(&map), "r"(bb), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(bb));
    for (int i = 0; i < nbytes / 2; ++i) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
  }
}

int main() {
  const int C = 64, W = 8, H = 4;
  std::vector<uint16_t> h(C * W * H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int c = 0; c < C; ++c) h[(y * W + x) * C + c] = (uint16_t)(1000 * y + 10 * x + (c % 8));
  void* d; cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  uint16_t* dout; cudaMalloc(&dout, 65536);
  CUtensorMap map;
  // dims (c, rx, x, ry, y): rx / ry replicate with stride 0
  cuuint64_t dims[5] = {(cuuint64_t)C, 2, (cuuint64_t)W, 2, (cuuint64_t)H};
  cuuint64_t strides[4] = {0, (cuuint64_t)C * 2, 0, (cuuint64_t)W * C * 2};
  cuuint32_t box[5] = {64, 2, 4, 2, 2};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode stride0: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 0;
  const int nbytes = 64 * 2 * 4 * 2 * 2 * 2;
  // start: rx=0, x=-1 (OOB column), ry=1, y=0
  load_kernel<<<1, 32>>>(map, 0, 0, -1, 1, 0, dout, nbytes);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> o(nbytes / 2);
  cudaMemcpy(o.data(), dout, nbytes, cudaMemcpyDeviceToHost);
  // print element 0 of each 128-byte row, unswizzled chunk 0 sits at ((0 ^ (row&7))*16)
  for (int row = 0; row < nbytes / 128; ++row) {
    int chunk_off = ((0 ^ (row & 7)) * 16) / 2;
    printf("row %2d: %u\n", row, o[row * 64 + chunk_off]);
  }
  return 0;
}
