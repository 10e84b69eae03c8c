// Probe: 3-D TMA tensor store {d, groups, rows} with box {64, 1, 32}, SWIZZLE_128B, at
// coordinates (c0, c1, c2) given on the command line (negative / past-extent allowed?).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void store3d(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int two) {
  __shared__ __align__(1024) unsigned char tile[32 * 128];
  const int lane = threadIdx.x;
  for (int i = 0; i < 64; ++i) {   // row `lane`, column i: value lane * 64 + i (swizzled 16-B chunks)
    int chunk = i / 8, w = i % 8;
    __nv_bfloat16 v = __float2bfloat16((float)(lane * 64 + i));
    *reinterpret_cast<__nv_bfloat16*>(tile + lane * 128 + (((chunk ^ (lane & 7)) << 4)) + 2 * w) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    unsigned s = (unsigned)__cvta_generic_to_shared(tile);
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     (unsigned long long)&map), "r"(s), "r"(c0), "r"(c1), "r"(c2) : "memory");
    if (two)
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                       (unsigned long long)&map), "r"(s), "r"(c0 - 188), "r"(c1 + 1), "r"(c2) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  int c0 = atoi(argv[1]), c1 = atoi(argv[2]), c2 = atoi(argv[3]), two = argc > 4 ? atoi(argv[4]) : 0;
  const int d = 188, dp = 192, groups = 4, rows = 64;
  cuInit(0);
  __nv_bfloat16* buf;
  cudaMalloc(&buf, (size_t)rows * groups * dp * 2);
  cudaMemset(buf, 0xff, (size_t)rows * groups * dp * 2);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)groups, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)dp * 2, (cuuint64_t)groups * dp * 2};
  cuuint32_t box[3] = {64, 1, 32};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  store3d<<<1, 32>>>(map, c0, c1, c2, two);
  cudaError_t e = cudaDeviceSynchronize();
  printf("coords (%d,%d,%d) two=%d: %s\n", c0, c1, c2, two, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<__nv_bfloat16> h((size_t)rows * groups * dp);
  cudaMemcpy(h.data(), buf, h.size() * 2, cudaMemcpyDeviceToHost);
  int written = 0, bad = 0;
  for (int row = 0; row < rows; ++row)
    for (int g = 0; g < groups; ++g)
      for (int j = 0; j < dp; ++j) {
        unsigned short raw = *reinterpret_cast<unsigned short*>(&h[((size_t)row * groups + g) * dp + j]);
        if (raw == 0xffff) continue;
        ++written;
        float v = __bfloat162float(h[((size_t)row * groups + g) * dp + j]);
        // expected: box element (i, row - c2) with i = j - c0 (first store) or j - (c0 - 188)
        int lr = row - c2, i = (g == c1) ? j - c0 : j - (c0 - 188);
        float want = __bfloat162float(__float2bfloat16((float)(lr * 64 + i)));
        if (v != want || j >= d) ++bad;
      }
  printf("written %d bad %d\n", written, bad);
  return 0;
}
