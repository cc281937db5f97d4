// Check of the TMA tile::gather4 semantics the FFN's activation operand relies on:
// a 2-D tensor map over x [T][d_h] bf16 (box {64, 1}, SWIZZLE_128B); one gather4 writes
// rows r0..r3 (128 B each) at smem dst .. dst+511 and must leave them in the UMMA SW128
// K-major layout (16-B chunk c of tile row i at chunk position c ^ (i & 7)) for a 1024-B
// aligned tile, also when dst = tile + 512 (rows 4..7 of an 8-row atom). Also times a
// gather4 stream.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2602_07616_b200/csrc/ptx.cuh"
using namespace sere;

__global__ void gather(const __grid_constant__ CUtensorMap tm, const int* rows, int n, int kt, uint16_t* out) {
  __shared__ __align__(1024) uint8_t tile[256 * 128];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar, n * 128);
    for (int i = 0; i < n; i += 4) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(tile + i * 128)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(kt * 64), "r"(rows[i]), "r"(rows[i + 1]), "r"(rows[i + 2]),
          "r"(rows[i + 3]), "r"(smem_u32(&bar))
          : "memory");
    }
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(tile)[i];
}

int main() {
  const int T = 512, D = 2048, n = 256;
  uint16_t* hx = (uint16_t*)malloc(T * D * 2);
  for (int r = 0; r < T; ++r)
    for (int c = 0; c < D; ++c) hx[r * D + c] = (uint16_t)((r * 131 + c) & 0xffff);
  uint16_t* x; cudaMalloc(&x, T * D * 2); cudaMemcpy(x, hx, T * D * 2, cudaMemcpyHostToDevice);
  int hrows[n];
  for (int i = 0; i < n; ++i) hrows[i] = (i * 37 + 11) % T;
  hrows[5] = hrows[6];  // duplicates allowed
  int* rows; cudaMalloc(&rows, sizeof(hrows)); cudaMemcpy(rows, hrows, sizeof(hrows), cudaMemcpyHostToDevice);
  uint16_t* out; cudaMalloc(&out, n * 64 * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)T};
  cuuint64_t gstr[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  int bad = 0;
  for (int kt : {0, 3}) {
    gather<<<1, 256>>>(tm, rows, n, kt, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kt=%d launch: %s\n", kt, cudaGetErrorString(e));
    uint16_t* ho = (uint16_t*)malloc(n * 128);
    cudaMemcpy(ho, out, n * 128, cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; ++i)
      for (int p = 0; p < 8; ++p) {  // chunk position p of tile row i holds logical chunk p ^ (i & 7)
        const int c = p ^ (i & 7);
        for (int w = 0; w < 8; ++w) {
          const uint16_t want = hx[hrows[i] * D + kt * 64 + c * 8 + w];
          const uint16_t got = ho[i * 64 + p * 8 + w];
          if (want != got && bad++ < 5) printf("mismatch row %d pos %d w %d: got %u want %u\n", i, p, w, got, want);
        }
      }
    free(ho);
  }
  printf("gather4 SW128 layout check: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
