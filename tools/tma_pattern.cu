// tma_pattern.cu -- memory-system rate of the sweeps' TMA access patterns
// without the physics (tools only): every warp streams work items (32 strips
// x 128 cells) through a two-buffer smem ring -- TMA load, TMA store to a
// second buffer -- like the sweeps' rings, over a 16384^2 state of 4 fp64
// variables in the library's row-interleaved layout.
//   x: column-sweep boxes {32 cols, 4 vars, 4 rows} (256-byte rows)
//   y: row-sweep boxes {8 cols, 1 var, 32 rows} x 4 (64-byte rows)
//   yt: the row sweep's chunk as one contiguous 8 KB block (a layout tiled
//       in 32-row x 8-column blocks; what such a layout would give)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tma_pattern tools/tma_pattern.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>

constexpr int N = 16384;
constexpr int PITCH = 16400;  // doubles per variable row
constexpr int ROWS = N + 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
extern __shared__ __align__(1024) unsigned char smem[];

__device__ __forceinline__ void mbar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned par) {
  unsigned done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(par) : "memory");
  } while (!done);
}
__device__ __forceinline__ void load3(void* d, const CUtensorMap* m, unsigned long long* b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(smem_u32(d)), "l"(m), "r"(smem_u32(b)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void store3(const CUtensorMap* m, const void* s, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(m), "r"(smem_u32(s)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void load5(void* d, const CUtensorMap* m, unsigned long long* b, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               ::"r"(smem_u32(d)), "l"(m), "r"(smem_u32(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4) : "memory");
}
__device__ __forceinline__ void store5(const CUtensorMap* m, const void* s, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];"
               ::"l"(m), "r"(smem_u32(s)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4) : "memory");
}
__device__ __forceinline__ void load_bulk(void* d, const void* g, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(d)), "l"(g), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void store_bulk(void* g, const void* s, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes) : "memory");
}

struct Args {
  int mode;  // 0 x, 1 y, 2 yt, 3 x on the tiled layout, 4 y tiled reads + row writes, 5 x row reads + tiled writes
  double* src;
  double* dst;
  unsigned* counter;
};

// items: 512 strip groups x 128 segments of 128 cells; 2 x 8 KB ring per warp
__global__ void __launch_bounds__(128) stream_kernel(Args a, const __grid_constant__ CUtensorMap ld,
                                                     const __grid_constant__ CUtensorMap st) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = smem + warp * 16384;
  unsigned long long* bar = (unsigned long long*)(smem + 4 * 16384) + warp * 2;
  if (lane == 0) { mbar_init(bar); mbar_init(bar + 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  unsigned ph[2] = {0, 0};
  const int groups = N / 32, segs = N / 128;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(a.counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= groups * segs) break;
    // x: segment-major over column groups; y: bands of 2 row groups
    int grp, sg;
    if (a.mode == 0 || a.mode == 3 || a.mode == 5) { grp = item % groups; sg = item / groups; }
    else { const int band = item / (2 * segs), r = item % (2 * segs); sg = r / 2; grp = band * 2 + r % 2; }
    if (lane == 0) {
      const int nchunk = (a.mode == 0 || a.mode == 3 || a.mode == 5) ? 32 : 16;  // 4-row or 8-col chunks of 8 or 4 KB... (8 KB for y)
      for (int q = 0; q < nchunk; ++q) {
        const int b = q & 1;
        unsigned char* buf = ring + b * 8192;
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer b's store (2 chunks ago) read out
        if (a.mode == 0 || a.mode == 5) {
          mbar_expect(bar + b, 4096);
          load3(buf, &ld, bar + b, grp * 32 + 8, 0, sg * 128 + q * 4);
        } else if (a.mode == 3) {  // {8 rj, 4 tj, 4 ri, 4 v, 1 ti}
          mbar_expect(bar + b, 4096);
          const int row = sg * 128 + q * 4;
          load5(buf, &ld, bar + b, 0, grp * 4, row & 31, 0, row >> 5);
        } else if (a.mode == 1) {
          mbar_expect(bar + b, 8192);
          for (int v = 0; v < 4; ++v) load3(buf + v * 2048, &ld, bar + b, sg * 128 + q * 8 + 8, v, grp * 32 + 2);
        } else {  // 2, 4: the 8 KB tile
          mbar_expect(bar + b, 8192);
          const size_t tile = ((size_t)grp * (N / 8) + (sg * 16 + q)) * 1024;  // 8 KB blocks
          load_bulk(buf, a.src + tile, 8192, bar + b);
        }
        mbar_wait(bar + b, ph[b]);
        ph[b] ^= 1;
        if (a.mode == 0) store3(&st, buf, grp * 32 + 8, 0, sg * 128 + q * 4);
        else if (a.mode == 5) {
          const int row = sg * 128 + q * 4;
          store5(&st, buf, 0, grp * 4, row & 31, 0, row >> 5);
        } else if (a.mode == 4) {
          for (int v = 0; v < 4; ++v) store3(&st, buf + v * 2048, sg * 128 + q * 8 + 8, v, grp * 32 + 2);
        } else if (a.mode == 3) {
          const int row = sg * 128 + q * 4;
          store5(&st, buf, 0, grp * 4, row & 31, 0, row >> 5);
        }
        else if (a.mode == 1)
          for (int v = 0; v < 4; ++v) store3(&st, buf + v * 2048, sg * 128 + q * 8 + 8, v, grp * 32 + 2);
        else store_bulk(a.dst + ((size_t)grp * (N / 8) + (sg * 16 + q)) * 1024, buf, 8192);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncwarp();
  }
}

int main() {
  double *A, *B;
  const size_t bytes = (size_t)ROWS * 4 * PITCH * 8;
  cudaMalloc(&A, bytes);
  cudaMalloc(&B, bytes);
  cudaMemset(A, 0, bytes);
  unsigned* counter;
  cudaMalloc(&counter, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap mx_l, mx_s, my_l, my_s;
  const cuuint64_t dims[3] = {PITCH, 4, ROWS};
  const cuuint64_t str[2] = {PITCH * 8, 4 * PITCH * 8};
  const cuuint32_t bx[3] = {32, 4, 4}, by[3] = {8, 1, 32}, e[3] = {1, 1, 1};
  enc(&mx_l, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, bx, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mx_s, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, B, dims, str, bx, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&my_l, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, by, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&my_s, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, B, dims, str, by, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // the 32-row x 8-column tiled layout seen by the column sweep: dims
  // {rj 8, tj, ri 32, v 4, ti} (strides not increasing)
  CUtensorMap mt_l, mt_s;
  const cuuint64_t d5[5] = {8, (cuuint64_t)N / 8, 32, 4, (cuuint64_t)N / 32};
  const cuuint64_t s5[4] = {8192, 64, 2048, 8192ull * (N / 8)};
  const cuuint32_t b5[5] = {8, 4, 4, 4, 1}, e5[5] = {1, 1, 1, 1, 1};
  CUresult r1 = enc(&mt_l, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, A, d5, s5, b5, e5, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mt_s, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, B, d5, s5, b5, e5, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("{\"encode_tiled_x\": [%d, %d]}\n", (int)r1, (int)r2);
  const int smem_bytes = 4 * 16384 + 64;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[6] = {"x (256-byte box rows)", "y (64-byte box rows)", "y tiled (8 KB blocks)",
                          "x on the tiled layout (16 x 256 B)", "y: tiled reads, row-layout writes",
                          "x: row-layout reads, tiled writes"};
  for (int ctas_per_sm = 2; ctas_per_sm <= 3; ++ctas_per_sm)
    for (int mode = 0; mode < 6; ++mode) {
      if (mode == 3 && (r1 || r2)) continue;
      Args a{mode, A, B, counter};
      const CUtensorMap& l = (mode == 0 || mode == 5) ? mx_l : mode == 3 ? mt_l : my_l;
      const CUtensorMap& s = mode == 0 ? mx_s : (mode == 3 || mode == 5) ? mt_s : my_s;
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaMemset(counter, 0, 4);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        stream_kernel<<<sms * ctas_per_sm, 128, smem_bytes>>>(a, l, s);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
      }
      const double moved = 2.0 * (double)N * N * 32;  // read + write of 4 fp64 per cell
      std::printf("{\"pattern\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
                  names[mode], ctas_per_sm, best, moved / (best * 1e-3) / 1e9,
                  cudaGetErrorString(cudaGetLastError()));
    }

  return 0;
}
