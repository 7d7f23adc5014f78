// Host side of the TMA-fed GEMM engine (tma_gemm.cuh): CUtensorMap encoding for row-major
// fp32 matrices.  The driver entry point is resolved through the runtime
// (cudaGetDriverEntryPoint), so the library does not link libcuda directly.
//
// A matrix is described by a 3-D view {W columns, rows, column blocks of W} (strides: row
// pitch, 4W bytes) and one of two box shapes:
//   K-major  (W = 16, SWIZZLE_64B):            box {16, R, 1}   -> R rows x one 64-byte K slice
//   MN-major (W = 32, SWIZZLE_128B_ATOM_32B):  box {32, 16, NB} -> 16 K rows x NB 32-column blocks
//            (the only shared-memory layout tcgen05 accepts for MN-major TF32: 128-byte rows
//            swizzled in 32-byte atoms; blocks 2 KB apart = LBO, 4-row K groups 512 B = SBO)
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace nb {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error("nnmd_b200: cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// rows x cols fp32 matrix with row pitch `pitch` floats (pitch % 4 == 0, base 16-byte
// aligned).  mn = 0: K-major box {16, box_rows, 1} (cols % 16 == 0); mn = 1: MN-major box
// {32, 16, box_rows / 32} (box_rows = MN extent, cols % 32 == 0).  Rows past `rows` read as
// zero.
inline void make_tmap(CUtensorMap* out, const float* base, long rows, long cols, long pitch, int mn, int box_rows) {
  const int W = mn ? 32 : 16;
  if (pitch % 4 || cols % W || (reinterpret_cast<uintptr_t>(base) & 15) || box_rows % W || box_rows > 256 ||
      rows < 1)
    throw std::runtime_error("nnmd_b200: bad tensor-map geometry");
  const cuuint64_t dim[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / W)};
  const cuuint64_t stride[2] = {static_cast<cuuint64_t>(pitch) * 4, static_cast<cuuint64_t>(4 * W)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(W), mn ? 16u : static_cast<cuuint32_t>(box_rows),
                             mn ? static_cast<cuuint32_t>(box_rows / W) : 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  static const int promo = getenv("NNMD_TMA_PROMO") ? atoi(getenv("NNMD_TMA_PROMO")) : 1;
  const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                  : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                               : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  const CUresult r = encode_tiled_fn()(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dim, stride,
                                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                                       pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("nnmd_b200: cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

}  // namespace nb
