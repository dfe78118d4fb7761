#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
    void *f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    float *d; cudaMalloc(&d, 1 << 28);
    CUtensorMap tm; cuuint32_t es[5] = {1,1,1,1,1};
    { cuuint64_t dims[3] = {32, 25088, 48}; cuuint64_t str[2] = {1536 * 4, 128}; cuuint32_t box[3] = {32, 32, 4};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("dy 3d: %d\n", r); }
    { cuuint64_t dims[4] = {32, 32, 1, 4704}; cuuint64_t str[3] = {128, 128, 4096}; cuuint32_t box[4] = {32, 32, 1, 2};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("val 4d: %d\n", r); }
    { cuuint64_t dims[3] = {32, 32, 4704}; cuuint64_t str[2] = {128, 4096}; cuuint32_t box[3] = {32, 32, 2};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("val 3d: %d\n", r); }
    { cuuint64_t dims[3] = {32, 48, 25088}; cuuint64_t str[2] = {128, 1536*4}; cuuint32_t box[3] = {32, 4, 32};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("dy 3d increasing: %d\n", r); }
    return 0;
}
