// Diagnostic (not part of the product): HBM ceiling of the fused round trip's
// traffic pattern -- read x once, write two arrays of the same size (1:2) --
// and of a plain 1:1 copy, with 16-byte vector loads / streaming stores.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
//        -o tools/diag/libcopy12.so tools/diag/copy12.cu
#include <cuda_runtime.h>
#include <cstdint>

__global__ void copy12(const float4* __restrict__ x, float4* __restrict__ y,
                       float4* __restrict__ z, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x + i);
    __stcs(y + i, v);
    __stcs(z + i, v);
  }
}
__global__ void copy11(const float4* __restrict__ x, float4* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    __stcs(y + i, __ldcs(x + i));
}

extern "C" int diag_copy(const void* x, void* y, void* z, int64_t nfloat4, int blocks,
                         void* stream) {
  if (z)
    copy12<<<blocks, 512, 0, (cudaStream_t)stream>>>((const float4*)x, (float4*)y, (float4*)z,
                                                     nfloat4);
  else
    copy11<<<blocks, 512, 0, (cudaStream_t)stream>>>((const float4*)x, (float4*)y, nfloat4);
  return (int)cudaGetLastError();
}
