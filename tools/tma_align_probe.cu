#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int c0, int c1, int c2, int variant, int bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t b = base;            // barrier at offset 0
  uint32_t d = base + 1024;     // data 1024-aligned
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(1));
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(bytes) : "memory");
  __syncthreads();
  if (variant == 10) {
    if (threadIdx.x < 32) {
      uint32_t pred;
      asm volatile("{\n.reg .pred p;\n.reg .b32 r;\nelect.sync r|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
      if (pred)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" :: "r"(d), "l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(b) : "memory");
    }
  } else {
    if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" :: "r"(d), "l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(b) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra.uni W;\n}\n" :: "r"(b), "r"(0) : "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < bytes/4; i += blockDim.x) out[i] = ((float*)(sm + 1024))[i];
}
int main(int argc, char** argv) {
  int variant = atoi(argv[1]);
  int bw = atoi(argv[2]);
  int isx=312, isy=240, slots=24, pitch=312;
  float* ring; cudaMalloc(&ring, (size_t)slots*isy*pitch*4);
  float* h = new float[(size_t)slots*isy*pitch]; for (size_t i=0;i<(size_t)slots*isy*pitch;i++) h[i]=(float)i;
  cudaMemcpy(ring, h, (size_t)slots*isy*pitch*4, cudaMemcpyHostToDevice);
  CUtensorMap tm; memset(&tm, 0, sizeof tm);
  cuuint64_t dims[3]={(cuuint64_t)isx,(cuuint64_t)isy,(cuuint64_t)slots};
  cuuint64_t str[2]={(cuuint64_t)pitch*4,(cuuint64_t)pitch*4*isy};
  cuuint32_t box[3]={(cuuint32_t)bw,8,1}, es[3]={1,1,1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ring, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float* out; cudaMalloc(&out, 65536);
  int bytes = bw*8*4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1,128,bytes+2048>>>(tm, out, 5, 3, 2, variant, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  float o[8]; cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
  printf("encode %d variant %d bw %d: %s  o[0]=%f expect %f\n", (int)r, variant, bw, cudaGetErrorString(e), o[0], h[(size_t)2*isy*pitch+3*pitch+5]);
  return e ? 1 : 0;
}
