#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  const int N = 16;
  float s[N]; int q[N];
  for (int i = 0; i < N; ++i) { s[i] = threadIdx.x * 1e-3f + i * 1.37f; q[i] = threadIdx.x + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (MODE == 0) { float f; asm volatile("cvt.rmi.f32.f32 %0, %1;" : "=f"(f) : "f"(s[i])); s[i] = f + 0.75f; }     // FRND + FADD
      if (MODE == 1) { s[i] = s[i] + 0.75f; }                                                                          // FADD only (baseline)
      if (MODE == 2) { asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(q[i]) : "r"(q[(i+1)%N])); }                     // IMAD
      if (MODE == 3) { asm volatile("add.u32 %0, %0, %1;" : "+r"(q[i]) : "r"(q[(i+1)%N])); }                          // IADD
      if (MODE == 4) { asm volatile("shl.b32 %0, %0, 2;\n\tadd.u32 %0, %0, %1;" : "+r"(q[i]) : "r"(q[(i+3)%N])); }     // LEA?
      if (MODE == 5) { int v; asm volatile("cvt.rmi.s32.f32 %0, %1;" : "=r"(v) : "f"(s[i])); s[i] = __int_as_float(v) + 1.0f; } // F2I + FADD
    }
  }
  float r = 0; for (int i = 0; i < N; ++i) r += s[i] + q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float* out; cudaMalloc(&out, 148*8*256*4*8);
  const char* names[] = {"FRND+FADD", "FADD", "IMAD", "IADD", "SHL+IADD", "F2I+FADD"};
  int iters = 4096;
  for (int m = 0; m < 6; ++m) {
    int blocks = 148 * 8, threads = 256;
    void (*fn)(float*, int) = m==0?k<0>:m==1?k<1>:m==2?k<2>:m==3?k<3>:m==4?k<4>:k<5>;
    fn<<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); fn<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double items = (double)blocks * threads * iters * 16;
    printf("%-10s items/clk/SM = %.1f  (ms %.3f)\n", names[m], items / (ms * 1e-3 * clk * 1e3) / 148, ms);
  }
  return 0;
}
