#include <cstdio>
#include <cuda_runtime.h>
struct f2 { float x, y; };
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm volatile("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}" : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y)); return d; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 d; asm volatile("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;}" : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)); return d; }
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  const int N = 8;
  f2 a[N]; float s[2*N];
  for (int i = 0; i < N; ++i) { a[i] = f2{threadIdx.x * 1e-3f + i, i * 0.5f}; s[2*i] = a[i].x; s[2*i+1] = a[i].y; }
  f2 b{1.0001f, 0.9999f}, c{1e-7f, -1e-7f};
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (MODE == 0) a[i] = fma2(a[i], b, c);
      if (MODE == 1) a[i] = add2(a[i], b);
      if (MODE == 2) { s[2*i] = fmaf(s[2*i], b.x, c.x); s[2*i+1] = fmaf(s[2*i+1], b.y, c.y); }
      if (MODE == 3) { s[2*i] = s[2*i] + b.x; s[2*i+1] = s[2*i+1] + b.y; }
      if (MODE == 4) { s[2*i] = __fdividef(1.0f, s[2*i]) ; s[2*i+1] = __fdividef(1.0f, s[2*i+1]); }
      if (MODE == 5) { int idx = ((int)s[2*i] + threadIdx.x) & 4095; s[2*i] += sm[idx]; s[2*i+1] += sm[(idx + 32) & 4095]; }
    }
  }
  long long t1 = clock64();
  float r = 0; for (int i = 0; i < N; ++i) r += a[i].x + a[i].y + s[2*i] + s[2*i+1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148*8*256*4*8); cudaMalloc(&cyc, 148*8*8*8);
  const char* names[] = {"FFMA2", "FADD2", "FFMA(scalar)", "FADD(scalar)", "MUFU.RCP", "LDS+FADD"};
  int iters = 4096;
  for (int m = 0; m < 6; ++m) for (int bps : {4, 8}) {
    int blocks = 148 * bps, threads = 256;
    void (*fn)(float*, int, long long*) = m==0?k<0>:m==1?k<1>:m==2?k<2>:m==3?k<3>:m==4?k<4>:k<5>;
    fn<<<blocks, threads>>>(out, 16, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); fn<<<blocks, threads>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148*8]; cudaMemcpy(h, cyc, blocks*8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
    // lane-ops: FP modes do 2*N per iteration per thread (pairs count as 2 lanes)
    double lane_ops = (double)blocks * threads * iters * 2 * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc_total = ms * 1e-3 * clk * 1e3;
    printf("%-14s blocks/SM=%d  lane-ops/clk/SM (event@%.0fMHz) = %.1f   (per-block clock64: %.1f)   ms=%.3f\n", names[m], bps, clk/1e3,
           lane_ops / cyc_total / 148, (double)bps * threads * iters * 16 / avg, ms);
  }
  return 0;
}
