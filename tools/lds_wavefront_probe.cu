// Shared-load wavefront probe: how many LSU wavefronts does one warp-wide LDS.{32,64,128}
// take for a given lane -> address pattern?  Run under
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum
// and divide wavefronts by instructions (each kernel = one pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_probe tools/lds_wavefront_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// addr(lane) in bytes, computed once; ITER loads
template <int W>
__global__ void probe(int pat, float* out) {
    __shared__ __align__(16) float sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i;
    __syncthreads();
    const int l = threadIdx.x & 31;
    int a = 0;  // in bytes
    switch (pat) {
        case 0: a = 0; break;                                   // all lanes same address
        case 1: a = ((l >> 2) & 3) * W; break;                   // 4 distinct contiguous (like line consts)
        case 2: a = (l & 7) * W; break;                          // 8 distinct contiguous, repeated per 8 lanes
        case 3: a = (l & 15) * W; break;                         // 16 distinct contiguous, repeated per half
        case 4: a = l * W; break;                                // 32 distinct contiguous
        case 5: a = (l >> 3) * W; break;                         // 4 distinct, lane groups of 8
        case 6: a = (l >> 4) * W; break;                         // 2 distinct (per half)
        case 7: a = (l & 1) * 128 * 4 + (l >> 1) * W; break;     // alternating halves of two 512B regions
        case 8: a = ((l & 7) * W) + ((l >> 3) & 1) * 4096; break; // lanes 8-15 same banks as 0-7, other row
        case 9: a = (l & 7) * W + (l >> 3) * 4096; break;        // 4 groups of 8 distinct, all same banks
        case 10: a = ((l * 5) & 31) * W; break;                  // 32 distinct permuted
        case 11: a = (l & 3) * W + ((l >> 2) & 3) * 2 * 128 + (l >> 4) * 4 * W; break;
        default: a = 0;
    }
    const unsigned base = su32(sm) + a;
    float acc = 0.f;
#pragma unroll 1
    for (int it = 0; it < 1024; ++it) {
        if (W == 4) {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(base));
            acc += v;
        } else if (W == 8) {
            float v0, v1;
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(base));
            acc += v0 + v1;
        } else {
            float v0, v1, v2, v3;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(base));
            acc += v0 + v1 + v2 + v3;
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    for (int w : {4, 8, 16})
        for (int p = 0; p < 12; ++p) {
            if (w == 4) probe<4><<<1, 32>>>(p, d);
            if (w == 8) probe<8><<<1, 32>>>(p, d);
            if (w == 16) probe<16><<<1, 32>>>(p, d);
            cudaDeviceSynchronize();
            printf("W=%d pat=%d\n", w, p);
        }
    return 0;
}
