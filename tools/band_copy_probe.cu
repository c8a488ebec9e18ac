// H2D throughput of row-band copies (the band tail): rows [a, b) of 112
// views of 1248x960 float32 from a pinned stack, as 2-D copies of 32 views, as one 3-D
// copy, and as per-view copies; each alone and beside a concurrent 0.54 GB D2H.
// Build: nvcc -O2 -o tools/band_copy_probe tools/band_copy_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
int main() {
    const int isx = 1248, isy = 960, nv = 112;
    const size_t row = isx * 4, view = row * isy;
    char *h, *hv; void *d, *dv;
    cudaHostAlloc((void**)&h, view * nv, 0);
    cudaHostAlloc((void**)&hv, (size_t)512 << 20, 0);
    cudaMalloc(&d, view * nv);
    cudaMalloc(&dv, (size_t)512 << 20);
    cudaStream_t s, s2; cudaStreamCreate(&s); cudaStreamCreate(&s2);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int band : {50, 100, 200, 960}) {
        for (int mode = 0; mode < 3; ++mode)
            for (int d2h = 0; d2h < 2; ++d2h) {
                float best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    if (d2h) cudaMemcpyAsync(hv, dv, (size_t)512 << 20, cudaMemcpyDeviceToHost, s2);
                    cudaEventRecord(e0, s);
                    for (int a = 0; a < isy; a += band) {
                        const int b = a + band < isy ? a + band : isy;
                        if (mode == 0) {
                            for (int v = 0; v < nv; v += 32)
                                cudaMemcpy2DAsync((char*)d + v * view + a * row, view, h + v * view + a * row, view,
                                                  (b - a) * row, 32 < nv - v ? 32 : nv - v, cudaMemcpyHostToDevice, s);
                        } else if (mode == 1) {
                            cudaMemcpy3DParms p{};
                            p.srcPtr = make_cudaPitchedPtr(h, row, isx * 4, isy);
                            p.dstPtr = make_cudaPitchedPtr(d, row, isx * 4, isy);
                            p.srcPos = make_cudaPos(0, a, 0);
                            p.dstPos = make_cudaPos(0, a, 0);
                            p.extent = make_cudaExtent(row, b - a, nv);
                            p.kind = cudaMemcpyHostToDevice;
                            cudaMemcpy3DAsync(&p, s);
                        } else {
                            for (int v = 0; v < nv; ++v)
                                cudaMemcpyAsync((char*)d + v * view + a * row, h + v * view + a * row, (b - a) * row,
                                                cudaMemcpyHostToDevice, s);
                        }
                    }
                    cudaEventRecord(e1, s);
                    cudaDeviceSynchronize();
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                printf("band %3d rows  %-9s %-10s %6.2f ms  %5.1f GB/s\n", band, mode == 0 ? "2-D x32" : mode == 1 ? "3-D" : "per-view",
                       d2h ? "with D2H" : "alone", best, view * nv / best / 1e6);
            }
    }
    return 0;
}
