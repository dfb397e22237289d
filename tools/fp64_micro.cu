// fp64 FMA throughput of the B200 (the ridge point of the fluid passes' roofline,
// "the fp64 peak is not in MP, so measure an fp64 FMA microbenchmark").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_micro tools/fp64_micro.cu
//   tools/fp64_micro            -> one JSON line: {"fp64_fma_tflops": ..., ...}
// Each thread runs ACC independent FMA chains for ITERS iterations (2 flops per FMA);
// the grid is a multiple of the SM count; best of 5 timed launches (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ACC = 16;

__global__ void k_fma(double* out, int iters, double a, double b)
{
    double x[ACC];
#pragma unroll
    for (int j = 0; j < ACC; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ACC; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < ACC; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;   // keep the chains live
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double));
    const int iters = 4096, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * ACC * (double)iters * threads * blocks;
    const cudaError_t err = cudaGetLastError();
    printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"blocks\": %d, \"threads\": %d, \"acc\": %d, "
           "\"iters\": %d, \"err\": \"%s\"}\n",
           flops / (best * 1e-3) / 1e12, best, sms, blocks, threads, ACC, iters, cudaGetErrorString(err));
    (void)clk;
    return err == cudaSuccess ? 0 : 1;
}
