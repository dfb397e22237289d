// Microbenchmarks that set the roofline of the IB kernels (not part of the product):
// the kernels of Steps 1a and 2b are bound by L2 gathers and fp64 reductions into an
// L2-resident band of cells, not by HBM.  This measures, on the target GPU,
//   red_scatter : fp64 atomicAdd (RED.ADD.F64) at random 8-byte addresses
//   red_quad    : the spread's pattern -- groups of 4 lanes reduce into 4 consecutive
//                 doubles of a random row (quad-lane spreading, ib.cu)
//   gather      : random 8-byte loads (the interpolation's gathers)
//   gather_quad : groups of 4 lanes load 4 consecutive doubles of a random row
// in a region of `mb` MiB (default 64: L2-resident on B200's 126 MB L2), and prints one
// JSON line per pattern with operations/s and L2 payload bytes/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ib_micro tools/ib_micro.cu && ./ib_micro [mb]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <bool QUAD>
__global__ void k_red(double* __restrict__ buf, unsigned mask, int iters)
{
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        unsigned a;
        if (QUAD) a = ((hash32((t >> 2) * 977u + (unsigned)i) << 2) + (t & 3)) & mask;
        else a = hash32(t * 131u + (unsigned)i * 7919u) & mask;
        atomicAdd(buf + a, 1.0);
    }
}

template <bool QUAD>
__global__ void k_gather(const double* __restrict__ buf, unsigned mask, int iters, double* __restrict__ out)
{
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        unsigned a;
        if (QUAD) a = ((hash32((t >> 2) * 977u + (unsigned)i) << 2) + (t & 3)) & mask;
        else a = hash32(t * 131u + (unsigned)i * 7919u) & mask;
        acc += __ldcg(buf + a);
    }
    if (acc == 12345.678) out[t] = acc;
}

int main(int argc, char** argv)
{
    const int mb = argc > 1 ? atoi(argv[1]) : 64;
    size_t n = 1;
    while (n * 2 * sizeof(double) <= (size_t)mb << 20) n *= 2;
    double *buf, *out;
    cudaMalloc(&buf, n * sizeof(double));
    cudaMalloc(&out, 1 << 24);
    cudaMemset(buf, 0, n * sizeof(double));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 256;
    const double ops = (double)blocks * threads * iters;
    const unsigned mask = (unsigned)(n - 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"red_scatter", "red_quad", "gather", "gather_quad"};
    for (int which = 0; which < 4; ++which) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (which == 0) k_red<false><<<blocks, threads>>>(buf, mask, iters);
            if (which == 1) k_red<true><<<blocks, threads>>>(buf, mask, iters);
            if (which == 2) k_gather<false><<<blocks, threads>>>(buf, mask, iters, out);
            if (which == 3) k_gather<true><<<blocks, threads>>>(buf, mask, iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        const cudaError_t err = cudaGetLastError();
        printf("{\"pattern\": \"%s\", \"region_mib\": %d, \"ops\": %.0f, \"ms\": %.4f, \"ops_per_s\": %.4e, "
               "\"payload_gbs\": %.1f, \"status\": \"%s\"}\n",
               names[which], mb, ops, best, ops / (best * 1e-3), ops * 8.0 / (best * 1e-3) / 1e9,
               cudaGetErrorString(err));
    }
    return 0;
}
