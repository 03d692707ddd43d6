// Shared-memory atomic throughput on B200 (sm_100a): one-off microbenchmark for the K4/K6 z-buffer
// design (ATOMS.CAS.64 min vs ATOMS.MIN.32 vs ATOMS.ADD.F32 vs plain LDS/STS).  Prints
// warp-instructions per SM-cycle for each variant.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256, IT = 2048;
__device__ __forceinline__ void cas_min64(unsigned long long *p, unsigned long long v)
{
    unsigned long long old = *p;
    while (v < old) {
        const unsigned long long r = atomicCAS(p, old, v);
        if (r == old) break;
        old = r;
    }
}
template <int MODE>
__global__ void __launch_bounds__(NT) k(unsigned long long *sink, int stride)
{
    __shared__ unsigned long long z[NT * 8];
    __shared__ float f[NT * 8];
    __shared__ unsigned u[NT * 8];
    for (int i = threadIdx.x; i < NT * 8; i += NT) { z[i] = ~0ull; f[i] = 0.f; u[i] = 0xffffffffu; }
    __syncthreads();
    unsigned long long v = 0xfffffff000000000ull - threadIdx.x;
    float acc = 0.f;
    unsigned a = (threadIdx.x * stride) & (NT * 8 - 1);
    for (int it = 0; it < IT; ++it) {
        const unsigned idx = (a + it * 33) & (NT * 8 - 1);
        if (MODE == 0) cas_min64(&z[idx], v - it);                 // always improves: one CAS each
        else if (MODE == 1) atomicMin(&u[idx], (unsigned)(0xfffff000u - it - threadIdx.x));
        else if (MODE == 2) atomicAdd(&f[idx], 1.0f);
        else if (MODE == 3) acc += f[idx];                          // plain LDS
        else if (MODE == 4) cas_min64(&z[idx], v + it);             // never improves: LDS + compare only
        else if (MODE == 5) { const unsigned long long o = z[idx]; if (v - it < o) z[idx] = v - it; }  // racy LDS/STS
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = z[0] + (unsigned long long)acc + u[1] + (unsigned long long)f[2];
}
template <int MODE>
void run(const char *name, int stride, int ctas, unsigned long long *d)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<ctas, NT>>>(d, stride);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<MODE><<<ctas, NT>>>(d, stride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double winst = 5.0 * ctas * (NT / 32) * (double)IT;     // warp-level ops
    const double cycles = ms * 1e-3 * clk * 1e3 * 148;            // SM-cycles (all SMs)
    printf("%-34s stride %2d: %.3f ms, %.3f warp-ops per SM-cycle, %.2f SM-cycles per warp-op\n", name, stride, ms,
           winst / cycles, cycles / winst);
}
int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 1 << 20);
    const int ctas = 148 * 8;
    for (int s : {1, 0}) {   // stride 1: 32 distinct banks-ish words; stride 0: all lanes one address
        run<0>("CAS64 min (improving)", s, ctas, d);
        run<4>("CAS64 min (not improving: LDS)", s, ctas, d);
        run<1>("atomicMin u32", s, ctas, d);
        run<2>("atomicAdd f32", s, ctas, d);
        run<3>("LDS f32", s, ctas, d);
        run<5>("LDS.64+STS.64 racy", s, ctas, d);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
