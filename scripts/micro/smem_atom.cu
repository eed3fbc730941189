// Microbenchmark: shared-memory scatter-add throughput on sm_100a, 15 warps x 1 CTA per SM:
// (0) float2 read-modify-write (LDS.64 + STS.64, warp-private accumulators),
// (1) 2 x red.shared.add.u32 into one shared accumulator, (2) 2 x red.shared.add.u64, (3) float atomicAdd (CAS loop)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(480, 1) k(const int* __restrict__ idx, int n_iter, int span, float* out)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = 0;
    __syncthreads();
    uint32_t h = 2654435761u * (blockIdx.x * 480 + tid + 1);
    int pos = (lane * 97) % span;
    float2 v = make_float2(1.f, 2.f);
    for (int it = 0; it < n_iter; ++it) {
        h = h * 1664525u + 1013904223u;
        pos += 1 + ((h >> 28) & 1);
        if (pos >= span) pos -= span;
        if (MODE == 0) {
            float2* a = reinterpret_cast<float2*>(sm) + warp * (span + 64) / 15 * 0 + pos + warp * 0;
            float2* acc = reinterpret_cast<float2*>(sm) + (warp % 15) * ((200 * 1024 / 8) / 15);
            float2* p = acc + (pos % ((200 * 1024 / 8) / 15 - 2));
            float2 t = *p; *p = make_float2(t.x + v.x, t.y + v.y);
            (void)a;
        } else if (MODE == 1) {
            uint32_t* p = reinterpret_cast<uint32_t*>(sm) + 2 * pos;
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(h & 1023));
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p + 1)), "r"(h & 511));
        } else if (MODE == 2) {
            unsigned long long* p = reinterpret_cast<unsigned long long*>(sm) + 2 * (pos % (200 * 1024 / 16 - 1));
            asm volatile("red.shared.add.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "l"((unsigned long long)(h & 1023)));
            asm volatile("red.shared.add.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p + 1)), "l"((unsigned long long)(h & 511)));
        } else {
            float* p = reinterpret_cast<float*>(sm) + 2 * pos;
            atomicAdd(p, v.x);
            atomicAdd(p + 1, v.y);
        }
    }
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = reinterpret_cast<float*>(sm)[5];
}
int main()
{
    float* out; cudaMalloc(&out, 4096);
    const int span = 136 * 100;   // float2 elements of a tall band
    const int n_iter = 20000;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[4] = {"float2 RMW (LDS.64+STS.64), warp-private", "2x red.shared.add.u32, shared", "2x red.shared.add.u64, shared", "2x atomicAdd(float) CAS, shared"};
    for (int m = 0; m < 4; ++m) {
        auto f = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            f<<<148, 480, 200 * 1024>>>(nullptr, n_iter, span, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%-45s %.3f ms  %.2f G pixel-updates/s  err=%s\n", names[m], ms, 148.0 * 480 * n_iter / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
