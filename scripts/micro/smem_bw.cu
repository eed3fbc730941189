// Microbenchmark: the shared-memory data path (LDS) peak of one B200 SM, the denominator of the
// projectors' roofline.  Every thread of 16 warps x 1 CTA per SM (and 32 x 1)
// streams conflict-free loads from a 64 KB shared array (LDS.128 / LDS.64 / LDS.32: lane l of a
// warp reads consecutive words, so each warp instruction is 4 / 2 / 1 wavefronts of 128 B with no
// bank conflict), unrolled 8 loads deep with independent XOR accumulators.  Reports bytes per clock
// per SM (SM cycles from clock64, per CTA) and the aggregate over the GPU from CUDA events.
// Build/run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_bw smem_bw.cu && ./smem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W>   // bytes per lane per load: 16, 8, 4
__global__ void lds_kernel(int n_iter, unsigned long long* cycles, uint32_t* sink)
{
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int kBytes = 64 * 1024;
    for (int i = threadIdx.x; i < kBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per warp a window of 8 consecutive 32-lane rows; each step moves the window by one row
    constexpr int row = 32 * W;                 // bytes of one warp-wide load
    constexpr int rows = kBytes / row;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int r = (warp * 8) % rows;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + lane * W;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < n_iter; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int rr = r + k;
            if (rr >= rows) rr -= rows;
            const uint32_t a = base + rr * row;
            if (W == 16) {
                uint32_t x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
                acc[k] ^= x ^ y ^ z ^ w;
            } else if (W == 8) {
                uint32_t x, y;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
                acc[k] ^= x ^ y;
            } else {
                uint32_t x;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
                acc[k] ^= x;
            }
        }
        r += 1;
        if (r >= rows) r -= rows;
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    uint32_t h = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) h ^= acc[k];
    if (h == 0x12345678u) sink[blockIdx.x] = h;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int W>
static void run(int sms, int warps, int n_iter)
{
    unsigned long long* d_cyc;
    uint32_t* d_sink;
    cudaMalloc(&d_cyc, sms * sizeof(unsigned long long));
    cudaMalloc(&d_sink, sms * sizeof(uint32_t));
    cudaFuncSetAttribute(lds_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    lds_kernel<W><<<sms, warps * 32, 64 * 1024>>>(n_iter / 10, d_cyc, d_sink);   // warm-up
    cudaEventRecord(a);
    lds_kernel<W><<<sms, warps * 32, 64 * 1024>>>(n_iter, d_cyc, d_sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long* cyc = new unsigned long long[sms];
    cudaMemcpy(cyc, d_cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double cmax = 0, csum = 0;
    for (int i = 0; i < sms; ++i) { csum += cyc[i]; cmax = cyc[i] > cmax ? cyc[i] : cmax; }
    const double bytes_cta = static_cast<double>(n_iter) * 8 * warps * 32 * W;
    const double b_per_clk = bytes_cta / (csum / sms);
    const double tbs = bytes_cta * sms / (ms * 1e-3) / 1e12;
    printf("{\"load\": \"LDS.%d\", \"warps_per_sm\": %d, \"bytes_per_clk_per_sm\": %.2f, \"aggregate_TBps\": %.2f, "
           "\"ms\": %.3f, \"implied_sm_mhz\": %.0f}\n",
           8 * W, warps, b_per_clk, tbs, ms, (cmax / (ms * 1e-3)) / 1e6);
    delete[] cyc;
    cudaFree(d_cyc);
    cudaFree(d_sink);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n_iter = 20000;
    for (int warps : {16, 32}) {
        run<16>(sms, warps, n_iter);
        run<8>(sms, warps, n_iter);
        run<4>(sms, warps, n_iter);
    }
    return 0;
}
