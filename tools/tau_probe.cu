// tau_probe.cu -- issue rate of the packed tau (tau4 / tau4c) alone: NCH independent chains per
// thread, 32 warps per SM.  Reports tau evaluations per SM cycle and warp-instructions per SMSP cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1903_10107_b200/csrc -o tau_probe tools/tau_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "swar.cuh"
using namespace qkd;

template <int NCH, bool C>
__global__ void k(uint32_t* out, Konst K0, long long* cyc, int iters) {
    const Konst K = K0.in_regs();
    uint32_t a[NCH], m[NCH];
    for (int i = 0; i < NCH; ++i) { a[i] = (threadIdx.x * 37 + i * 11) & 0x3F3F3F3Fu; m[i] = (threadIdx.x * 13 + i * 7) & 0x3F3F3F3Fu; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            a[i] = C ? tau4c(a[i], m[i], K) : tau4(a[i], m[i], K);
            m[i] = (m[i] + 0x01010101u * (i + 1)) & 0x3F3F3F3Fu;   // keep inputs changing
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < NCH; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NCH, bool C>
void run(const char* name, int threads) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, 4 * sms * 1024); cudaMalloc(&cyc, 8 * sms);
    Konst K{1u, 2u, 0xFFFFFFFFu, 0xFFFFFFFEu, 0xFFFFFF00u, 0xFF80FF80u, 0x3F3F3F3Fu, 0x7F7F7F7Fu};
    const int iters = 2048;
    k<NCH, C><<<sms, threads>>>(out, K, cyc, iters);
    k<NCH, C><<<sms, threads>>>(out, K, cyc, iters);
    cudaDeviceSynchronize();
    long long h[1024]; cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double taus = (double)threads * iters * NCH;
    const double per_sm_cycle = taus / mx;                 // thread-level tau evaluations per SM cycle
    const int ipt = (C ? 14 : 16) + 2;                      // SASS per tau + the 2-op input update
    printf("%-6s chains=%d threads=%4d  tau(x4 frames)/SM-cycle = %6.2f   est. warp-IPC/SMSP = %.2f\n",
           name, NCH, threads, per_sm_cycle, per_sm_cycle / 32.0 * ipt / 4.0);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run<1, false>("tau4", 1024); run<2, false>("tau4", 1024); run<4, false>("tau4", 1024);
    run<1, true>("tau4c", 1024); run<2, true>("tau4c", 1024); run<4, true>("tau4c", 1024);
    run<2, true>("tau4c", 512); run<4, true>("tau4c", 512); run<2, true>("tau4c", 256); run<4, true>("tau4c", 128);
    return 0;
}
