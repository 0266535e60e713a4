// pipe_probe3.cu -- issue rate of IMAD.HI (a*b >> 32 + c) alone and beside ALU-pipe ops on sm_100a:
// can the tau's SHF (>> 1) and LEA.HI (g + (y >> 6)) move to the FMA pipe at full IMAD rate?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe3 tools/pipe_probe3.cu && ./pipe_probe3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048
#define OP_IMADHI(r, c, k) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r) : "r"(k), "r"(c))
#define OP_IMAD(r, c, k) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r) : "r"(k), "r"(c))
#define OP_LOP3(r, c, k) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r) : "r"(c), "r"(k))
#define OP_SHF(r, c, k) asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(r) : "r"(c))
#define OP_IMADWIDE(r, c, k) asm volatile("{.reg .u64 t; mad.wide.u32 t, %0, %1, 5; cvt.u32.u64 %0, t;}" : "+r"(r) : "r"(k))

#define KERNEL1(NAME, OP)                                                   \
    __global__ void NAME(uint32_t* out, uint32_t k, long long* cyc) {       \
        uint32_t r[CH];                                                     \
        for (int i = 0; i < CH; ++i) r[i] = threadIdx.x * 7 + i;            \
        __syncthreads();                                                    \
        long long t0 = clock64();                                           \
        for (int it = 0; it < ITERS; ++it) {                                \
            _Pragma("unroll") for (int i = 0; i < CH; ++i) { OP(r[i], r[(i + 1) & 7], k); } \
        }                                                                   \
        __syncthreads();                                                    \
        long long t1 = clock64();                                           \
        uint32_t s = 0;                                                     \
        for (int i = 0; i < CH; ++i) s ^= r[i];                             \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                     \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                    \
    }
#define KERNEL2(NAME, OPA, OPB)                                                                 \
    __global__ void NAME(uint32_t* out, uint32_t k, long long* cyc) {                           \
        uint32_t r[CH];                                                                         \
        for (int i = 0; i < CH; ++i) r[i] = threadIdx.x * 7 + i;                                \
        __syncthreads();                                                                        \
        long long t0 = clock64();                                                               \
        for (int it = 0; it < ITERS; ++it) {                                                    \
            _Pragma("unroll") for (int i = 0; i < CH; i += 2) { OPA(r[i], r[(i + 3) & 7], k); OPB(r[i + 1], r[(i + 2) & 7], k); } \
        }                                                                                       \
        __syncthreads();                                                                        \
        long long t1 = clock64();                                                               \
        uint32_t s = 0;                                                                         \
        for (int i = 0; i < CH; ++i) s ^= r[i];                                                 \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                         \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                        \
    }
KERNEL1(k1, OP_IMADHI) KERNEL1(k2, OP_IMAD) KERNEL1(k3, OP_IMADWIDE)
KERNEL2(p1, OP_IMADHI, OP_LOP3) KERNEL2(p2, OP_IMADHI, OP_IMAD) KERNEL2(p3, OP_IMAD, OP_LOP3) KERNEL2(p4, OP_IMADHI, OP_SHF)
typedef void (*kfn)(uint32_t*, uint32_t, long long*);
int main() {
    struct { const char* name; kfn f; } ks[] = {{"IMAD.HI", k1}, {"IMAD", k2}, {"IMAD.WIDE", k3}, {"IMAD.HI+LOP3", p1},
                                                 {"IMAD.HI+IMAD", p2}, {"IMAD+LOP3", p3}, {"IMAD.HI+SHF", p4}};
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 1024;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * sms * threads);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    long long h[1024];
    printf("op, warp-inst per SM cycle (issue limit 4.0)\n");
    for (auto& k : ks) {
        k.f<<<sms, threads>>>(out, 0x01030507u, cyc);
        k.f<<<sms, threads>>>(out, 0x01030507u, cyc);
        if (cudaDeviceSynchronize() != cudaSuccess) return 1;
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-22s %.3f\n", k.name, (double)(threads / 32) * ITERS * CH / mx);
    }
    return 0;
}
