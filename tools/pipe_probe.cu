// pipe_probe.cu -- which sm_100a pipe does each packed-integer op issue on, and at what rate?
// Runs NW warps per SM, each with 8 independent dependency chains of one op (or of two ops
// interleaved), and reports warp-instructions per SM cycle.  Two ops on different pipes
// co-issue (sum of rates up to the 4 warp-inst/clk/SM issue limit); on one pipe they share it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe tools/pipe_probe.cu && ./pipe_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048

#define OP_IADD3(r, c) asm volatile("add.u32 %0, %0, %1;" : "+r"(r) : "r"(c))
#define OP_LOP3(r, c) asm volatile("xor.b32 %0, %0, %1;" : "+r"(r) : "r"(c))
#define OP_SHF(r, c) asm volatile("shr.b32 %0, %0, %1;" : "+r"(r) : "r"(c))
#define OP_PRMT(r, c) asm volatile("prmt.b32 %0, %0, %1, 0x6240;" : "+r"(r) : "r"(c))
#define OP_VABS(r, c) r = __vabsdiffu4(r, c)
#define OP_VADD2(r, c) r = __vadd2(r, c)
#define OP_VMIN2(r, c) r = __vmins2(r, c)
#define OP_VAMX(r, c) r = __viaddmax_s16x2(r, c, 0x00100010u)
#define OP_RELU(r, c) r = __viaddmin_s16x2_relu(r, c, 0x007E007Eu)
#define OP_IMAD(r, c) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(r) : "r"(c))
#define OP_LEAHI(r, c) asm volatile("{.reg .u32 t; shr.b32 t, %1, 7; add.u32 %0, %0, t;}" : "+r"(r) : "r"(c))

#define KERNEL1(NAME, OP)                                                   \
    __global__ void NAME(uint32_t* out, uint32_t c, long long* cyc) {       \
        uint32_t r[CH];                                                     \
        for (int i = 0; i < CH; ++i) r[i] = threadIdx.x * 7 + i;            \
        __syncthreads();                                                    \
        long long t0 = clock64();                                           \
        for (int it = 0; it < ITERS; ++it) {                                \
            _Pragma("unroll") for (int i = 0; i < CH; ++i) { OP(r[i], r[(i + 1) & 7]); } \
        }                                                                   \
        __syncthreads();                                                    \
        long long t1 = clock64();                                           \
        uint32_t s = 0;                                                     \
        for (int i = 0; i < CH; ++i) s ^= r[i];                             \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                     \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                    \
    }

#define KERNEL2(NAME, OPA, OPB)                                                                 \
    __global__ void NAME(uint32_t* out, uint32_t c, long long* cyc) {                           \
        uint32_t r[CH];                                                                         \
        for (int i = 0; i < CH; ++i) r[i] = threadIdx.x * 7 + i;                                \
        __syncthreads();                                                                        \
        long long t0 = clock64();                                                               \
        for (int it = 0; it < ITERS; ++it) {                                                    \
            _Pragma("unroll") for (int i = 0; i < CH; i += 2) { OPA(r[i], r[(i + 3) & 7]); OPB(r[i + 1], r[(i + 2) & 7]); } \
        }                                                                                       \
        __syncthreads();                                                                        \
        long long t1 = clock64();                                                               \
        uint32_t s = 0;                                                                         \
        for (int i = 0; i < CH; ++i) s ^= r[i];                                                 \
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                         \
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                        \
    }

KERNEL1(k_iadd3, OP_IADD3)
KERNEL1(k_lop3, OP_LOP3)
KERNEL1(k_shf, OP_SHF)
KERNEL1(k_prmt, OP_PRMT)
KERNEL1(k_vabs, OP_VABS)
KERNEL1(k_vadd2, OP_VADD2)
KERNEL1(k_vmin2, OP_VMIN2)
KERNEL1(k_vamx, OP_VAMX)
KERNEL1(k_relu, OP_RELU)
KERNEL1(k_imad, OP_IMAD)
KERNEL2(k_lop3_imad, OP_LOP3, OP_IMAD)
KERNEL2(k_prmt_imad, OP_PRMT, OP_IMAD)
KERNEL2(k_vabs_imad, OP_VABS, OP_IMAD)
KERNEL2(k_vadd2_imad, OP_VADD2, OP_IMAD)
KERNEL2(k_vmin2_imad, OP_VMIN2, OP_IMAD)
KERNEL2(k_relu_imad, OP_RELU, OP_IMAD)
KERNEL2(k_vamx_imad, OP_VAMX, OP_IMAD)
KERNEL2(k_prmt_lop3, OP_PRMT, OP_LOP3)
KERNEL2(k_vabs_lop3, OP_VABS, OP_LOP3)
KERNEL2(k_relu_lop3, OP_RELU, OP_LOP3)
KERNEL2(k_vadd2_lop3, OP_VADD2, OP_LOP3)
KERNEL2(k_iadd3_lop3, OP_IADD3, OP_LOP3)
KERNEL2(k_shf_imad, OP_SHF, OP_IMAD)
KERNEL2(k_iadd3_imad, OP_IADD3, OP_IMAD)

typedef void (*kfn)(uint32_t*, uint32_t, long long*);

int main() {
    struct { const char* name; kfn f; } ks[] = {
        {"IADD3", k_iadd3}, {"LOP3", k_lop3}, {"SHF", k_shf}, {"PRMT", k_prmt}, {"VABSDIFF4", k_vabs},
        {"VIADD.16x2", k_vadd2}, {"VIMNMX.S16x2", k_vmin2}, {"VIADDMNMX", k_vamx}, {"VIADDMNMX.RELU", k_relu},
        {"IMAD", k_imad}, {"LOP3+IMAD", k_lop3_imad}, {"PRMT+IMAD", k_prmt_imad}, {"VABSDIFF4+IMAD", k_vabs_imad},
        {"VIADD.16x2+IMAD", k_vadd2_imad}, {"VIMNMX+IMAD", k_vmin2_imad}, {"RELU+IMAD", k_relu_imad},
        {"VIADDMNMX+IMAD", k_vamx_imad}, {"PRMT+LOP3", k_prmt_lop3}, {"VABSDIFF4+LOP3", k_vabs_lop3},
        {"RELU+LOP3", k_relu_lop3}, {"VIADD.16x2+LOP3", k_vadd2_lop3}, {"IADD3+LOP3", k_iadd3_lop3},
        {"SHF+IMAD", k_shf_imad}, {"IADD3+IMAD", k_iadd3_imad}};
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
        k.f<<<sms, threads>>>(out, 0x01030507u, cyc);   // warm
        k.f<<<sms, threads>>>(out, 0x01030507u, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", k.name, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double inst = (double)(threads / 32) * ITERS * CH;
        printf("%-18s %.3f\n", k.name, inst / mx);
    }
    return 0;
}
