// pipe_probe2.cu -- issue rates of immediate-operand forms on sm_100a (does an immediate
// relieve the 3-register-read limit, as the microarch notes report for FFMA?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe2 tools/pipe_probe2.cu && ./pipe_probe2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048

// r: chain register, c: another live register, k: opaque runtime constant register
#define OP_IMAD_RRR(r, c, k) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r) : "r"(k), "r"(c))
#define OP_IMAD_RRI(r, c, k) asm volatile("mad.lo.u32 %0, %0, %1, 0x3D3D3D3D;" : "+r"(r) : "r"(k))
#define OP_IMAD_RIR(r, c, k) asm volatile("mad.lo.u32 %0, %0, 0x01010101, %1;" : "+r"(r) : "r"(c))
#define OP_IMAD_RI(r, c, k) asm volatile("mul.lo.u32 %0, %0, 0x01010101;" : "+r"(r))
#define OP_FFMA_RRR(r, c, k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r) : "r"(k), "r"(c))
#define OP_FFMA_RIR(r, c, k) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, %1;" : "+r"(r) : "r"(c))
#define OP_HFMA2_RRR(r, c, k) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r) : "r"(k), "r"(c))
#define OP_HADD2(r, c, k) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(r) : "r"(c))
#define OP_LOP3_RRR(r, c, k) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r) : "r"(c), "r"(k))
#define OP_LOP3_RRI(r, c, k) asm volatile("lop3.b32 %0, %0, %1, 0x40404040, 0x20;" : "+r"(r) : "r"(c))
#define OP_IADD3_RRR(r, c, k) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(r) : "r"(c), "r"(k))
#define OP_IADD_RI(r, c, k) asm volatile("add.u32 %0, %0, 0x3D3D3D3D;" : "+r"(r))
#define OP_SHF_I(r, c, k) asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(r) : "r"(c))
#define OP_PRMT_I(r, c, k) asm volatile("prmt.b32 %0, %0, %1, 0x6240;" : "+r"(r) : "r"(c))
#define OP_VABS(r, c, k) r = __vabsdiffu4(r, c)
#define OP_RELU_RRI(r, c, k) r = __viaddmin_s16x2_relu(r, c, 0x007E007Eu)
#define OP_RELU_RRR(r, c, k) r = __viaddmin_s16x2_relu(r, c, k)
#define OP_DP4A(r, c, k) asm volatile("dp4a.u32.u32 %0, %0, %1, %0;" : "+r"(r) : "r"(c))
#define OP_VMIN2(r, c, k) r = __vmins2(r, c)
#define OP_IMNMX(r, c, k) asm volatile("min.u32 %0, %0, %1;" : "+r"(r) : "r"(c))
#define OP_VADD2(r, c, k) r = __vadd2(r, c)

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

KERNEL1(k1, OP_IMAD_RRR) KERNEL1(k2, OP_IMAD_RRI) KERNEL1(k3, OP_IMAD_RIR) KERNEL1(k4, OP_IMAD_RI)
KERNEL1(k5, OP_FFMA_RRR) KERNEL1(k6, OP_FFMA_RIR) KERNEL1(k7, OP_HFMA2_RRR) KERNEL1(k8, OP_HADD2)
KERNEL1(k9, OP_LOP3_RRR) KERNEL1(k10, OP_LOP3_RRI) KERNEL1(k11, OP_IADD3_RRR) KERNEL1(k12, OP_IADD_RI)
KERNEL1(k13, OP_SHF_I) KERNEL1(k14, OP_PRMT_I) KERNEL1(k15, OP_VABS) KERNEL1(k16, OP_RELU_RRI)
KERNEL1(k17, OP_RELU_RRR) KERNEL1(k18, OP_DP4A) KERNEL1(k19, OP_VMIN2) KERNEL1(k20, OP_IMNMX)
KERNEL1(k21, OP_VADD2)
KERNEL2(p1, OP_LOP3_RRI, OP_IMAD_RRI) KERNEL2(p2, OP_LOP3_RRR, OP_IMAD_RRR) KERNEL2(p3, OP_IMAD_RRI, OP_FFMA_RIR)
KERNEL2(p4, OP_LOP3_RRI, OP_FFMA_RIR) KERNEL2(p5, OP_IMAD_RRI, OP_HFMA2_RRR) KERNEL2(p6, OP_LOP3_RRI, OP_HFMA2_RRR)
KERNEL2(p7, OP_IMAD_RRI, OP_DP4A) KERNEL2(p8, OP_LOP3_RRI, OP_DP4A) KERNEL2(p9, OP_IMAD_RRI, OP_VADD2)
KERNEL2(p10, OP_LOP3_RRI, OP_VADD2) KERNEL2(p11, OP_IMAD_RRI, OP_IMAD_RIR) KERNEL2(p12, OP_IMAD_RRI, OP_IMAD_RRR)
KERNEL2(p13, OP_IMAD_RRI, OP_IMNMX) KERNEL2(p14, OP_VABS, OP_IMAD_RRI) KERNEL2(p15, OP_IMAD_RRI, OP_HADD2)

typedef void (*kfn)(uint32_t*, uint32_t, long long*);

int main() {
    struct { const char* name; kfn f; } ks[] = {
        {"IMAD r,r,R,R", k1}, {"IMAD r,r,R,imm", k2}, {"IMAD r,r,imm,R", k3}, {"IMUL r,r,imm", k4},
        {"FFMA RRR", k5}, {"FFMA R,imm,R", k6}, {"HFMA2 RRR", k7}, {"HADD2", k8},
        {"LOP3 RRR", k9}, {"LOP3 RR,imm", k10}, {"IADD3 RRR(2x)", k11}, {"IADD r,imm", k12},
        {"SHF imm", k13}, {"PRMT imm", k14}, {"VABSDIFF4", k15}, {"RELU RR,imm", k16},
        {"RELU RRR", k17}, {"DP4A", k18}, {"VMIN S16x2", k19}, {"IMNMX", k20}, {"VADD2", k21},
        {"LOP3i+IMADi", p1}, {"LOP3+IMAD RRR", p2}, {"IMADi+FFMAi", p3}, {"LOP3i+FFMAi", p4},
        {"IMADi+HFMA2", p5}, {"LOP3i+HFMA2", p6}, {"IMADi+DP4A", p7}, {"LOP3i+DP4A", p8},
        {"IMADi+VADD2", p9}, {"LOP3i+VADD2", p10}, {"IMADi+IMAD imm-mul", p11}, {"IMADi+IMAD RRR", p12},
        {"IMADi+IMNMX", p13}, {"VABS+IMADi", p14}, {"IMADi+HADD2", p15}};
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
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", k.name, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double inst = (double)(threads / 32) * ITERS * CH;
        printf("%-22s %.3f\n", k.name, inst / mx);
    }
    return 0;
}
