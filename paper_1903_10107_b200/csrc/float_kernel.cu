// float_kernel.cu -- exact floating-point layered / flooding BP kernel (decode_float.cuh; SURVEY §8(f)
// N1, N4), one frame per slot; instantiated here for qkd_ldpc.cu's fkernel().
#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"
#include "decode_float.cuh"

namespace qkd {

template <bool ESM, bool FLOOD, int FD>
__global__ void __launch_bounds__(1024, 1) decode_float_kernel(const FParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    int4* s_layer = reinterpret_cast<int4*>(smem + p.tab_off);
    int2* s_edge = reinterpret_cast<int2*>(s_layer + p.Mb);
    for (int i = threadIdx.x; i < p.Mb; i += blockDim.x) s_layer[i] = p.layer[i];
    for (int i = threadIdx.x; i < p.nbase; i += blockDim.x) s_edge[i] = p.edge[i];
    __syncthreads();
    const int slot = threadIdx.x / p.TG;
    const int t = threadIdx.x - slot * p.TG;
    const int bar = 1 + slot;
    const long long gslot = (long long)blockIdx.x * p.GPC + slot;
    unsigned char* sbase = smem + (size_t)slot * p.slot_bytes;
    float* E = ESM ? reinterpret_cast<float*>(sbase) : p.Ews + gslot * (long long)p.n;
    uint8_t* sSyn = sbase + p.e_bytes;
    int* ctl = reinterpret_cast<int*>(sSyn + ((p.m + 15) & ~15));
    float* Ls = p.Lws + gslot * p.ws_words;
    const int lane = threadIdx.x & 31;

    auto syndrome_ok = [&]() -> bool {   // every check row's parity of (E < 0) equals its target bit
        int v = 0;
        for (int I = 0; I < p.Mb; ++I) {
            const int4 li = s_layer[I];
            for (int r = t; r < p.Z; r += p.TG) {
                int par = sSyn[I * p.Z + r];
                for (int k = 0; k < li.x; ++k) par ^= E[col_f(s_edge[li.y + k], r, p.Z)] < 0.0f;
                v |= par;
            }
        }
        v = __reduce_or_sync(0xffffffffu, v);
        if (lane == 0 && v) atomicOr(&ctl[1], 1);
        group_bar(bar, p.TG);
        const int res = *(volatile int*)&ctl[1];
        group_bar(bar, p.TG);
        if (t == 0) ctl[1] = 0;
        return res == 0;
    };

    for (;;) {
        if (t == 0) { ctl[0] = atomicAdd(p.work, 1); ctl[1] = 0; }
        group_bar(bar, p.TG);
        const long long f = *(volatile int*)&ctl[0];
        if (f >= p.F) break;
        for (int j = t; j < p.n; j += p.TG) E[j] = p.llr[f * p.n + j];
        for (int i = t; i < p.m; i += p.TG) sSyn[i] = (p.syn[f * p.mb8 + (i >> 3)] >> (i & 7)) & 1;
        group_bar(bar, p.TG);
        int it = 0;
        bool ok = false;
        if (p.early_stop) ok = syndrome_ok();   // iteration-0 check (R10)
        while (!ok && it < p.T) {
            ++it;
            if constexpr (!FLOOD) {   // layered: each block row sees the previous ones' E
                for (int I = 0; I < p.Mb; ++I) {
                    const int4 li = s_layer[I];
                    for (int r = t; r < p.Z && li.x > 0; r += p.TG)
                        row_update_f<FD>(s_edge + li.y, li.x, p.Z, r, E, Ls + li.z + (long long)r * li.w,
                                     sSyn[I * p.Z + r], it == 1);
                    group_bar(bar, p.TG);
                }
            } else {                  // flooding (N4): all checks from the old state, then all VNs
                for (int I = 0; I < p.Mb; ++I) {
                    const int4 li = s_layer[I];
                    for (int r = t; r < p.Z && li.x > 0; r += p.TG)
                        row_check_f<FD>(s_edge + li.y, li.x, p.Z, r, E, Ls + li.z + (long long)r * li.w,
                                    sSyn[I * p.Z + r], it == 1);
                }
                group_bar(bar, p.TG);
                for (int j = t; j < p.n; j += p.TG) E[j] = p.llr[f * p.n + j];
                group_bar(bar, p.TG);
                for (int I = 0; I < p.Mb; ++I) {   // E_j = LLR_j + sum_i L_ij (float atomics: order varies)
                    const int4 li = s_layer[I];
                    for (int r = t; r < p.Z; r += p.TG) {
                        const float* Lrow = Ls + li.z + (long long)r * li.w;
                        for (int k = 0; k < li.x; ++k) atomicAdd(&E[col_f(s_edge[li.y + k], r, p.Z)], Lrow[k]);
                    }
                }
                group_bar(bar, p.TG);
            }
            if (p.early_stop) ok = syndrome_ok();
        }
        if (!p.early_stop) ok = syndrome_ok();   // R12
        // outputs: bits (E < 0, R9), iters, success; optional final L (canonical order) and E
        uint8_t* brow = p.bits + f * p.nb8;
        for (int jw = t & ~31; jw < p.n; jw += p.TG) {
            const int j = jw + lane;
            const bool b = j < p.n && E[j < p.n ? j : 0] < 0.0f;
            const uint32_t bal = __ballot_sync(0xffffffffu, b);
            const int byte = (jw >> 3) + lane;
            if (lane < 4 && byte < p.nb8) brow[byte] = (uint8_t)(bal >> (8 * lane));
        }
        if (p.fE)
            for (int j = t; j < p.n; j += p.TG) p.fE[f * p.n + j] = E[j];
        if (p.fL) {
            for (int I = 0; I < p.Mb; ++I) {
                const int4 li = s_layer[I];
                for (int q = t; q < li.x * p.Z; q += p.TG) {
                    const int k = q / p.Z, r = q - k * p.Z;
                    p.fL[f * p.n_edges + (long long)(li.y + k) * p.Z + r] =
                        it == 0 ? 0.0f : Ls[li.z + (long long)r * li.w + k];
                }
            }
        }
        if (t == 0) {
            p.iters[f] = it;
            p.success[f] = ok ? 1 : 0;
        }
        group_bar(bar, p.TG);
    }
}

template __global__ void decode_float_kernel<true, false, 20>(const FParams);
template __global__ void decode_float_kernel<true, true, 20>(const FParams);
template __global__ void decode_float_kernel<false, false, 20>(const FParams);
template __global__ void decode_float_kernel<false, true, 20>(const FParams);
template __global__ void decode_float_kernel<true, false, kFloatDMax>(const FParams);
template __global__ void decode_float_kernel<true, true, kFloatDMax>(const FParams);
template __global__ void decode_float_kernel<false, false, kFloatDMax>(const FParams);
template __global__ void decode_float_kernel<false, true, kFloatDMax>(const FParams);

}  // namespace qkd
