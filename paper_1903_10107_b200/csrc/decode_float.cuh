// decode_float.cuh -- exact floating-point layered BP (R26) on sm_100a:
// the reference the quantized decoder is measured against ("the floating-point version").
//
// Same schedule, stopping rule and outputs as the quantized decode_kernel (R10-R13, R16), but one
// frame per slot and fp32 state:
//   E (a posteriori LLR, Eq.(9)) in shared memory (global memory when n floats do not fit),
//   L (check-to-variable messages) in the per-slot global workspace, row-contiguous like the
//   quantized layout (word li.z + r * li.w + k), one float per word.
// Check node: Eq.(1) sign with the syndrome bit folded in (R5); Eq.(2)/(4) magnitude as the box-plus
// of Eq.(6) by the forward/backward schedule of R6, beta in the stable form of R26 with the
// accurate expf / log1pf (not the approximate intrinsics).  Variable node: Eq.(8) x = E - L,
// Eq.(9) E = x + L_new, no saturation.  Infinite LLRs are +-1000 (R26).
#pragma once
#include <cstdint>

namespace qkd {

constexpr int kFloatDMax = 32;          // check degrees handled by the float kernel (instances FD = 20, 32)
constexpr float kLlrKnown = 1000.0f;    // R26

struct FParams {
    const int4* layer;       // [Mb] (degree, first base edge, workspace offset, row stride)
    const int2* edge;        // [nbase] (J*Z, shift)
    int Mb, Z, nbase, n, m, mb8, nb8;
    long long n_edges, ws_words;
    const float* llr;        // [F][n]
    const uint8_t* syn;      // [F][mb8]
    long long F;
    int T, early_stop;
    float* Lws;              // [slots][ws_words]
    float* Ews;              // [slots][n] (global-E variant)
    int* work;
    uint8_t* bits;
    int32_t* iters;
    uint8_t* success;
    float* fL;               // [F][n_edges] canonical order, or null
    float* fE;               // [F][n], or null
    int TG, GPC, slot_bytes, e_bytes, tab_off;
};

// Eq.(6) for magnitudes, R26 stable form: min(a,b) + ln(1 + e^-(a+b)) - ln(1 + e^-|a-b|)
__device__ __forceinline__ float beta_f(float a, float b) {
    return fminf(a, b) + log1pf(expf(-(a + b))) - log1pf(expf(-fabsf(a - b)));
}

__device__ __forceinline__ int col_f(const int2 e, int r, int Z) {
    int idx = r + e.y;
    idx = idx >= Z ? idx - Z : idx;
    return e.x + idx;
}

// one check row r of a block row (degree D <= FD)
template <int FD>
__device__ __forceinline__ void row_update_f(const int2* __restrict__ et, int D, int Z, int r, float* E,
                                             float* __restrict__ Lrow, int s_i, bool first) {
    float x[FD], mg[FD], o[FD];
    int sg = s_i, neg = 0;
#pragma unroll
    for (int k = 0; k < FD; ++k) {
        if (k < D) {
            const float xv = E[col_f(et[k], r, Z)] - (first ? 0.0f : Lrow[k]);   // Eq.(8)
            x[k] = xv;
            mg[k] = fabsf(xv);
            const int nk = xv < 0.0f;
            neg |= nk << k;
            sg ^= nk;
        }
    }
    if (D == 1) {
        o[0] = kLlrKnown;                                  // empty box-plus (R26)
    } else {
        // forward chain F_k in o[k+1] scratch, backward chain accumulated in b; o_k = beta(F_{k-1}, B_{k+1})
        float F[FD];
        F[0] = mg[0];
#pragma unroll
        for (int k = 1; k < FD; ++k)
            if (k < D - 1) F[k] = beta_f(F[k - 1], mg[k]);
        float b = mg[D - 1];
        o[D - 1] = F[D - 2];
#pragma unroll
        for (int k = FD - 2; k >= 1; --k) {
            if (k <= D - 2) {
                o[k] = beta_f(F[k - 1], b);
                b = beta_f(mg[k], b);
            }
        }
        o[0] = b;
    }
#pragma unroll
    for (int k = 0; k < FD; ++k) {
        if (k < D) {
            const float ln = ((sg ^ (neg >> k)) & 1) ? -o[k] : o[k];     // Eq.(1)
            Lrow[k] = ln;
            E[col_f(et[k], r, Z)] = x[k] + ln;                          // Eq.(9)
        }
    }
}

// Flooding schedule: the check-node half of an iteration -- every row from the
// previous iteration's E and L (Eq.(8)), L_new stored; E is left untouched (the variable-node half,
// E_j = LLR_j + sum_i L_ij, runs after a barrier).
template <int FD>
__device__ __forceinline__ void row_check_f(const int2* __restrict__ et, int D, int Z, int r, const float* E,
                                            float* __restrict__ Lrow, int s_i, bool first) {
    float mg[FD], o[FD];
    int sg = s_i, neg = 0;
#pragma unroll
    for (int k = 0; k < FD; ++k) {
        if (k < D) {
            const float xv = E[col_f(et[k], r, Z)] - (first ? 0.0f : Lrow[k]);
            mg[k] = fabsf(xv);
            const int nk = xv < 0.0f;
            neg |= nk << k;
            sg ^= nk;
        }
    }
    if (D == 1) {
        o[0] = kLlrKnown;
    } else {
        float F[FD];
        F[0] = mg[0];
#pragma unroll
        for (int k = 1; k < FD; ++k)
            if (k < D - 1) F[k] = beta_f(F[k - 1], mg[k]);
        float b = mg[D - 1];
        o[D - 1] = F[D - 2];
#pragma unroll
        for (int k = FD - 2; k >= 1; --k) {
            if (k <= D - 2) {
                o[k] = beta_f(F[k - 1], b);
                b = beta_f(mg[k], b);
            }
        }
        o[0] = b;
    }
#pragma unroll
    for (int k = 0; k < FD; ++k)
        if (k < D) Lrow[k] = ((sg ^ (neg >> k)) & 1) ? -o[k] : o[k];
}

}  // namespace qkd
