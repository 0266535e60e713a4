// decode.cuh -- the fused layered decode (check node + variable node + syndrome check +
// early exit) for one frame group of 4 frames held in byte lanes.
//
// Storage forms:
//   E word   (shared memory, or global for very long frames): byte f = E_j(frame f) + 128
//   N word   (global workspace, canonical edge order):          byte f = 64 - L_ij(frame f)
// so that x + 192 = E' + N' (Eq.(8): x = L_ji = E_j' - L_ij^{t-1}) is a plain 16-bit lane add
// with no overflow (x in [-190, 190]).
#pragma once
#include "swar.cuh"

namespace qkd {

struct DecParams {
    const int2* layer;        // [Mb] (degree, first base edge)
    const int2* edge;         // [nbase] (J*Z, shift)
    int Mb, Z, nbase, n, m, mb8, nb8;
    long long n_edges;
    const int8_t* llr;        // [F][n]
    const uint8_t* syn;       // [F][mb8]
    long long F, ngroups;
    int T, early_stop, vec_llr;
    uint32_t* Lws;            // [slots][n_edges]
    uint32_t* Ews;            // [slots][n]   (global-E variant only)
    int* work;                // group work counter
    uint8_t* bits;            // [F][nb8]
    int32_t* iters;
    uint8_t* success;
    int8_t* fL;               // [F][n_edges] or null
    int8_t* fE;               // [F][n] or null
    unsigned long long* counters;   // [5] or null
    int TG, GPC, tab_bytes, group_bytes, e_smem;
};

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <bool ESM>
__device__ __forceinline__ uint32_t ldE(const uint32_t* E, int j) {
    return E[j];   // shared (ESM) or global; bar.sync orders both for the group
}
template <bool ESM>
__device__ __forceinline__ void stE(uint32_t* E, int j, uint32_t v) {
    E[j] = v;
}

// x192 = x + 192 in two 16x2 words, clamped/packed check input cw = clamp(x,-63,63)+192
struct EdgeIn {
    uint32_t xlo, xhi, cw;
};

__device__ __forceinline__ EdgeIn edge_in(uint32_t ew, uint32_t nw) {
    EdgeIn r;
    r.xlo = __vadd2(lo16z(ew), lo16z(nw));
    r.xhi = __vadd2(hi16z(ew), hi16z(nw));
    const uint32_t clo = __vmins2(__vmaxs2(r.xlo, 0x00810081u), 0x00FF00FFu);
    const uint32_t chi = __vmins2(__vmaxs2(r.xhi, 0x00810081u), 0x00FF00FFu);
    r.cw = pack16(clo, chi);          // bytes in [129, 255]; bit 6 = (x >= 0)
    return r;
}
// check-node magnitude min(|x|, 63) (MSG_max = 63)
__device__ __forceinline__ uint32_t edge_mag(uint32_t cw) { return __vabsdiffu4(cw, 0xC0C0C0C0u); }

// Given the leave-one-out magnitude o, the sign flag (bit 6 of negf = 1 -> L_new < 0), the
// edge's x192 words and the pre-layer E word: returns the new N word (stored) and writes
// the new E word (Algorithm 2 guard on |E'| = E_max, Eq.(9) saturated to +-127).
__device__ __forceinline__ uint32_t edge_out(uint32_t o, uint32_t negf, const EdgeIn& in, uint32_t ew,
                                             uint32_t& e_out) {
    const uint32_t M = bmask7(negf << 1);                    // 0xFF where L_new < 0
    const uint32_t a = o ^ (M & 0x3F3F3F3Fu);                // o or 63-o
    const uint32_t bp = (M & 0x41414141u) ^ 0xC0C0C0C0u;     // 192 or 129
    const uint32_t Tp = a + bp;                              // (64 + L_new) + 128
    const uint32_t Np = 0x01010100u - a - bp;                // 64 - L_new
    // E' + L_new - L_old clamped: lanes = max(x192 + T - 128, 1) then min 255
    const uint32_t elo = __vmins2(__viaddmax_s16x2(in.xlo, lo16s(Tp), 0x00010001u), 0x00FF00FFu);
    const uint32_t ehi = __vmins2(__viaddmax_s16x2(in.xhi, hi16s(Tp), 0x00010001u), 0x00FF00FFu);
    const uint32_t enew = pack16(elo, ehi);
    const uint32_t G = bmask7(__vabsdiffu4(ew, 0x80808080u) + 0x01010101u);   // |E| == 127
    e_out = (G & ew) | (~G & enew);
    return Np;
}

// One check row r of a block row with D edges (layered update, Alg. 1/2).
template <int D, bool ESM>
__device__ __forceinline__ void row_update(const int2* __restrict__ et, int Z, int r, uint32_t* E,
                                           uint32_t* __restrict__ Lrow, uint32_t nib, bool first) {
    int addr[D];
    EdgeIn in[D];
    uint32_t P = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const int2 e = et[k];
        int idx = r + e.y;
        idx = idx >= Z ? idx - Z : idx;
        addr[k] = e.x + idx;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const uint32_t ew = ldE<ESM>(E, addr[k]);
        const uint32_t nw = first ? 0x40404040u : Lrow[(size_t)k * Z + r];
        in[k] = edge_in(ew, nw);
        P ^= in[k].cw;
    }
    // Eq.(1) with the target bit: L_new of edge k is negative iff
    // s_i ^ XOR_{j != k} [x_j < 0] = s_i ^ ((D-1)&1) ^ P ^ nonneg_k   (bit 6)
    const uint32_t Q = P ^ nib_to_bit6(nib) ^ (((D - 1) & 1) ? 0x40404040u : 0u);
    // emit edge k as soon as its leave-one-out magnitude is known (keeps the live set small)
    auto emit = [&](int k, uint32_t o) {
        const uint32_t ew = ldE<ESM>(E, addr[k]);
        uint32_t eo;
        const uint32_t np = edge_out(o, Q ^ in[k].cw, in[k], ew, eo);
        stE<ESM>(E, addr[k], eo);
        Lrow[(size_t)k * Z + r] = np;
    };
    if constexpr (D == 1) {
        emit(0, 0x3F3F3F3Fu);                       // empty box-plus -> MSG_max (R6)
    } else if constexpr (D == 2) {
        emit(0, edge_mag(in[1].cw));
        emit(1, edge_mag(in[0].cw));
    } else {
        // forward/backward leave-one-out in ascending block column (R6)
        uint32_t F[D - 1];
        F[0] = edge_mag(in[0].cw);
#pragma unroll
        for (int k = 1; k <= D - 2; ++k) F[k] = tau4(F[k - 1], edge_mag(in[k].cw));
        emit(D - 1, F[D - 2]);
        uint32_t B = edge_mag(in[D - 1].cw);
#pragma unroll
        for (int k = D - 2; k >= 1; --k) {
            emit(k, tau4(F[k - 1], B));
            B = tau4(edge_mag(in[k].cw), B);
        }
        emit(0, B);
    }
}

// Runtime-degree variant (any degree <= 64), same arithmetic; state in local memory.
template <bool ESM>
__device__ __noinline__ void row_update_generic(const int2* __restrict__ et, int D, int Z, int r,
                                                uint32_t* E, uint32_t* __restrict__ Lrow, uint32_t nib,
                                                bool first) {
    int addr[64];
    EdgeIn in[64];
    uint32_t F[64], o[64];
    uint32_t P = 0;
    for (int k = 0; k < D; ++k) {
        const int2 e = et[k];
        int idx = r + e.y;
        idx = idx >= Z ? idx - Z : idx;
        addr[k] = e.x + idx;
        const uint32_t ew = ldE<ESM>(E, addr[k]);
        const uint32_t nw = first ? 0x40404040u : Lrow[(size_t)k * Z + r];
        in[k] = edge_in(ew, nw);
        P ^= in[k].cw;
    }
    const uint32_t Q = P ^ nib_to_bit6(nib) ^ (((D - 1) & 1) ? 0x40404040u : 0u);
    if (D == 1) {
        o[0] = 0x3F3F3F3Fu;
    } else if (D == 2) {
        o[0] = edge_mag(in[1].cw);
        o[1] = edge_mag(in[0].cw);
    } else {
        F[0] = edge_mag(in[0].cw);
        for (int k = 1; k <= D - 2; ++k) F[k] = tau4(F[k - 1], edge_mag(in[k].cw));
        uint32_t B = edge_mag(in[D - 1].cw);
        o[D - 1] = F[D - 2];
        for (int k = D - 2; k >= 1; --k) {
            o[k] = tau4(F[k - 1], B);
            B = tau4(edge_mag(in[k].cw), B);
        }
        o[0] = B;
    }
    for (int k = 0; k < D; ++k) {
        const uint32_t ew = ldE<ESM>(E, addr[k]);
        uint32_t eo;
        const uint32_t np = edge_out(o[k], Q ^ in[k].cw, in[k], ew, eo);
        stE<ESM>(E, addr[k], eo);
        Lrow[(size_t)k * Z + r] = np;
    }
}

}  // namespace qkd
