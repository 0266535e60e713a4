// swar.cuh -- packed 4-frame (u8x4) and 2-frame (s16x2) integer arithmetic for the
// sm_100a decode kernels.  Each 32-bit word holds one int8 quantity for 4 independent
// frames (frame f in byte f).  Only ops that are native on sm_100a are used on the hot
// path: VABSDIFF4.U8, VIADD.16x2, VIMNMX.S16x2, VIADDMNMX.S16x2 (DPX), PRMT, LOP3, IADD3,
// SHF (see DESIGN.md §5 "instruction budget").
#pragma once
#include <cstdint>

namespace qkd {

// PTX prmt.b32 in its default mode: selector nibble bit 3 replicates the sign (bit 7) of the
// selected byte.  (__byte_perm masks the selector to 3 bits and loses that mode.)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ uint32_t rep4(uint32_t byte) { return byte * 0x01010101u; }

// Algorithm 1 on 4 byte lanes, inputs already clamped to [0, 63].
//   d = |a-b|, l = min(a,b) = (a+b-d)/2
//   tau = l - c,  c = [l>=3]([d<2]+[d<6]) + [1<=l<=2][d<4]      (l = 0 -> 0)
// The comparisons are read from bit 7 of (v + (128-k)), which never carries across a byte
// because v <= 63.  tau >= 0 in every lane, so the final subtraction never borrows.
__device__ __forceinline__ uint32_t tau4(uint32_t a, uint32_t b) {
    const uint32_t d = __vabsdiffu4(a, b);
    const uint32_t l = (a + b - d) >> 1;           // a+b-d = 2*min: even, so no byte leaks
    const uint32_t P = l + 0x7D7D7D7Du;            // bit7: l >= 3
    const uint32_t Q = l + 0x7F7F7F7Fu;            // bit7: l >= 1
    const uint32_t U = d + 0x7E7E7E7Eu;            // bit7: d >= 2
    const uint32_t W = d + 0x7C7C7C7Cu;            // bit7: d >= 4
    const uint32_t V = d + 0x7A7A7A7Au;            // bit7: d >= 6
    const uint32_t g1 = P & ~U & 0x80808080u;               // l>=3 and d<2
    const uint32_t t2 = P & ~V & 0x80808080u;               // l>=3 and d<6
    const uint32_t t1 = Q & ~W & 0x80808080u;               // l>=1 and d<4
    const uint32_t g2 = t2 | (t1 & ~P);                     // ... and l<=2
    return l - (g1 >> 7) - (g2 >> 7);
}

// zero-extend bytes {0,2} / {1,3} into 16-bit lanes
__device__ __forceinline__ uint32_t lo16z(uint32_t w) { return prmt(w, 0u, 0x4240u); }
__device__ __forceinline__ uint32_t hi16z(uint32_t w) { return prmt(w, 0u, 0x4341u); }
// sign-extend bytes {0,2} / {1,3} into 16-bit lanes
__device__ __forceinline__ uint32_t lo16s(uint32_t w) { return prmt(w, 0u, 0xA280u); }
__device__ __forceinline__ uint32_t hi16s(uint32_t w) { return prmt(w, 0u, 0xB391u); }
// pack the low bytes of two 16x2 words back into frame order {0,1,2,3}
__device__ __forceinline__ uint32_t pack16(uint32_t lo, uint32_t hi) { return prmt(lo, hi, 0x6240u); }
// byte mask 0xFF where bit 7 of the byte is set
__device__ __forceinline__ uint32_t bmask7(uint32_t w) { return prmt(w, 0u, 0xBA98u); }

// syndrome nibble (bit f = frame f) -> flag at bit 6 / bit 7 of byte f
__device__ __forceinline__ uint32_t nib_to_bit6(uint32_t nib) { return (nib * 0x08102040u) & 0x40404040u; }
__device__ __forceinline__ uint32_t nib_to_bit7(uint32_t nib) { return (nib * 0x10204080u) & 0x80808080u; }

}  // namespace qkd
