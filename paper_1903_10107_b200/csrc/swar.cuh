// swar.cuh -- packed 4-frame (u8x4) and 2-frame (16x2) integer arithmetic for the sm_100a
// decode kernels.  Each 32-bit word holds one int8 quantity for 4 independent frames (frame f
// in byte f).  Only ops that are native on sm_100a are used:
//   ALU pipe: LOP3, IADD3, SHF, PRMT, VABSDIFF4.U8, VIMNMX/VIADDMNMX(.RELU).S16x2 (one warp
//             instruction every 2 cycles per SM sub-partition)
//   FMA pipe: IMAD (every operand form), VIADD.16x2 (one every 2 cycles)
// (tools/pipe_probe*.cu on the B200, profiles/r2_pipe_probe*.txt).  The row update is bound by
// instruction issue first, then by these pipes: adds of constants, shifts-left, negations
// and 16-bit lane unpacking go through IMAD with an opaque runtime multiplier (Konst) where that keeps
// the ALU pipe's half-rate ops from queueing, IADD3 where the ALU pipe has room.
#pragma once
#include <cstdint>


namespace qkd {

// runtime constants 1, 2, -1, -2, -256, the lane bias -128|-128, the byte constants
// 0x3F3F3F3F / 0x7F7F7F7F, 0 and 256 (kernel parameters, opaque
// to the compiler); in_regs() pins them in ordinary registers so ptxas neither folds them nor
// re-materialises them per use.
struct Konst {
    uint32_t one, two, m1, m2, m256, b128, c63, c127, zero, p256, p31, p26;
    __device__ __forceinline__ Konst in_regs() const {
        Konst k;
        asm volatile("mov.b32 %0, %1;" : "=r"(k.one) : "r"(one));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.two) : "r"(two));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.m1) : "r"(m1));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.m2) : "r"(m2));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.m256) : "r"(m256));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.b128) : "r"(b128));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.c63) : "r"(c63));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.c127) : "r"(c127));
        k.zero = zero;   // used only as an opaque operand (scheduling dependencies), not pinned
        asm volatile("mov.b32 %0, %1;" : "=r"(k.p256) : "r"(p256));
#if QKD_TAU_WIDE == 2
        asm volatile("mov.b32 %0, %1;" : "=r"(k.p31) : "r"(p31));
        asm volatile("mov.b32 %0, %1;" : "=r"(k.p26) : "r"(p26));
#else
        k.p31 = p31;
        k.p26 = p26;
#endif
        return k;
    }
};

// PTX prmt.b32 in its default mode: selector nibble bit 3 replicates the sign (bit 7) of the
// selected byte.  (__byte_perm masks the selector to 3 bits and loses that mode.)
template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "n"(SEL));
    return r;
}
__device__ __forceinline__ uint32_t rep4(uint32_t byte) { return byte * 0x01010101u; }

// a*m + c on the FMA pipe
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t m, uint32_t c) { return a * m + c; }
// a*M + c with an immediate multiplier (|M| != 1: ptxas keeps these as IMAD, no constant register)
template <int M>
__device__ __forceinline__ uint32_t imadi(uint32_t a, uint32_t c) {
    uint32_t r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "n"(M), "r"(c));
    return r;
}
// LOP3 with an explicit truth table (a = 0xF0, b = 0xCC, c = 0xAA).  Written as PTX so ptxas does
// not fold a NOT into a neighbouring add (it rewrites ~(d + k) as -d - k - 1, costing a negate).
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return r;
}
template <uint32_t LUT, uint32_t C>
__device__ __forceinline__ uint32_t lop3i(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "n"(C), "n"(LUT));
    return r;
}
// max(min(a + b, c), 0) per signed 16-bit lane (DPX VIADDMNMX.S16x2.RELU)
__device__ __forceinline__ uint32_t relu_min(uint32_t a, uint32_t b, uint32_t c) {
    return __viaddmin_s16x2_relu(a, b, c);
}

// Algorithm 1 on 4 byte lanes, inputs already clamped to [0, 63].
//   d = |a-b|, l = min(a,b) = (a+b-d)/2
//   tau = l - c,  c = [l>=3]([d<2] + [d<6]) + [1<=l<=2][d<4]      (l = 0 -> 0)
// Each comparison v >= k is bit 6 of v + (64 - k), clean because v <= 63 (no carry leaves
// the byte).  The two correction flags g1, g2 sit at bit 6, so g1 + g2 <= 0x80 never carries
// and c = (g1 + g2) >> 6.  tau >= 0 in every lane, so l - c never borrows.
__device__ __forceinline__ uint32_t tau4(uint32_t a, uint32_t b, const Konst& K) {
    const uint32_t d = __vabsdiffu4(a, b);                       // ALU
    const uint32_t l = imad(d, K.m1, imad(a, K.one, b)) >> 1;    // 2 FMA + SHF
    const uint32_t P = imad(l, K.one, 0x3D3D3D3Du);              // bit6: l >= 3
    const uint32_t Q = imad(l, K.one, 0x3F3F3F3Fu);              // bit6: l >= 1
    const uint32_t U = imad(d, K.one, 0x3E3E3E3Eu);              // bit6: d >= 2
    const uint32_t W = imad(d, K.one, 0x3C3C3C3Cu);              // bit6: d >= 4
    const uint32_t V = imad(d, K.one, 0x3A3A3A3Au);              // bit6: d >= 6
    const uint32_t g1 = lop3i<0x20, 0x40404040u>(P, U);          // P & ~U & M: l>=3, d<2
    const uint32_t t2 = lop3i<0x20, 0x40404040u>(P, V);          // P & ~V & M: l>=3, d<6
    const uint32_t t1 = lop3i<0x20, 0x40404040u>(Q, W);          // Q & ~W & M: l>=1, d<4
    const uint32_t g2 = lop3<0xF4>(t2, t1, P);                   // t2 | (t1 & ~P): ... l<=2
    const uint32_t c = imad(g1, K.one, g2) >> 6;
    return imad(c, K.m1, l);
}

// The same Algorithm 1 in complement form: a' = 63 - a, b' = 63 - b in, 63 - tau(a, b) out.
// Then g = max(a', b') = 63 - l = (a' + b' + d) / 2 is one IADD3 + SHF, and 63 - tau = g + c is one
// LEA.HI of the flag word (c = (g1 + g2) >> 6), two instructions fewer than tau4.
//   l <= 2  <=>  g >= 61  (bit 6 of g + 3);   l == 0  <=>  g == 63  (bit 6 of g + 1)
//   c = [l>=3]([d<2] + [d<6]) + [1<=l<=2][d<4]  as above.
//
// Default form (12 SASS: 7 ALU, 5 FMA): the same correction regrouped by the rows of Algorithm 1's
// table,  c = [l>=1][d<4] + [l>=3][d in {0,1,4,5}]
//   (l>=3: d<2 -> 1+1, d in 2..3 -> 1+0, d in 4..5 -> 0+1, d>=6 -> 0;  l in 1..2: [d<4];  l = 0: 0)
// and d in {0,1,4,5} <=> (d & 0x3A) == 0 for d <= 63 (bits 1, 3, 4, 5 clear), so two masked flag
// words replace three.  Checked against Algorithm 1 over all 64 x 64 inputs on the device (qkd_tau_table).
#ifndef QKD_TAU_WIDE
#define QKD_TAU_WIDE 0   // experiment (bit-exact, slower: C5a +3.9 % with 1, +13 % with 3; profiles/r2q_ab.txt)
#endif
__device__ __forceinline__ uint32_t tau4c(uint32_t a, uint32_t b, const Konst& K) {
    const uint32_t d = __vabsdiffu4(a, b);                       // ALU
#if QKD_TAU_WIDE
    // Right shifts on the FMA pipe as the high word of a wide multiply by an opaque power of two (IMAD.WIDE):
    // bit 0: g = hi((a + b + d) 2^31) instead of SHF;  bit 1: c = hi(y 2^26) + a plain add instead of LEA.HI.
    unsigned long long w1;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(w1) : "r"(a + b + d), "r"(K.p31));
    const uint32_t g = (uint32_t)(w1 >> 32);
    const uint32_t z = g + 0x01010101u;
    const uint32_t p = g + 0x03030303u;
    const uint32_t W = d + 0x3C3C3C3Cu;
    const uint32_t Ep = (d & 0x3A3A3A3Au) + 0x3F3F3F3Fu;
    const uint32_t t1 = lop3i<0x02, 0x40404040u>(z, W);
    const uint32_t t2 = lop3i<0x02, 0x40404040u>(p, Ep);
    const uint32_t y = t1 + t2;
#if QKD_TAU_WIDE & 2
    unsigned long long w2;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(w2) : "r"(y), "r"(K.p26));
    return g + (uint32_t)(w2 >> 32);
#else
    return g + (y >> 6);
#endif
#elif QKD_TAU_S
    // experiment: the l-flags from s = 2g (bit 7) so the shift leaves the dependent chain; costs a second LEA.HI
    const uint32_t s = a + b + d;
    const uint32_t g = s >> 1;
    const uint32_t z = s + 0x02020202u;                          // bit7: l == 0
    const uint32_t p = s + 0x06060606u;                          // bit7: l <= 2
    const uint32_t W = d + 0x7C7C7C7Cu;                          // bit7: d >= 4
    const uint32_t Ep = (d & 0x3A3A3A3Au) + 0x7F7F7F7Fu;         // bit7: d not in {0,1,4,5}
    const uint32_t t1 = lop3i<0x02, 0x80808080u>(z, W);
    const uint32_t t2 = lop3i<0x02, 0x80808080u>(p, Ep);
    return g + (t1 >> 7) + (t2 >> 7);
#else
#if QKD_TAU_IMAD
    const uint32_t g = imad(a, K.one, imad(b, K.one, d)) >> 1;   // 2 IMAD + SHF (experiment)
#else
    const uint32_t g = (a + b + d) >> 1;                         // IADD3 + SHF (a+b+d = 2 max <= 126)
#endif
#ifndef QKD_TAU14
#ifndef QKD_TAU_ADDS
#define QKD_TAU_ADDS 3   // which of the tau's constant adds are plain adds (ptxas: VIADD) instead of IMAD;
                         // 3 (the four threshold adds) measured 1 % faster on C5a than 0 (all IMAD)
#endif
#define QKD_ADD(x, c, BIT) ((QKD_TAU_ADDS & (BIT)) ? (x) + (c) : imad((x), K.one, (c)))
    const uint32_t z = QKD_ADD(g, 0x01010101u, 1);               // bit6: l == 0
    const uint32_t p = QKD_ADD(g, 0x03030303u, 1);               // bit6: l <= 2
    const uint32_t W = QKD_ADD(d, 0x3C3C3C3Cu, 2);               // bit6: d >= 4
    const uint32_t Ep = QKD_ADD(d & 0x3A3A3A3Au, 0x3F3F3F3Fu, 2);   // bit6: d not in {0,1,4,5}
    const uint32_t t1 = lop3i<0x02, 0x40404040u>(z, W);          // ~z & ~W & M: l>=1, d<4
    const uint32_t t2 = lop3i<0x02, 0x40404040u>(p, Ep);         // ~p & ~Ep & M: l>=3, d in {0,1,4,5}
    const uint32_t y = QKD_ADD(t1, t2, 4);                       // 64 c per byte (<= 0x80)
#undef QKD_ADD
    return g + (y >> 6);                                         // LEA.HI: 63 - (l - c)
#else
    const uint32_t p = imad(g, K.one, 0x03030303u);              // bit6: l <= 2
    const uint32_t z = imad(g, K.one, 0x01010101u);              // bit6: l == 0
    const uint32_t U = imad(d, K.one, 0x3E3E3E3Eu);              // bit6: d >= 2
    const uint32_t W = imad(d, K.one, 0x3C3C3C3Cu);              // bit6: d >= 4
    const uint32_t V = imad(d, K.one, 0x3A3A3A3Au);              // bit6: d >= 6
    const uint32_t g1 = lop3i<0x02, 0x40404040u>(p, U);          // ~p & ~U & M: l>=3, d<2
    const uint32_t A = lop3i<0x02, 0x40404040u>(z, W);           // ~z & ~W & M: l>=1, d<4
    const uint32_t t2 = lop3i<0x02, 0x40404040u>(p, V);          // ~p & ~V & M: l>=3, d<6
    const uint32_t g2 = lop3<0xF8>(t2, p, A);                    // t2 | (p & A)
    const uint32_t y = imad(g1, K.one, g2);                      // 64 c per byte (g1 => g2: <= 0x80)
    return g + (y >> 6);                                         // LEA.HI: 63 - (l - c)
#endif
#endif
}

// sign-extend bytes {1,3} into 16-bit lanes / zero-extend bytes {1,3}
__device__ __forceinline__ uint32_t hi16s(uint32_t w) { return prmt<0xB391u>(w, 0u); }
__device__ __forceinline__ uint32_t hi16z(uint32_t w) { return prmt<0x4341u>(w, 0u); }
// sign-extend bytes {0,2} into 16-bit lanes
__device__ __forceinline__ uint32_t lo16s(uint32_t w) { return prmt<0xA280u>(w, 0u); }
// pack the low bytes of two 16x2 words back into frame order {0,1,2,3}
__device__ __forceinline__ uint32_t pack16(uint32_t lo, uint32_t hi) { return prmt<0x6240u>(lo, hi); }
// the same for clean lanes (every 16-bit lane in [0, 255]) on the FMA pipe: lo + 256 hi
__device__ __forceinline__ uint32_t pack16c(uint32_t lo, uint32_t hi, const Konst& K) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(r) : "r"(hi), "r"(lo));
    return r;
}
// byte mask 0xFF where bit 7 of the byte is set
__device__ __forceinline__ uint32_t bmask7(uint32_t w) { return prmt<0xBA98u>(w, 0u); }

// lane nibble (bit f = frame lane f) -> byte mask 0xFF in byte f
__device__ __forceinline__ uint32_t fresh_mask(uint32_t nib) { return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu; }

// syndrome nibble (bit f = frame f) -> flag at bit 6 / bit 7 of byte f
__device__ __forceinline__ uint32_t nib_to_bit6(uint32_t nib) { return (nib * 0x08102040u) & 0x40404040u; }
__device__ __forceinline__ uint32_t nib_to_bit7(uint32_t nib) { return (nib * 0x10204080u) & 0x80808080u; }

}  // namespace qkd
