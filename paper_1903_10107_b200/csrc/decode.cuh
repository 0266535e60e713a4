// decode.cuh -- the fused layered decode (check node + variable node) for one check row of
// one frame group (4 frames held in the 4 byte lanes of every 32-bit word).
//
// Storage forms:
//   E word (shared memory, or global for very long frames): byte f = E_j(frame f) + 127
//   T word (global workspace):                               byte f = 192 + L_ij(frame f)
// so that X = x + 191 = E'' + 256 - T (Eq.(8): x = L_ji = E_j' - L_ij^{t-1}, exact, in
// [-190, 190]) is a sum of non-negative 16-bit lanes, and the check node's output byte
// T = 192 + L_new is stored as computed.
//
// Workspace layout: per slot, per block row I, the rows' message words in emission order,
// position-major (msg_word below); the lane-pair variant keeps its own row layout.
#pragma once
#include "swar.cuh"


namespace qkd {

struct DecParams {
    const int4* layer;        // [Mb] (degree, first base edge, L offset in words, words per row)
    const int2* edge;         // [nbase] (J*Z, shift)
    const int* soff;          // [Mb] split-table offset of block row I (entries; split layout only)
    int nsplit;               // split-table entries per slot (sum over I of 2 * HB_I)
    int Mb, Z, nbase, n, m, mb8, nb8;
    long long n_edges;        // canonical message count (nbase * Z)
    long long ws_words;       // workspace words per slot (sum over I of Z * words per row)
    const int8_t* llr;        // [F][n]
    const uint8_t* syn;       // [F][mb8]
    long long F, ngroups;
    const long long* F_dev;   // device-resident frame count (<= F) read at kernel start, or null
    int T, early_stop, vec_llr;
    int refill;               // per-frame lane refill (early_stop only, not the lane-pair variant)
    uint32_t* Lws;            // [slots][ws_words]
    uint32_t* Ews;            // [slots][n]   (global-E variant only)
    int* work;                // group work counter
    uint8_t* bits;            // [F][nb8]
    int32_t* iters;
    uint8_t* success;
    int8_t* fL;               // [F][n_edges] or null
    int8_t* fE;               // [F][n] or null
    unsigned long long* counters;   // [5] or null
    unsigned* dbg;            // QKD_RACECHECK builds only: [16] error record, then [slots][n] layer stamps
    const int* dbg_delta;     // QKD_RACECHECK builds only: per base edge, layers back to the previous writer
    int TG, GPC, slot_bytes, e_bytes, tab_off;
    Konst K;
};

constexpr int kFramesPerGroup = 4;   // frames per SWAR word (one byte lane each)

#ifndef QKD_KEEP_ADDR
#define QKD_KEEP_ADDR 10   // rows of degree <= this keep their E addresses in registers
#endif
#ifndef QKD_D32_THREADS
#define QKD_D32_THREADS 512
#endif
#define QKD_D32_TG(DMAX) ((DMAX) == 32 ? QKD_D32_THREADS : 512)
#ifndef QKD_V1_THREADS
#define QKD_V1_THREADS 1024   // variant 1 (degree <= 8, E in shared memory): threads per CTA.  768 (80 registers, no
                              // spill in the refill kernel) speeds C2 at its 1024 frames up 10 % but slows the bench's
                              // 65536-frame C5b by 3 % (17.6 -> 18.2 ms), so the bench's configuration keeps 1024.
#endif
#ifndef QKD_G8_THREADS
#define QKD_G8_THREADS 1024   // variant 7 (degree <= 8, E in global memory): threads per CTA (C4: 512 -> 1024
#endif                        // with QKD_G8_LOWREG, 69.2 -> 61.7 ms; 768 threads: 72.2 ms, uneven rows)
#ifndef QKD_G32_THREADS
#define QKD_G32_THREADS 256   // variant 8 (degree <= 32, E in global memory): 254 registers, no spills
#endif

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// E addressing.  POW2: a = ((r4 + s4) & (4Z - 1)) | cb4, all in bytes, cb4 = slot E base + J*Z*4
// (slot bases are multiples of 4Z, see make_plan), one IMAD + one LOP3 per edge.  Otherwise
// words: j = J*Z + (r + s) mod Z.
// experiments (A/B): bit 1 the guard's +1, bit 2 the magnitude's 63 - v, bit 4 the circulant address add
// as plain adds (ptxas: VIADD / IADD3) instead of IMAD with the opaque multiplier
#ifndef QKD_VIADD_MISC
#define QKD_VIADD_MISC 0
#endif
#define QKD_MISC_ADD(x, c, BIT) ((QKD_VIADD_MISC & (BIT)) ? (x) + (c) : imad((x), K.one, (c)))

template <bool POW2>
struct Addr {
    __device__ __forceinline__ static uint32_t at(int2 e, uint32_t r4, uint32_t zm4, int Z, const Konst& K) {
        if constexpr (POW2) {
            return (QKD_MISC_ADD(r4, (uint32_t)e.y, 4) & zm4) | (uint32_t)e.x;
        } else {
            int idx = (int)(r4 >> 2) + e.y;
            idx = idx >= Z ? idx - Z : idx;
            return (uint32_t)(e.x + idx) << 2;
        }
    }
};

template <bool ESM>
__device__ __forceinline__ uint32_t ldE(const unsigned char* Eb, uint32_t a) {
    return *reinterpret_cast<const uint32_t*>(Eb + a);
}
template <bool ESM>
__device__ __forceinline__ void stE(unsigned char* Eb, uint32_t a, uint32_t v) {
    *reinterpret_cast<uint32_t*>(Eb + a) = v;
}

// X = x + 191 in two 16-bit-lane words; cw = clamp(x + 63, 0, 126) packed per frame byte.
struct EdgeIn {
    uint32_t xlo, xhi, cw;
};

// e: E word (E + 127 per byte), tw: T word of the old message (192 + L_old per byte).
// Per byte X = e + (256 - T); as words e + sum_i (256 - T_i) 256^i = e - T + 0x01010100 (mod 2^32).
__device__ __forceinline__ EdgeIn edge_in(uint32_t e, uint32_t tw, const Konst& K) {
    EdgeIn r;
    // lanes {1,3}: e + 256 - T.  prmt(e, one) = hi16z(e) with byte 0 of K.one (0x01) in bytes 1, 3,
    // i.e. + 0x01000100, so the subtraction stays one IMAD (FMA pipe)
    r.xhi = imad(hi16z(tw), K.m1, prmt<0x4341u>(e, K.one));
#if QKD_EIN_FMA   // experiment: the three-term sum on the FMA pipe (2 IMAD instead of 1 IADD3)
    r.xlo = imadi<-256>(r.xhi, imad(tw, K.m1, imad(e, K.one, 0x01010100u)));
#else
    r.xlo = imadi<-256>(r.xhi, e - tw + 0x01010100u);    // lanes {0,2}: (e + S) - 256 * xhi
#endif
    const uint32_t clo = relu_min(r.xlo, K.b128, 0x007E007Eu);   // clamp(X - 128, 0, 126)
    const uint32_t chi = relu_min(r.xhi, K.b128, 0x007E007Eu);
    r.cw = pack16c(clo, chi, K);      // bytes in [0, 126]; bit 6 = (x >= 1) -- x = 0 counts as
    return r;                         // negative, which is immaterial (R23)
}
// The output sign of Eq.(1) for edge k at bit 7 of each byte: Q2 = 2 (Q & 0x40404040), Q = the row's
// sign product (bit 6, target bit included), cw = the edge's clamp word (sign of x at bit 6).  As an
// add, 2 (Q6 + cw): bit 6 of Q6 + cw is Q6 ^ cw (Q6 has no low bits, so nothing carries into bit 6),
// doubled it sits at bit 7; the carry out of a byte only sets bit 0 of the next (an even value + 1),
// never its bit 7.  One IMAD instead of an XOR and a shift.
__device__ __forceinline__ uint32_t sign_s7(uint32_t Q2, uint32_t cw) { return imadi<2>(cw, Q2); }
// check-node magnitude min(|x|, 63) (MSG_max = 63)
__device__ __forceinline__ uint32_t edge_mag(uint32_t cw, const Konst& K) { return __vabsdiffu4(cw, K.c63); }

// complement form 63 - min(|x|, 63) of the same magnitude (input of tau4c)
__device__ __forceinline__ uint32_t edge_magc(uint32_t cw, const Konst& K) {
    return (QKD_VIADD_MISC & 2) ? 0x3F3F3F3Fu - __vabsdiffu4(cw, K.c63) : imad(__vabsdiffu4(cw, K.c63), K.m1, 0x3F3F3F3Fu);
}

// The same value by a different instruction sequence (immediate operand, IADD3): ptxas cannot
// merge it with edge_magc, so the split kernel recomputes it instead of keeping it live.
__device__ __forceinline__ uint32_t edge_magc_alt(uint32_t cw) { return 0x3F3F3F3Fu - __vabsdiffu4(cw, 0x3F3F3F3Fu); }

// Emit for the split kernel, from the pre-layer E word ew and the old message word t_old only
// (no 16-bit X words kept from edge_in): with oc = 63 - o and M = 0xFF where L_new < 0,
//   T_new = 192 + L_new = ~(oc ^ (M & 0x7F)) + [L_new < 0]         (129 + oc or 255 - oc)
//   E_new'' = clamp(ew + T_new - T_old, 0, 254) = clamp(E + L_new - L_old, -127, 127) + 127,
// with d = T_new - T_old + 128 in [2, 254] per byte and the sum in 16-bit lanes; Algorithm 2
// keeps ew where |E| = 127.  Returns T_new.
__device__ __forceinline__ uint32_t edge_out_s(uint32_t oc, uint32_t s7, uint32_t t_old, uint32_t ew,
                                               const Konst& K, uint32_t& e_out) {
    const uint32_t M = bmask7(s7);                                // 0xFF where L_new < 0
    const uint32_t nx = lop3i<0x87, 0x7F7F7F7Fu>(oc, M);          // ~(oc ^ (M & 0x7F))
    const uint32_t sn = imad(lop3i<0xA0, 0x01010101u>(M, 0u), K.one, nx);   // + (M & 1)
    const uint32_t d = sn - t_old + 0x80808080u;                  // IADD3, exact per byte
    const uint32_t hi = imad(hi16z(ew), K.one, hi16z(d));         // lanes {1,3}: ew + d
    const uint32_t lo = imadi<-256>(hi, imad(ew, K.one, d));     // lanes {0,2}
    const uint32_t enew = pack16c(relu_min(lo, K.b128, 0x00FE00FEu), relu_min(hi, K.b128, 0x00FE00FEu), K);
    const uint32_t G = bmask7(QKD_MISC_ADD(__vabsdiffu4(ew, K.c127), 0x01010101u, 1));   // |E| == 127
    e_out = lop3<0xCA>(G, ew, enew);
    return sn;
}

// Given the leave-one-out magnitude o, the sign flag (bit 7 of s7 = 1 -> L_new < 0; sign_s7 below), the
// edge's X words and the pre-layer E word: returns the new S word (stored) and writes the new
// E word (Algorithm 2 guard on |E| = E_max, Eq.(9) saturated to +-127).
__device__ __forceinline__ uint32_t edge_out(uint32_t o, uint32_t s7, const EdgeIn& in, uint32_t ew,
                                             const Konst& K, uint32_t& e_out) {
    const uint32_t M = bmask7(s7);                                // 0xFF where L_new < 0
    const uint32_t om = o & M;
    const uint32_t Tb = imad(om, K.m2, imad(o, K.one, 0xC0C0C0C0u));   // bytes (64 + L_new) + 128
    const uint32_t thi = hi16s(Tb);                               // lanes {1,3}: 64 + L_new - 128
    const uint32_t tlo = imad(imad(thi, K.m256, Tb), K.one, 0xFFFFFF00u);   // lanes {0,2}, same
    // E + L_new - L_old = x + L_new: lanes relu(min(X + T - 128, 254)) = clamp(.., -127, 127) + 127
    const uint32_t enew = pack16c(relu_min(in.xlo, tlo, 0x00FE00FEu), relu_min(in.xhi, thi, 0x00FE00FEu), K);
    const uint32_t G = bmask7(QKD_MISC_ADD(__vabsdiffu4(ew, K.c127), 0x01010101u, 1));   // |E| == 127
    e_out = lop3<0xCA>(G, ew, enew);                              // G ? ew : enew
    return Tb;                                                    // 192 + L_new (stored as is)
}

// edge_out with the leave-one-out magnitude in complement form oc = 63 - o (tau4c output):
// o & M = (oc ^ 63) & M is still one LOP3 and o + 0xC0 = 0xFF - oc one IMAD, so nothing is added.
__device__ __forceinline__ uint32_t edge_out_c(uint32_t oc, uint32_t s7, const EdgeIn& in, uint32_t ew,
                                               const Konst& K, uint32_t& e_out) {
    const uint32_t M = bmask7(s7);                                // 0xFF where L_new < 0
    const uint32_t om = lop3i<0x48, 0x3F3F3F3Fu>(oc, M);          // (oc ^ 63) & M = o & M
    const uint32_t Tb = imadi<-2>(om, imad(oc, K.m1, 0xFFFFFFFFu));   // 255 - oc - 2 om = 192 + L_new
    const uint32_t thi = hi16s(Tb);                               // lanes {1,3}: L_new - 64
#ifndef QKD_TLO_IMAD   // the FMA-pipe form below measured 0.6% slower on C5a
    const uint32_t tlo = lo16s(Tb);                               // lanes {0,2}: L_new - 64
#else
    // lanes {0,2} on the FMA pipe: Tb + 0xFFFFFF00 - 256 thi = (b0 - 256, b2 - 256) for bytes with
    // bit 7 set (the identity edge_out uses)
    const uint32_t tlo = imadi<-256>(thi, imad(Tb, K.one, 0xFFFFFF00u));
#endif
    const uint32_t enew = pack16c(relu_min(in.xlo, tlo, 0x00FE00FEu), relu_min(in.xhi, thi, 0x00FE00FEu), K);
    const uint32_t G = bmask7(QKD_MISC_ADD(__vabsdiffu4(ew, K.c127), 0x01010101u, 1));   // |E| == 127
    e_out = lop3<0xCA>(G, ew, enew);
    return Tb;                                                    // 192 + L_new
}

__device__ __forceinline__ uint4 ld4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
// global 128-bit store / load kept in program order with the other volatile accesses of the row
// (the table reloads): ptxas otherwise sinks a row's message stores to its end, and with them the
// next row's prefetch loads, which may alias them as far as it knows
__device__ __forceinline__ void st4_pinned(uint32_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void ld4_pinned(const uint32_t* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
}
__device__ __forceinline__ void st4(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ uint32_t& w4(uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Message loads / stores.  With E in shared memory (ESM) the slot's messages (85 MB for C5a) are
// re-read from L2 every sweep: plain accesses.  With E in global memory (long frames, variants 7 / 8 /
// 4) the messages of the resident slots exceed L2 (C4: 148 x 1.3 MB) and would evict the E words
// every row gathers, so they stream with the evict-first (.cs) policy and E keeps L2.
#ifndef QKD_MSG_CS
#define QKD_MSG_CS 1
#endif
template <bool ESM>
__device__ __forceinline__ uint32_t ld_msg(const uint32_t* p) {
    if constexpr (!ESM && QKD_MSG_CS) return __ldcs(p);
    else return *p;
}
template <bool ESM>
__device__ __forceinline__ void st_msg(uint32_t* p, uint32_t v) {
    if constexpr (!ESM && QKD_MSG_CS) __stcs(p, v);
    else *p = v;
}

// ---- message layout (every variant but the lane-pair one) -----------------------------------
// Row r of a block row of degree D keeps its D message words in EMISSION order (word q = the
// q-th edge row_update emits, emit_pos below), interleaved by 32-row chunks: word q of row r at
// base + (r / 32) 32 D + 32 q + r % 32 (base = li.z words from the slot base).  A warp's access
// to one position is 128 contiguous bytes, a thread's words are at immediate offsets 128 q from
// one pointer, no padding word is ever moved (write traffic = the algorithmic bytes), a row's
// words are stored one by one as they are emitted (nothing buffered in registers for a vector
// store).  (Loading the next row's words early -- after this row's gather, late in its emit, or
// before the block-row barrier -- was measured slower on C5a, 57-61 vs 52.8 ms: every form keeps
// extra words live across code ptxas then schedules worse.)
__host__ __device__ constexpr int emit_pos(int D, int k) {    // emission step of edge k
    return k >= D / 2 ? 2 * (k - D / 2) : 2 * (D / 2 - 1 - k) + 1;
}
__host__ __device__ constexpr int emit_edge(int D, int p) {   // edge emitted at step p
    return (p & 1) ? D / 2 - 1 - (p >> 1) : D / 2 + (p >> 1);
}
// word 0 of row r (block row of degree D at word offset base); word q is at + 32 q
__device__ __forceinline__ uint32_t* msg_row(uint32_t* Lslot, int base, int D, int r) {
    return Lslot + base + (r >> 5) * 32 * D + (r & 31);
}
__device__ __forceinline__ uint32_t* msg_word(uint32_t* Lslot, int base, int D, int Z, int r, int q) {
    return msg_row(Lslot, base, D, r) + 32 * q;
}
// One check row r of a block row with D edges (layered update, Alg. 1/2).
//   et   : the row's D (cb, s) entries;  nib : target syndrome bits
//   FM   : 0 = `first_rt` read at run time, 1 = first sweep (compile time), 2 = not the first sweep.
//          On a group's first sweep all messages are L = 0 (R16) and are not loaded.
//   (A lane refilled alone has its bytes of the workspace reset to T = 192 when its frame is loaded.)
template <int D, bool ESM, bool POW2, int KEEP_ADDR_MAX, int FM>
__device__ __forceinline__ void row_update(const int2* __restrict__ et, int Z, uint32_t r4, uint32_t zm4,
                                           unsigned char* Eb, uint32_t* __restrict__ Lslot, int base, int r,
                                           uint32_t nib, bool first_rt, const Konst& K) {
    const bool first = FM == 1 || (FM == 0 && first_rt);
    // High degrees recompute each E address in the emit phase (one smem table load + IMAD + LOP3)
    // instead of holding D addresses in registers through the forward/backward passes.
    constexpr bool KEEP_ADDR = D <= KEEP_ADDR_MAX;
    // Degrees above 20 (the degree <= 32 kernel) keep only cw and the old message word per edge
    // between the gather and the emit (edge_out_s recomputes x from them): 2 registers per edge
    // instead of 3, so rows up to degree 32 stay in registers.
#ifndef QKD_LOWREG_MIN
#define QKD_LOWREG_MIN 21
#endif
#ifndef QKD_G8_LOWREG
#define QKD_G8_LOWREG 1   // variant 7 (E in global memory, degree <= 8) rows keep only cw + old message per edge
                          // (64 registers at 1024 threads without spills in the row loop)
#endif
    constexpr bool LOWREG = D >= QKD_LOWREG_MIN || (!ESM && D <= 8 && QKD_G8_LOWREG);
    uint32_t addr[D];
    EdgeIn in[D];
    uint32_t S[D];                                 // the row's message words, emission order
    uint32_t P = 0;
    const uint32_t* Lr = msg_row(Lslot, base, D, r);   // word q at Lr[32 q]
#pragma unroll
    for (int q = 0; q < D; ++q) S[q] = first ? 0xC0C0C0C0u : ld_msg<ESM>(Lr + 32 * q);
#pragma unroll
    for (int k = 0; k < D; ++k) addr[k] = Addr<POW2>::at(et[k], r4, zm4, Z, K);
#pragma unroll
    for (int q = 0; q < D; ++q) {      // gather in emission order
        const int k = emit_edge(D, q);
        in[k] = edge_in(ldE<ESM>(Eb, addr[k]), S[q], K);
        P ^= in[k].cw;
    }
    // Eq.(1) with the target bit: L_new of edge k is negative iff
    // s_i ^ XOR_{j != k} [x_j < 0] = s_i ^ ((D-1)&1) ^ P ^ nonneg_k   (bit 6)
    const uint32_t Q = P ^ nib_to_bit6(nib) ^ (((D - 1) & 1) ? 0x40404040u : 0u);
    const uint32_t Q2 = (Q & 0x40404040u) << 1;
    // an opaque GENERIC pointer: ptxas keeps generic stores in order with the row's shared-memory
    // E accesses (they might alias), which pins each message store at its edge's emit; through a
    // global pointer it sinks them all to the end of the row, holding D words in registers
    uint32_t* Lw;
    asm("mov.b64 %0, %1;" : "=l"(Lw) : "l"(msg_row(Lslot, base, D, r)));
    // emit edge k as soon as its leave-one-out magnitude is known (keeps the live set small); its
    // new message word goes straight to position q = emit_pos(D, k)
    auto emit = [&](int k, uint32_t o) {
        const int q = emit_pos(D, k);
        uint32_t a;
        if constexpr (KEEP_ADDR) {
            a = addr[k];
        } else {
            int2 e;   // volatile: force the reload so ptxas does not keep the table entry live
            asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"((uint32_t)__cvta_generic_to_shared(et + k)));
            a = Addr<POW2>::at(e, r4, zm4, Z, K);
        }
        const uint32_t ew = ldE<ESM>(Eb, a);
        uint32_t eo, tn;
        if constexpr (LOWREG) {
            tn = edge_out_s(o, sign_s7(Q2, in[k].cw), S[q], ew, K, eo);
        } else {
            tn = edge_out_c(o, sign_s7(Q2, in[k].cw), in[k], ew, K, eo);
        }
        stE<ESM>(Eb, a, eo);
        st_msg<ESM>(Lw + 32 * q, tn);
    };
    // magnitudes in complement form (tau4c / edge_magc / edge_out_c): two instructions fewer per tau
#define QKD_TAU tau4c
#define QKD_MAG edge_magc
#define QKD_O63 0u
    if constexpr (D == 1) {
        emit(0, QKD_O63);                           // empty box-plus -> MSG_max (R6)
    } else if constexpr (D == 2) {
        emit(1, QKD_MAG(in[0].cw, K));
        emit(0, QKD_MAG(in[1].cw, K));
    } else {
        // Leave-one-out by the forward/backward schedule of R6, evaluated meet-in-the-middle: the
        // forward chain over edges [0, H) and the backward chain over [H, D) run concurrently, then
        // each continues across the other half while emitting outputs.  Every tau has exactly the
        // arguments of the plain F/B schedule (F_k = tau(F_{k-1}, m_k), B_k = tau(m_k, B_{k+1}),
        // o_k = tau(F_{k-1}, B_{k+1})), so results are identical; two independent chains double the ILP.
        constexpr int H = D / 2;
        uint32_t F[H], B[D];                        // F_0..F_{H-1}; B_H..B_{D-1}
        F[0] = QKD_MAG(in[0].cw, K);
        B[D - 1] = QKD_MAG(in[D - 1].cw, K);
#pragma unroll
        for (int j = 1; j < D; ++j) {               // phase 1: both chains, interleaved
            if (j <= H - 1) F[j] = QKD_TAU(F[j - 1], QKD_MAG(in[j].cw, K), K);
            const int kb = D - 1 - j;
            if (kb >= H) B[kb] = QKD_TAU(QKD_MAG(in[kb].cw, K), B[kb + 1], K);
        }
        uint32_t f = F[H - 1], b = B[H];
#pragma unroll
        for (int j = 0; j < D; ++j) {               // phase 2: continue across, emitting (steps 2j, 2j+1)
            const int kf = H + j;                   // forward: o_kf = tau(F_{kf-1}, B_{kf+1})
            if (kf <= D - 2) {
                emit(kf, QKD_TAU(f, B[kf + 1], K));
                f = QKD_TAU(f, QKD_MAG(in[kf].cw, K), K);
            } else if (kf == D - 1) {
                emit(D - 1, f);                     // o_{D-1} = F_{D-2}
            }
            const int kb = H - 1 - j;               // backward: o_kb = tau(F_{kb-1}, B_{kb+1})
            if (kb >= 1) {
                emit(kb, QKD_TAU(F[kb - 1], b, K));
                b = QKD_TAU(QKD_MAG(in[kb].cw, K), b, K);
            } else if (kb == 0) {
                emit(0, b);                         // o_0 = B_1
            }
        }
    }
#undef QKD_TAU
#undef QKD_MAG
#undef QKD_O63
}

// ---------------------------------------------------------------------------------------------
// Split row: the D edges of check row r are shared by a lane pair (lanes 2i, 2i+1 of one warp),
// which halves the per-thread state so a CTA can run 1024 threads (32 warps per SM).
//   side A (even lane): edges k = 0 .. HA-1, local j = k            HA = D / 2
//   side B (odd lane):  edges k = D-1 .. HA,  local j = D-1-k        HB = D - HA
// Each side first runs one chain of the forward/backward schedule of R6 over its own edges
// (A: F_0..F_{HA-1}, B: B_{D-1}..B_{HA}; tau is symmetric), the two boundary values cross once
// by shuffle, and each side then continues the other chain across its own edges, emitting
// o_k = tau(F_{k-1}, B_{k+1}) -- every tau has the arguments of the plain schedule, so results
// are identical.  The sign product of Eq.(1) is the XOR of both halves (one more shuffle).
// Messages: a lane owns words [side*WA, side*WA + n) of the row (WA = roundup2(HA)) and moves
// them with 64-bit loads/stores.  Magnitudes run in complement form (tau4c).
//   et2 : 2*HB table entries, [2j + side] = the lane's j-th edge (side A's empty slot of an odd
//         degree repeats side B's entry so its load stays in bounds; its results are unused).
// All 32 lanes of the warp call this (the shuffles need them); `act` = the row exists.
template <int D, bool POW2>
__device__ __forceinline__ void row_update_split(const int2* __restrict__ et2, int Z, uint32_t r4, uint32_t zm4,
                                                 unsigned char* Eb, uint32_t* __restrict__ Lh, uint32_t nib,
                                                 bool first, bool act, int side, const Konst& K) {
    constexpr int HA = D / 2, HB = D - HA, NW = (HB + 1) / 2;
    const int n = side ? HB : HA;
    uint2 S[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        if (first || !act || 2 * w >= n) S[w] = make_uint2(0xC0C0C0C0u, 0xC0C0C0C0u);   // L = 0
        else S[w] = *reinterpret_cast<const uint2*>(Lh + 2 * w);
    }
    auto sw = [&](int j) -> uint32_t& { return (j & 1) ? S[j >> 1].y : S[j >> 1].x; };
    // E address of local edge j: the table entry is re-read (volatile) at both uses, so ptxas
    // neither keeps HB addresses live nor hoists the loop-invariant entries and spills them
    auto addr = [&](int j) -> uint32_t {
        int2 e;
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y)
                     : "r"((uint32_t)__cvta_generic_to_shared(et2 + 2 * j + side)));
        return Addr<POW2>::at(e, r4, zm4, Z, K);
    };
    uint32_t cw[HB];
    uint32_t P = 0;
#pragma unroll
    for (int j = 0; j < HB; ++j) {
        cw[j] = edge_in(ldE<true>(Eb, addr(j)), sw(j), K).cw;
        if (HA == HB || j < n) P ^= cw[j];
    }
    P ^= __shfl_xor_sync(0xffffffffu, P, 1);
    const uint32_t Q = P ^ nib_to_bit6(nib) ^ (((D - 1) & 1) ? 0x40404040u : 0u);
    auto emit = [&](int j, uint32_t oc) {
        const uint32_t aj = addr(j);
        const uint32_t ew = ldE<true>(Eb, aj);        // pre-layer E (no other row of the layer touches it)
        uint32_t eo;
        const uint32_t sn = edge_out_s(oc, sign_s7((Q & 0x40404040u) << 1, cw[j]), sw(j), ew, K, eo);
        sw(j) = sn;
        if (act) {
            stE<true>(Eb, aj, eo);
            if ((j & 1) == 0) *reinterpret_cast<uint2*>(Lh + j) = S[j >> 1];   // j+1 was emitted before j
        }
    };
    if constexpr (D == 1) {
        if (side) emit(0, 0u);                      // empty box-plus -> MSG_max = 63 (R6)
    } else {
        uint32_t ch[HB];
        ch[0] = edge_magc(cw[0], K);
#pragma unroll
        for (int j = 1; j < HB; ++j)
            if (HA == HB || j < n) ch[j] = tau4c(ch[j - 1], edge_magc(cw[j], K), K);
        const uint32_t send = (HA == HB || side) ? ch[HB - 1] : ch[HA - 1];
        uint32_t acc = __shfl_xor_sync(0xffffffffu, send, 1);   // A: B_HA, B: F_{HA-1}
#pragma unroll
        for (int j = HB - 1; j >= 1; --j) {
            if (HA == HB || j < n) {
                const uint32_t o = tau4c(ch[j - 1], acc, K);       // o_k = tau(F_{k-1}, B_{k+1})
                acc = tau4c(edge_magc_alt(cw[j]), acc, K);         // continue the other chain
                emit(j, o);
            }
        }
        emit(0, acc);                                          // A: o_0 = B_1, B: o_{D-1} = F_{D-2}
    }
}

// Stopping criterion for one check row: bit 7 of the result is set in lane f iff the row's
// parity of hard decisions differs from the target bit.  Hard decision = (E < 0) = NOT bit 7 of
// (E'' + 1), so the parity of the d decisions is bit 7 of XOR(E''_k + 1) ^ (d odd ? 0x80 : 0).
template <int D, bool POW2>
__device__ __forceinline__ uint32_t syndrome_row(const int2* __restrict__ et, int Z, uint32_t r4, uint32_t zm4,
                                                 const unsigned char* Eb, uint32_t nib, const Konst& K) {
    uint32_t e[D];
#pragma unroll
    for (int k = 0; k < D; ++k) e[k] = ldE<true>(Eb, Addr<POW2>::at(et[k], r4, zm4, Z, K));
    uint32_t acc = nib_to_bit7(nib) ^ ((D & 1) ? 0x80808080u : 0u);
#pragma unroll
    for (int k = 0; k < D; ++k) acc ^= imad(e[k], K.one, 0x01010101u);
    return acc;
}

// Runtime-degree variant (any degree <= 64), same arithmetic; state in local memory.
template <bool ESM>
__device__ __noinline__ void row_update_generic(const int2* __restrict__ et, int D, int Z, uint32_t r4,
                                                unsigned char* Eb, uint32_t* __restrict__ Lslot, int base, int r,
                                                uint32_t nib, bool first, const Konst K) {
    uint32_t addr[64], S[64], F[64], o[64];
    uint32_t* wp[64];
    EdgeIn in[64];
    uint32_t P = 0;
    for (int k = 0; k < D; ++k) {
        addr[k] = Addr<false>::at(et[k], r4, 0u, Z, K);
        wp[k] = msg_word(Lslot, base, D, Z, r, emit_pos(D, k));   // same layout as row_update
        S[k] = first ? 0xC0C0C0C0u : *wp[k];
        in[k] = edge_in(ldE<ESM>(Eb, addr[k]), S[k], K);
        P ^= in[k].cw;
    }
    const uint32_t Q = P ^ nib_to_bit6(nib) ^ (((D - 1) & 1) ? 0x40404040u : 0u);
    if (D == 1) {
        o[0] = 0x3F3F3F3Fu;
    } else if (D == 2) {
        o[0] = edge_mag(in[1].cw, K);
        o[1] = edge_mag(in[0].cw, K);
    } else {
        F[0] = edge_mag(in[0].cw, K);
        for (int k = 1; k <= D - 2; ++k) F[k] = tau4(F[k - 1], edge_mag(in[k].cw, K), K);
        uint32_t B = edge_mag(in[D - 1].cw, K);
        o[D - 1] = F[D - 2];
        for (int k = D - 2; k >= 1; --k) {
            o[k] = tau4(F[k - 1], B, K);
            B = tau4(edge_mag(in[k].cw, K), B, K);
        }
        o[0] = B;
    }
    for (int k = 0; k < D; ++k) {
        const uint32_t ew = ldE<ESM>(Eb, addr[k]);
        uint32_t eo;
        *wp[k] = edge_out(o[k], sign_s7((Q & 0x40404040u) << 1, in[k].cw), in[k], ew, K, eo);
        stE<ESM>(Eb, addr[k], eo);
    }
}

}  // namespace qkd
