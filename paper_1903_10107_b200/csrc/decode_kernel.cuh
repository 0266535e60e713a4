// decode_kernel.cuh -- the layered decode kernel template (persistent CTAs; each "slot" of TG threads,
// with its own named barrier, decodes frame groups of 4 frames taken from an atomic work counter).
// Included by the decode_inst_*.cu translation units, which instantiate the variants that
// qkd_ldpc.cu's kernel_of() launches (split across units so they compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "decode.cuh"

namespace qkd {

// QKD_MUTATE_NOBAR (race-check mutation builds only): drop the barrier between block rows, so the
// race check must report the resulting stale reads (tools/racecheck.sh)
#ifdef QKD_MUTATE_NOBAR
#define QKD_MUTATE_BAR(x)
#else
#define QKD_MUTATE_BAR(x) x
#endif

// the slot's named barrier; with one slot per CTA (e.g. C5a) the id is the immediate 1, so no
// register holds it across the row updates (it was spilled and reloaded before every barrier)
__device__ __forceinline__ void slot_bar(const DecParams& p, int bar) {
    if (p.GPC == 1)
        asm volatile("bar.sync 1, %0;" ::"r"(p.TG) : "memory");
    else
        group_bar(bar, p.TG);
}

#ifdef QKD_RACECHECK
// Layer-order race check (debug builds: tools/racecheck.sh; compute-sanitizer is closed on this GPU
// pool).  Layers of a slot are numbered lc = 1, 2, ... across sweeps and groups; the row update of
// layer lc stamps every E word it writes with lc, and before it reads an E word it checks the stamp:
// the previous writer of that column is the layer delta back (delta = distance to the previous block
// row holding the same block column, precomputed per base edge), so the stamp must be exactly
// lc - delta -- smaller means a stale read (the writer's update was not yet visible: a missing or
// misplaced barrier), larger means a layer ran ahead.  Writers from before the slot's current group
// (lc - delta < lc0, the group's first layer) are only checked for "not from the future".
static __device__ __noinline__ void rc_row(const DecParams& p, long long gslot, int4 li, int r, int lc, int lc0, bool write) {
    unsigned* st = p.dbg + 16 + gslot * (long long)p.n;
    for (int k = 0; k < li.x; ++k) {
        const int2 e = p.edge[li.y + k];
        int idx = r + e.y;
        idx = idx >= p.Z ? idx - p.Z : idx;
        const int j = e.x + idx;
        if (write) {
            st[j] = (unsigned)lc;
            continue;
        }
        const int want = lc - p.dbg_delta[li.y + k];
        const int got = (int)st[j];
        const bool bad = want >= lc0 ? got != want : got >= lc0;
        if (bad && atomicAdd(p.dbg, 1u) == 0u) {
            p.dbg[1] = (unsigned)lc; p.dbg[2] = (unsigned)r; p.dbg[3] = (unsigned)(li.y + k);
            p.dbg[4] = (unsigned)got; p.dbg[5] = (unsigned)want; p.dbg[6] = (unsigned)gslot;
        }
    }
    if (write) __threadfence_block();
}
#define QKD_RC(write) rc_row(p, rc_gslot, li, r, rc_lc, rc_lc0, write)
#else
#define QKD_RC(write)
#endif

// One layer (block row) of the slot's rows.  rc_*: layer-order race check (QKD_RACECHECK builds).
template <int DMAX, bool ESM, bool POW2, bool SPLIT, int FM = 0>
__device__ __forceinline__ void layer_pass(const DecParams& p, const int4 li, const int2* et, int t,
                                           unsigned char* Eb, uint32_t* Lslot, const uint8_t* synI, uint32_t fresh,
                                           const Konst& K, int rc_lc = 0, int rc_lc0 = 0, long long rc_gslot = 0) {
    const bool first = fresh == 0xFu;   // all four lanes on their first sweep: L = 0 without loading
    const uint32_t zm4 = 4u * (uint32_t)p.Z - 1u;
    if (li.x == 0) return;              // a check row with no variables: nothing to update (oracle: no-op)
    if constexpr (SPLIT) {
        // lane pairs: warp-uniform trip count (the shuffles need all 32 lanes), 16 rows per warp pass
        const int side = t & 1, pairs = p.TG >> 1, wa = ((li.x >> 1) + 1) & ~1;
        switch (li.x) {
#define QKD_SCASE2(DD)                                                                                   \
    case DD:                                                                                             \
        for (int rb = (t >> 1) & ~15; rb < p.Z; rb += pairs) {                                           \
            const int r0 = rb + ((t >> 1) & 15);                                                         \
            const bool act = r0 < p.Z;                                                                   \
            const int r = act ? r0 : p.Z - 1;                                                            \
            row_update_split<DD, POW2>(et, p.Z, 4u * r, zm4, Eb, Lslot + li.z + r * li.w + side * wa, synI[r], \
                                       first, act, side, K);                                            \
        }                                                                                                \
        return;
            QKD_SCASE2(1) QKD_SCASE2(2) QKD_SCASE2(3) QKD_SCASE2(4) QKD_SCASE2(5) QKD_SCASE2(6)
            QKD_SCASE2(7) QKD_SCASE2(8) QKD_SCASE2(9) QKD_SCASE2(10) QKD_SCASE2(11) QKD_SCASE2(12)
            QKD_SCASE2(13) QKD_SCASE2(14) QKD_SCASE2(15) QKD_SCASE2(16) QKD_SCASE2(17) QKD_SCASE2(18)
            QKD_SCASE2(19) QKD_SCASE2(20)
#undef QKD_SCASE2
            default:
                break;
        }
        __trap();
    } else if constexpr (DMAX > 0) {
        switch (li.x) {
#define QKD_CASE(DD)                                                                                     \
    case DD:                                                                                             \
        if constexpr (DD <= DMAX) {                                                                      \
            for (int r = t; r < p.Z; r += p.TG) {                                                        \
                QKD_RC(false);                                                                           \
                row_update<DD, ESM, POW2, (DMAX <= 8 ? 4 : QKD_KEEP_ADDR), FM>(et, p.Z, 4u * r, zm4, Eb, Lslot,   \
                                                                               li.z, r, synI[r], first, K);     \
                QKD_RC(true);                                                                            \
            }                                                                                            \
            return;                                                                                      \
        }                                                                                                \
        break;
            QKD_CASE(1) QKD_CASE(2) QKD_CASE(3) QKD_CASE(4) QKD_CASE(5) QKD_CASE(6) QKD_CASE(7)
            QKD_CASE(8) QKD_CASE(9) QKD_CASE(10) QKD_CASE(11) QKD_CASE(12) QKD_CASE(13)
            QKD_CASE(14) QKD_CASE(15) QKD_CASE(16) QKD_CASE(17) QKD_CASE(18) QKD_CASE(19)
            QKD_CASE(20) QKD_CASE(21) QKD_CASE(22) QKD_CASE(23) QKD_CASE(24) QKD_CASE(25) QKD_CASE(26)
            QKD_CASE(27) QKD_CASE(28) QKD_CASE(29) QKD_CASE(30) QKD_CASE(31) QKD_CASE(32)
#undef QKD_CASE
            default:
                break;
        }
        __trap();   // the host never selects a DMAX kernel for a code with a larger degree
    } else {
        for (int r = t; r < p.Z; r += p.TG) {
            QKD_RC(false);
            row_update_generic<ESM>(et, li.x, p.Z, 4u * r, Eb, Lslot, li.z, r, synI[r], first, K);
            QKD_RC(true);
        }
    }
}
#undef QKD_RC

// per-lane syndrome violation mask (bit f set = frame f violates some parity check),
// group-uniform, exact for the lanes in `active`.  Hard decision bit = (E < 0) = NOT bit 7 of
// (E'' + 1), E'' = E + 127 (R9).  A warp whose own rows already show a violation in every
// active lane stops early: the group's answer for those lanes ("not yet") cannot change.

template <int DMAX, bool ESM, bool POW2>
__device__ __forceinline__ uint32_t syndrome_viol(const DecParams& p, const int4* s_layer, const int2* s_edge,
                                                  const unsigned char* Eb, const uint8_t* sSyn, int t,
                                                  uint32_t* flags, int& chk, int bar, const Konst& K,
                                                  uint32_t active) {
    const uint32_t zm4 = 4u * (uint32_t)p.Z - 1u;
    const uint32_t act7 = nib_to_bit7(active);
    uint32_t v = 0;
    for (int I = 0; I < p.Mb; ++I) {
        if (I > 0 && (__reduce_or_sync(0xffffffffu, v & 0x80808080u) & act7) == act7) break;
        const int4 li = s_layer[I];
        const int2* et = s_edge + li.y;
        const uint8_t* synI = sSyn + I * p.Z;
        bool done = false;
        if constexpr (DMAX > 0 && ESM) {
            switch (li.x) {
#define QKD_SCASE(DD)                                                                                  \
    case DD:                                                                                           \
        if constexpr (DD <= DMAX) {                                                                    \
            for (int r = t; r < p.Z; r += p.TG) v |= syndrome_row<DD, POW2>(et, p.Z, 4u * r, zm4, Eb, synI[r], K); \
            done = true;                                                                               \
        }                                                                                              \
        break;
                QKD_SCASE(1) QKD_SCASE(2) QKD_SCASE(3) QKD_SCASE(4) QKD_SCASE(5) QKD_SCASE(6) QKD_SCASE(7)
                QKD_SCASE(8) QKD_SCASE(9) QKD_SCASE(10) QKD_SCASE(11) QKD_SCASE(12) QKD_SCASE(13)
                QKD_SCASE(14) QKD_SCASE(15) QKD_SCASE(16) QKD_SCASE(17) QKD_SCASE(18) QKD_SCASE(19)
                QKD_SCASE(20)
#undef QKD_SCASE
                default:
                    break;
            }
        }
        if (!done) {
            const uint32_t par = (li.x & 1) ? 0x80808080u : 0u;
            for (int r = t; r < p.Z; r += p.TG) {
                uint32_t acc = nib_to_bit7(synI[r]) ^ par;
                for (int k = 0; k < li.x; ++k)
                    acc ^= imad(ldE<ESM>(Eb, Addr<POW2>::at(et[k], 4u * r, zm4, p.Z, K)), K.one, 0x01010101u);
                v |= acc;
            }
        }
    }
    v &= 0x80808080u;
    v = __reduce_or_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicOr(&flags[chk & 1], v);
    slot_bar(p, bar);
    const uint32_t res = *(volatile uint32_t*)&flags[chk & 1];
    if (t == 0) flags[(chk + 1) & 1] = 0;   // next check's flag: last read before this barrier
    ++chk;
    return ((res >> 7) & 1u) | ((res >> 14) & 2u) | ((res >> 21) & 4u) | ((res >> 28) & 8u);
}

// write the outputs of the lanes in `mask` (state at their stopping iteration)
static __device__ void finalize(const DecParams& p, const int4* s_layer, const uint32_t* Eslot, const uint32_t* Lslot,
                         const long long* fr, uint32_t mask, const int* itv, uint32_t succ_mask, uint32_t fresh, int t) {
    const int lane = threadIdx.x & 31;
    for (int f = 0; f < kFramesPerGroup; ++f) {
        if (!((mask >> f) & 1u)) continue;
        const long long frame = fr[f];
        const int it = itv[f];
        const bool first = (fresh >> f) & 1u;
        uint8_t* brow = p.bits + frame * p.nb8;
        for (int jw = t & ~31; jw < p.n; jw += p.TG) {
            const int j = jw + lane;
            const bool b = j < p.n && !(((Eslot[j < p.n ? j : 0] + 0x01010101u) >> (8 * f + 7)) & 1u);
            const uint32_t bal = __ballot_sync(0xffffffffu, b);
            const int byte = (jw >> 3) + lane;
            if (lane < 4 && byte < p.nb8) brow[byte] = (uint8_t)(bal >> (8 * lane));
        }
        if (p.fE) {
            int8_t* erow = p.fE + frame * p.n;
            for (int j = t; j < p.n; j += p.TG) erow[j] = (int8_t)((int)((Eslot[j] >> (8 * f)) & 0xFFu) - 127);
        }
        if (p.fL) {
            int8_t* lrow = p.fL + frame * p.n_edges;
            for (int I = 0; I < p.Mb; ++I) {
                const int4 li = s_layer[I];
                const int cnt = li.x * p.Z;
                for (int q = t; q < cnt; q += p.TG) {
                    const int k = q / p.Z, r = q - k * p.Z;
                    const long long e = (long long)(li.y + k) * p.Z + r;     // canonical edge order
                    const uint32_t* wp;   // word of canonical edge k (split: side A, then side B)
                    if (p.soff) {
                        const int ha = li.x >> 1;
                        wp = Lslot + li.z + r * li.w + (k < ha ? k : ((ha + 1) & ~1) + (li.x - 1 - k));
                    } else {
                        wp = msg_word(const_cast<uint32_t*>(Lslot), li.z, li.x, p.Z, r, emit_pos(li.x, k));
                    }
                    lrow[e] = first ? (int8_t)0 : (int8_t)((int)((*wp >> (8 * f)) & 0xFFu) - 192);
                }
            }
        }
        if (t == 0) {
            const int s = (succ_mask >> f) & 1;
            p.iters[frame] = it;
            p.success[frame] = (uint8_t)s;
            if (p.counters) {
                atomicAdd(p.counters + 0, 1ull);
                atomicAdd(p.counters + 1, (unsigned long long)s);
                atomicAdd(p.counters + 4, (unsigned long long)it);
            }
        }
    }
}

template <int DMAX, bool ESM, bool POW2, bool SPLIT, bool REFILL>
__global__ void __launch_bounds__(SPLIT ? 1024 : (DMAX == 8 && ESM) ? QKD_V1_THREADS : (DMAX == 8 && !ESM ? QKD_G8_THREADS : (DMAX == 32 && !ESM ? QKD_G32_THREADS : (DMAX == 20 || DMAX == 32 || DMAX == 8 ? QKD_D32_TG(DMAX) : 256))), 1)
    decode_kernel(const DecParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Konst K = p.K.in_regs();
    // frames of this launch: the host count, or a device-resident count (interactive rounds compact
    // the still-failed frames on the device, qkd_reconcile_adaptive; the grid is planned for p.F)
    const long long nF = p.F_dev ? *p.F_dev : p.F;
    const long long ngroups = (nF + kFramesPerGroup - 1) / kFramesPerGroup;
    // tables: layer info, then one edge table per slot with the slot's E base folded in
    int4* s_layer = reinterpret_cast<int4*>(smem + p.tab_off);
    int2* s_edges = reinterpret_cast<int2*>(s_layer + p.Mb);
    int2* s_split = s_edges + p.GPC * p.nbase;   // [GPC][nsplit] lane-pair order (SPLIT only)
    int* s_soff = reinterpret_cast<int*>(s_split + (SPLIT ? p.GPC * p.nsplit : 0));   // [Mb] (SPLIT only)
    for (int i = threadIdx.x; i < p.Mb; i += blockDim.x) {
        s_layer[i] = p.layer[i];
        if (SPLIT) s_soff[i] = p.soff[i];
    }
    for (int i = threadIdx.x; i < p.GPC * p.nbase; i += blockDim.x) {
        const int sl = i / p.nbase;
        const int2 e = p.edge[i - sl * p.nbase];
        s_edges[i] = POW2 ? make_int2((ESM ? sl * p.slot_bytes : 0) + 4 * e.x, 4 * e.y) : e;   // global E: per-slot base pointer
    }
    if constexpr (SPLIT) {
        for (int I = 0; I < p.Mb; ++I) {
            const int4 li = p.layer[I];
            const int ha = li.x >> 1, hb = li.x - ha;
            for (int i = threadIdx.x; i < p.GPC * 2 * hb; i += blockDim.x) {
                const int sl = i / (2 * hb), q = i - sl * 2 * hb, j = q >> 1, side = q & 1;
                const int k = (side || j >= ha) ? li.x - 1 - j : j;
                const int2 e = p.edge[li.y + k];
                s_split[sl * p.nsplit + p.soff[I] + q] = POW2 ? make_int2(sl * p.slot_bytes + 4 * e.x, 4 * e.y) : e;
            }
        }
    }
    __syncthreads();

    const int slot = threadIdx.x / p.TG;
    const int t = threadIdx.x - slot * p.TG;
    const int bar = 1 + slot;
    const int2* s_edge = s_edges + slot * p.nbase;
    const int2* s_edge2 = s_split + slot * p.nsplit;
    unsigned char* sbase = smem + (size_t)slot * p.slot_bytes;
    const long long gslot = (long long)blockIdx.x * p.GPC + slot;
    uint32_t* Eslot = ESM ? reinterpret_cast<uint32_t*>(sbase) : p.Ews + gslot * (long long)p.n;
    unsigned char* Eb = ESM ? (POW2 ? smem : sbase) : reinterpret_cast<unsigned char*>(Eslot);
    uint8_t* sSyn = sbase + p.e_bytes;
    int* ctl = reinterpret_cast<int*>(sSyn + ((p.m + 15) & ~15));   // [0] group id, [1..2] flags
    uint32_t* flags = reinterpret_cast<uint32_t*>(ctl + 1);
    uint32_t* Lslot = p.Lws + gslot * p.ws_words;
    int rc_lc = 0, rc_lc0 = 1;   // layer counters of the race check (QKD_RACECHECK builds; otherwise unused)

    if constexpr (!SPLIT && REFILL) {
        // ---- per-frame scheduling: a lane whose frame stops is refilled with the next frame at
        // once (frames are taken one at a time from p.work), so a slot never waits for the
        // slowest of its 4 frames.  Lanes never interact, so every frame's result is the same as
        // in a fresh group.
        // per-lane frame ids and start sweeps live in shared memory (written by thread 0 before a
        // barrier): registers stay with the row updates
        int* s_fr = ctl + 4;        // [4] frame id per lane (-1: none; frames < 2^31, p.work is an int)
        int* s_start = ctl + 8;     // [4] this slot's sweep count when the lane's frame was loaded
        uint32_t active = 0, fresh = 0;
        int chk = 0, sweeps = 0;
        auto lane_state = [&](long long* fr, int* itv) {
            for (int f = 0; f < 4; ++f) {
                fr[f] = s_fr[f];
                itv[f] = sweeps - s_start[f];
            }
        };
        // take up to popc(mask) new frames into the lanes of `mask`; returns the lanes that got one
        auto refill_lanes = [&](uint32_t mask) -> uint32_t {
            const int k = __popc(mask);
            if (t == 0) ctl[0] = atomicAdd(p.work, k);
            slot_bar(p, bar);
            const long long a = *(volatile int*)&ctl[0];
            long long fid[4];
            uint32_t got = 0;
            int q = 0;
            for (int f = 0; f < 4; ++f) {
                fid[f] = -1;
                if (!((mask >> f) & 1u)) continue;
                const long long v = a + q++;
                if (v < nF) { fid[f] = v; got |= 1u << f; }
            }
            if (t == 0)
                for (int f = 0; f < 4; ++f)
                    if ((mask >> f) & 1u) { s_fr[f] = (int)fid[f]; s_start[f] = sweeps; }
            if (got == 0xFu && p.vec_llr) {
                // all four lanes, frames a..a+3: 32-bit loads transposed into frame-interleaved
                // words (E + 127 = (llr ^ 0x80) - 1), and the messages reset by plain stores
                const long long f0 = fid[0];
                const int n4 = p.n >> 2;
                for (int q = t; q < n4; q += p.TG) {
                    uint32_t r[4];
#pragma unroll
                    for (int f = 0; f < 4; ++f) r[f] = __ldcs(reinterpret_cast<const uint32_t*>(p.llr + (f0 + f) * p.n) + q);
                    const uint32_t pa = prmt<0x5140u>(r[0], r[1]), pb = prmt<0x5140u>(r[2], r[3]);
                    const uint32_t pc = prmt<0x7362u>(r[0], r[1]), pd = prmt<0x7362u>(r[2], r[3]);
                    Eslot[4 * q + 0] = (prmt<0x5410u>(pa, pb) ^ 0x80808080u) - 0x01010101u;
                    Eslot[4 * q + 1] = (prmt<0x7632u>(pa, pb) ^ 0x80808080u) - 0x01010101u;
                    Eslot[4 * q + 2] = (prmt<0x5410u>(pc, pd) ^ 0x80808080u) - 0x01010101u;
                    Eslot[4 * q + 3] = (prmt<0x7632u>(pc, pd) ^ 0x80808080u) - 0x01010101u;
                }
                // no message reset: the next sweep is every lane's first (fresh == 0xF) and uses L = 0
            } else if (got) {
                unsigned char* E8 = reinterpret_cast<unsigned char*>(Eslot);
#pragma unroll 4
                for (int j = t; j < p.n; j += p.TG) {          // E byte lane f <- LLR (stored as E + 127)
#pragma unroll
                    for (int f = 0; f < 4; ++f)
                        if ((got >> f) & 1u) E8[4 * j + f] = (uint8_t)(((uint8_t)p.llr[fid[f] * p.n + j] ^ 0x80u) - 1u);
                }
                const uint32_t Mg = fresh_mask(got);           // this slot's messages of those lanes: L = 0
                long long w = t;
                for (; w + 7LL * p.TG < p.ws_words; w += 8LL * p.TG) {   // 8 independent loads in flight
                    uint32_t v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = Lslot[w + (long long)u * p.TG];
#pragma unroll
                    for (int u = 0; u < 8; ++u) Lslot[w + (long long)u * p.TG] = lop3<0xB8>(v[u], Mg, 0xC0C0C0C0u);
                }
                for (; w < p.ws_words; w += p.TG) Lslot[w] = lop3<0xB8>(Lslot[w], Mg, 0xC0C0C0C0u);
            }
            if (got) {
                for (int i = t; i < p.m; i += p.TG) {          // syndrome nibble bit f (bits 4-7 kept 0:
                    uint32_t b = sSyn[i] & 0xFu;               // nib_to_bit6/7 multiply the whole byte)
#pragma unroll
                    for (int f = 0; f < 4; ++f)
                        if ((got >> f) & 1u)
                            b = (b & ~(1u << f)) | (((uint32_t)(p.syn[fid[f] * p.mb8 + (i >> 3)] >> (i & 7)) & 1u) << f);
                    sSyn[i] = (uint8_t)b;
                }
            }
            slot_bar(p, bar);
            return got;
        };
        auto finish = [&](uint32_t mask, uint32_t succ, uint32_t zeroL) {
            long long fr[4];
            int itv[4];
            lane_state(fr, itv);
            finalize(p, s_layer, Eslot, Lslot, fr, mask, itv, succ, zeroL, t);
            slot_bar(p, bar);
        };
        if (t == 0) { flags[0] = 0; flags[1] = 0; }
        uint32_t pend = refill_lanes(0xFu);
        active = fresh = pend;
        if (!p.early_stop) pend = 0;
        while (active) {
            while (pend) {   // iteration-0 check of newly loaded frames (R10)
                const uint32_t viol = syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, pend);
                const uint32_t done0 = pend & ~viol;
                pend = 0;
                if (done0) {
                    finish(done0, done0, done0);
                    active &= ~done0;
                    const uint32_t got = refill_lanes(done0);
                    active |= got;
                    fresh |= got;
                    pend = got;
                }
            }
            uint32_t cap = 0;   // lanes out of sweeps stop with their state after sweep T (R12)
            for (int f = 0; f < 4; ++f)
                if (((active >> f) & 1u) && sweeps - s_start[f] >= p.T) cap |= 1u << f;
            if (cap) {
                // early_stop: failure; otherwise success = syndrome matched after sweep T
                const uint32_t succ = p.early_stop ? 0u
                    : cap & ~syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, cap);
                finish(cap, succ, fresh & cap);
                active &= ~cap;
                fresh &= ~cap;
                const uint32_t got = refill_lanes(cap);
                active |= got;
                fresh |= got;
                pend = p.early_stop ? got : 0u;
                continue;
            }
            if (!active) break;
            for (int I = 0; I < p.Mb; ++I) {   // idle lanes (no frame left) compute harmlessly
                const int4 li = s_layer[I];
                layer_pass<DMAX, ESM, POW2, SPLIT>(p, li, s_edge + li.y, t, Eb, Lslot, sSyn + I * p.Z,
                                                   fresh == 0xFu ? 0xFu : 0u, K, ++rc_lc, rc_lc0, gslot);
                slot_bar(p, bar);
            }
            ++sweeps;
            fresh = 0;
            if (!p.early_stop) continue;
            const uint32_t viol = syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, active);
            const uint32_t done = active & ~viol;
            if (done) {
                finish(done, done, 0u);
                active &= ~done;
                const uint32_t got = refill_lanes(done);
                active |= got;
                fresh |= got;
                pend = got;
            }
        }
    } else {
    for (;;) {   // whole 4-frame groups: a slot takes the next 4 frames when all of its lanes stop
        if (t == 0) ctl[0] = atomicAdd(p.work, 1);
        slot_bar(p, bar);
        const long long g = *(volatile int*)&ctl[0];
        if (g >= ngroups) break;
        rc_lc0 = rc_lc + 1;   // the group's first layer (race check)
        const long long f0 = g * kFramesPerGroup;
        const int nl = (int)min((long long)kFramesPerGroup, nF - f0);
        // frames f0 + f, all with the group's sweep count (built at each finalize call, not kept live)
        auto fin = [&](uint32_t mask, int it, uint32_t succ, uint32_t zeroL) {
            long long fr[4];
            int itv[4];
            for (int f = 0; f < 4; ++f) { fr[f] = f0 + f; itv[f] = it; }
            finalize(p, s_layer, Eslot, Lslot, fr, mask, itv, succ, zeroL, t);
        };

        // ---- E <- channel LLR, frame-interleaved, stored as E + 127 = (llr ^ 0x80) - 1
        if (p.vec_llr) {
            const int n4 = p.n >> 2;
            for (int q = t; q < n4; q += p.TG) {
                uint32_t r[4];
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    r[f] = f < nl ? __ldcs(reinterpret_cast<const uint32_t*>(p.llr + (f0 + f) * p.n) + q) : 0x7F7F7F7Fu;
                const uint32_t a = prmt<0x5140u>(r[0], r[1]), b = prmt<0x5140u>(r[2], r[3]);
                const uint32_t c = prmt<0x7362u>(r[0], r[1]), d = prmt<0x7362u>(r[2], r[3]);
                Eslot[4 * q + 0] = (prmt<0x5410u>(a, b) ^ 0x80808080u) - 0x01010101u;
                Eslot[4 * q + 1] = (prmt<0x7632u>(a, b) ^ 0x80808080u) - 0x01010101u;
                Eslot[4 * q + 2] = (prmt<0x5410u>(c, d) ^ 0x80808080u) - 0x01010101u;
                Eslot[4 * q + 3] = (prmt<0x7632u>(c, d) ^ 0x80808080u) - 0x01010101u;
            }
        } else {
            for (int j = t; j < p.n; j += p.TG) {
                uint32_t w = 0;
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const uint32_t v = f < nl ? (uint8_t)p.llr[(f0 + f) * p.n + j] : 0x7Fu;
                    w |= ((v ^ 0x80u) - 1u) << (8 * f);
                }
                Eslot[j] = w;
            }
        }
        // ---- target syndrome: one nibble per check row (bit f = frame f)
        for (int i8 = t; i8 < p.mb8; i8 += p.TG) {
            uint32_t bf[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) bf[f] = f < nl ? p.syn[(f0 + f) * p.mb8 + i8] : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = 8 * i8 + q;
                if (i < p.m)
                    sSyn[i] = (uint8_t)(((bf[0] >> q) & 1u) | (((bf[1] >> q) & 1u) << 1) |
                                        (((bf[2] >> q) & 1u) << 2) | (((bf[3] >> q) & 1u) << 3));
            }
        }
        if (t == 0) {
            flags[0] = 0;
            flags[1] = 0;
        }
        slot_bar(p, bar);

        uint32_t active = (1u << nl) - 1u;
        int chk = 0;
        if (p.early_stop) {   // iteration-0 check (R10)
            const uint32_t viol = syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, active);
            const uint32_t done = active & ~viol;
            if (done) {
                fin(done, 0, done, 0xFu);
                slot_bar(p, bar);
            }
            active &= viol;
        }
        int it = 0;
        // one sweep over the block rows; the first sweep of a group (L = 0, R16) is a separate
        // instance so the row update carries no run-time `first` test
#define QKD_SWEEP(FM)                                                                                    \
    for (int I = 0; I < p.Mb; ++I) {                                                                     \
        const int4 li = s_layer[I];                                                                      \
        layer_pass<DMAX, ESM, POW2, SPLIT, FM>(p, li, SPLIT ? s_edge2 + s_soff[I] : s_edge + li.y, t, Eb,   \
                                               Lslot, sSyn + I * p.Z, FM == 1 ? 0xFu : 0u, K, ++rc_lc,   \
                                               rc_lc0, gslot);                                           \
        QKD_MUTATE_BAR(slot_bar(p, bar));                                                                \
    }
        while (active && it < p.T) {
            ++it;
            if (it == 1) {
                QKD_SWEEP(1)
            } else {
                QKD_SWEEP(2)
            }
#undef QKD_SWEEP
            if (p.early_stop) {
                const uint32_t viol = syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, active);
                const uint32_t done = active & ~viol;
                if (done) {
                    fin(done, it, done, 0u);
                    slot_bar(p, bar);
                }
                active &= viol;
            }
        }
        if (active) {   // ran out of iterations (or early_stop = 0): state after sweep T (R12)
            uint32_t succ = 0;
            if (!p.early_stop)
                succ = active & ~syndrome_viol<DMAX, ESM, POW2>(p, s_layer, s_edge, Eb, sSyn, t, flags, chk, bar, K, active);
            fin(active, it, succ, it == 0 ? 0xFu : 0u);
        }
        slot_bar(p, bar);
    }
    }
}

}  // namespace qkd
