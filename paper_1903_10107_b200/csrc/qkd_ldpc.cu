// qkd_ldpc.cu -- B200 (sm_100a) batched quantized LDPC syndrome decoder + C ABI.
// See include/qkd_ldpc.h for the contract and DESIGN.md for the design.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <string>
#include <vector>

#include "decode.cuh"
#include "decode_float.cuh"

#include "qkd_ldpc.h"

using namespace qkd;

// --------------------------------------------------------------------------------------
// errors
// --------------------------------------------------------------------------------------
namespace {
thread_local std::string g_err;
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace
#define QKD_CK(x)                                                                    \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess)                                                       \
            return fail(QKD_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// --------------------------------------------------------------------------------------
// code handle
// --------------------------------------------------------------------------------------
struct Plan {
    int variant = 0;   // 1: degree <= 8 smem E, 2: degree <= 20 smem E, 3: generic smem E, 4: generic global E
    bool pow2 = false; // Z a power of two (byte-OR circulant addressing)
    int TG = 0, GPC = 0, grid = 0, smem = 0, slot_bytes = 0, e_bytes = 0, tab_off = 0;
    long long ngroups = 0, slots = 0;
    size_t ws_L = 0, ws_E = 0, ws_total = 0;
};
// qkd_reconcile_host's copy streams and events (up to 8 chunks), kept in the handle and reused
struct ReconcileCtx {
    static constexpr int kMaxChunks = 8;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t entry = nullptr;
    cudaEvent_t ev[2 * kMaxChunks] = {};
    bool ok = false;
    ReconcileCtx() {
        ok = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking) == cudaSuccess &&
             cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&entry, cudaEventDisableTiming) == cudaSuccess;
        for (auto& e : ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    }
    ~ReconcileCtx() {
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        if (entry) cudaEventDestroy(entry);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_out) cudaStreamDestroy(s_out);
    }
};

struct qkd_code {
    int32_t Mb = 0, Nb = 0, Z = 0;
    int64_t n = 0, m = 0, n_edges = 0;
    int32_t nbase = 0, maxdeg = 0;
    std::vector<int4> layer;   // (deg, first base edge, workspace word offset of the block row, Dp)
    int64_t ws_words = 0;      // workspace words per slot: sum_I Z * deg_I (lane-pair layout: padded rows)
    std::vector<int2> edge;    // (J*Z, shift)
    int4* d_layer = nullptr;
    int2* d_edge = nullptr;
    uint8_t* d_kind = nullptr;     // pos kind or null
    uint8_t* d_payload = nullptr;  // packed payload mask or null (= all payload)
    bool has_short = false;
    int device = 0;
    // split layout (decode variant 5, lane-pair rows): per block row, side A's words then side B's,
    // row stride roundup2(HA) + roundup2(HB); the split table holds 2*HB entries per block row
    bool split = false;
    std::vector<int> soff;
    int nsplit = 0;
    int* d_soff = nullptr;
    int* d_dbg_delta = nullptr;    // QKD_RACECHECK builds: layers back to each base edge's previous writer
    // host-side caches (the handle is shared between threads): launch plans per (device, F,
    // QKD_TG_MAX) and the streams/events of qkd_reconcile_host, one context per concurrent call
    std::mutex mu;
    std::map<std::tuple<int, long long, int>, Plan> plans;
    std::vector<ReconcileCtx*> ctx_free;
};

// --------------------------------------------------------------------------------------
// decode kernel: persistent CTAs; each "slot" (TG threads, own named barrier) decodes
// frame groups of 4 frames taken from an atomic work counter.
// --------------------------------------------------------------------------------------
namespace qkd {
// decode_kernel.cuh, instantiated in decode_inst_*.cu; decode_float_kernel in float_kernel.cu
template <int DMAX, bool ESM, bool POW2, bool SPLIT, bool REFILL>
__global__ void decode_kernel(const DecParams p);
template <bool ESM, bool FLOOD, int FD>
__global__ void decode_float_kernel(const FParams p);
}  // namespace qkd

namespace {

// --------------------------------------------------------------------------------------
// Alice's syndrome: one CTA per frame, frame bits staged in shared memory.
// --------------------------------------------------------------------------------------
__global__ void syndrome_kernel(const int4* __restrict__ layer, const int2* __restrict__ edge, int Mb, int Z,
                                int n, int m, int nb8, int mb8, long long F, const uint8_t* __restrict__ bits,
                                uint8_t* __restrict__ syn) {
    extern __shared__ __align__(16) unsigned char sb[];
    const int lane = threadIdx.x & 31;
    for (long long f = blockIdx.x; f < F; f += gridDim.x) {
        __syncthreads();
        for (int i = threadIdx.x; i < nb8; i += blockDim.x) sb[i] = bits[f * nb8 + i];
        __syncthreads();
        for (int iw = threadIdx.x & ~31; iw < m; iw += blockDim.x) {
            const int i = iw + lane;
            uint32_t par = 0;
            if (i < m) {
                const int I = i / Z, r = i - I * Z;
                const int4 li = layer[I];
                for (int k = 0; k < li.x; ++k) {
                    const int2 e = edge[li.y + k];
                    int idx = r + e.y;
                    idx = idx >= Z ? idx - Z : idx;
                    const int j = e.x + idx;
                    par ^= (sb[j >> 3] >> (j & 7)) & 1u;
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, par != 0);
            const int byte = (iw >> 3) + lane;
            if (lane < 4 && byte < mb8) syn[f * mb8 + byte] = (uint8_t)(bal >> (8 * lane));
        }
    }
}

// Z % 32 == 0: syndrome block I = XOR over its blocks J of x_J rotated by s_IJ (bit r of the
// rotated Z-bit segment is x_J[(r + s) mod Z]), 32 checks per word: word w of the rotation by
// s = 32 q + t is the funnel shift of words w+q and w+q+1 (mod Z/32) right by t.  One CTA per frame,
// the frame's words staged in shared memory.
__global__ void syndrome_qc_kernel(const int4* __restrict__ layer, const int2* __restrict__ edge, int Mb, int Z,
                                   int nw, int mb8, long long F, const uint8_t* __restrict__ bits,
                                   uint8_t* __restrict__ syn) {
    extern __shared__ __align__(16) uint32_t sx[];
    const int W = Z >> 5;
    for (long long f = blockIdx.x; f < F; f += gridDim.x) {
        __syncthreads();
        const uint32_t* xf = reinterpret_cast<const uint32_t*>(bits + f * (long long)nw * 4);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) sx[i] = xf[i];
        __syncthreads();
        uint32_t* so = reinterpret_cast<uint32_t*>(syn + f * (long long)mb8);
        for (int idx = threadIdx.x; idx < Mb * W; idx += blockDim.x) {
            const int I = idx / W, w = idx - I * W;
            const int4 li = layer[I];
            uint32_t acc = 0;
            for (int k = 0; k < li.x; ++k) {
                const int2 e = edge[li.y + k];            // (J*Z, shift)
                const int q = e.y >> 5, t = e.y & 31;
                int w0 = w + q;
                w0 = w0 >= W ? w0 - W : w0;
                const int w1 = w0 + 1 == W ? 0 : w0 + 1;
                const uint32_t* seg = sx + (e.x >> 5);
                acc ^= __funnelshift_r(seg[w0], seg[w1], t);
            }
            so[idx] = acc;
        }
    }
}

// --------------------------------------------------------------------------------------
// Bob's channel LLRs (P:103-112 quantization, P:157 puncture/shorten)
// --------------------------------------------------------------------------------------
__global__ void build_llr_kernel(int n, int nb8, long long F, int Lq, const uint8_t* __restrict__ y,
                                 const uint8_t* __restrict__ known, const uint8_t* __restrict__ kind,
                                 int8_t* __restrict__ llr, const long long* __restrict__ F_dev = nullptr) {
    const long long total = (F_dev ? *F_dev : F) * nb8;   // F_dev: device-resident count (adaptive rounds)
    if ((n & 7) == 0 && (reinterpret_cast<uintptr_t>(llr) & 7) == 0) {
        // one input byte -> one 8-byte store: bit s of y selects -Lq / +Lq for position 8b + s
        const uint32_t pos = (uint32_t)(Lq & 0xFF) * 0x01010101u, neg = (uint32_t)(-Lq & 0xFF) * 0x01010101u;
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
             q += (long long)gridDim.x * blockDim.x) {
            const long long f = q / nb8;
            const int b = (int)(q - f * nb8);
            const uint32_t yb = y[q];
            // byte mask of set bits: bit s -> byte s (0xFF)
            const uint32_t lo = ((yb & 0x0Fu) * 0x00204081u & 0x01010101u) * 0xFFu;
            const uint32_t hi = (((yb >> 4) & 0x0Fu) * 0x00204081u & 0x01010101u) * 0xFFu;
            uint2 v = make_uint2((neg & lo) | (pos & ~lo), (neg & hi) | (pos & ~hi));
            if (kind) {
                const uint2 kd = *reinterpret_cast<const uint2*>(kind + 8LL * b);
                const uint32_t kb = known ? known[q] : 0u;
                const uint32_t klo = ((kb & 0x0Fu) * 0x00204081u & 0x01010101u) * 0xFFu;
                const uint32_t khi = (((kb >> 4) & 0x0Fu) * 0x00204081u & 0x01010101u) * 0xFFu;
                uint32_t w[2] = {v.x, v.y};
                const uint32_t kw[2] = {kd.x, kd.y}, km[2] = {klo, khi};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // punctured (1) -> 0, shortened (2) -> +-127 by the known bit (R19)
                    const uint32_t p1 = ((kw[h] & 0x01010101u) & ~(kw[h] >> 1)) * 0xFFu;   // kind == 1
                    const uint32_t s2 = ((kw[h] >> 1) & 0x01010101u) * 0xFFu;             // kind == 2
                    const uint32_t sv = (0x81818181u & km[h]) | (0x7F7F7F7Fu & ~km[h]);
                    w[h] = (w[h] & ~(p1 | s2)) | (sv & s2);
                }
                v = make_uint2(w[0], w[1]);
            }
            *reinterpret_cast<uint2*>(llr + f * n + 8LL * b) = v;
        }
        return;
    }
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long f = q / nb8;
        const int b = (int)(q - f * nb8);
        const uint32_t yb = y[q];
        const uint32_t kb = known ? known[q] : 0u;
        int8_t* out = llr + f * n;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int j = 8 * b + s;
            if (j >= n) break;
            int v = ((yb >> s) & 1u) ? -Lq : Lq;
            if (kind) {
                const uint8_t kd = kind[j];
                if (kd == 1) v = 0;
                else if (kd == 2) v = ((kb >> s) & 1u) ? -127 : 127;
            }
            out[j] = (int8_t)v;
        }
    }
}

// --------------------------------------------------------------------------------------
// scoring against Alice's key (harness)
// --------------------------------------------------------------------------------------
__global__ void score_kernel(int nb8, long long F, const uint8_t* __restrict__ bits, const uint8_t* __restrict__ x,
                             const uint8_t* __restrict__ payload, const uint8_t* __restrict__ success,
                             int32_t* __restrict__ errors, unsigned long long* counters) {
    __shared__ int red[32];
    for (long long f = blockIdx.x; f < F; f += gridDim.x) {
        int c = 0;
        for (int i = threadIdx.x; i < nb8; i += blockDim.x) {
            uint32_t d = (uint32_t)(bits[f * nb8 + i] ^ x[f * nb8 + i]);
            if (payload) d &= payload[i];
            c += __popc(d);
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
            if (errors) errors[f] = tot;
            if (counters && tot > 0) {
                atomicAdd(counters + 2, 1ull);
                if (success[f]) atomicAdd(counters + 3, 1ull);
            }
        }
        __syncthreads();
    }
}

__global__ void tau_table_kernel(uint8_t* out, Konst K) {
    const int p = threadIdx.x;   // 64 threads
    for (int w = 0; w < 16; ++w) {
        const uint32_t a = rep4((uint32_t)p);
        const uint32_t b = (uint32_t)(4 * w) | ((uint32_t)(4 * w + 1) << 8) | ((uint32_t)(4 * w + 2) << 16) |
                           ((uint32_t)(4 * w + 3) << 24);
        const uint32_t t = tau4(a, b, K);
        // the complement form used by the split kernel must agree byte for byte (else 0xFF)
        const uint32_t tc = tau4c(a ^ 0x3F3F3F3Fu, b ^ 0x3F3F3F3Fu, K) ^ 0x3F3F3F3Fu;
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = (t >> (8 * q)) & 0xFFu;
            out[p * 64 + 4 * w + q] = (uint8_t)(v == ((tc >> (8 * q)) & 0xFFu) ? v : 0xFFu);
        }
    }
}


// --------------------------------------------------------------------------------------
// interactive rate adaptation (qkd_reconcile_adaptive): per-round pattern, compaction
// --------------------------------------------------------------------------------------
// kind[order[i]] = 2 (shortened) for i < s, 1 (punctured) for s <= i < d; kind is zeroed first
__global__ void reveal_kind_kernel(const int32_t* __restrict__ order, long long d, long long s, int n,
                                   uint8_t* __restrict__ kind) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < d; i += (long long)gridDim.x * blockDim.x) {
        const int j = order[i];
        if (j >= 0 && j < n) kind[j] = i < s ? 2 : 1;
    }
}

// The active-frame list of the interactive rounds lives on the device: idx[0..*cnt) are the frame ids
// still failing, in increasing order; every kernel of a round reads the count from device memory,
// so the rounds are enqueued back to back without a host synchronisation.
__global__ void init_active_kernel(int32_t* __restrict__ idx, long long F, long long* __restrict__ cnt) {
    for (long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x; a < F; a += (long long)gridDim.x * blockDim.x)
        idx[a] = (int32_t)a;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = F;
}

// dst row a = src row idx[a] (row_bytes each) for a < *cnt; one CTA per row, 4-byte moves when aligned
__global__ void gather_rows_kernel(const int32_t* __restrict__ idx, const long long* __restrict__ cnt,
                                   const uint8_t* __restrict__ src, int row_bytes, uint8_t* __restrict__ dst) {
    const long long rows = *cnt;
    for (long long a = blockIdx.x; a < rows; a += gridDim.x) {
        const uint8_t* s = src + (long long)idx[a] * row_bytes;
        uint8_t* d = dst + a * row_bytes;
        if ((row_bytes & 3) == 0) {
            for (int i = threadIdx.x; i < row_bytes / 4; i += blockDim.x)
                reinterpret_cast<uint32_t*>(d)[i] = reinterpret_cast<const uint32_t*>(s)[i];
        } else {
            for (int i = threadIdx.x; i < row_bytes; i += blockDim.x) d[i] = s[i];
        }
    }
}

// results of compacted frame a go to frame idx[a] when it matched (or on the last round)
__global__ void scatter_results_kernel(const int32_t* __restrict__ idx, const long long* __restrict__ cnt, int nb8,
                                       int round, int last, const uint8_t* __restrict__ cbits,
                                       const int32_t* __restrict__ citers, const uint8_t* __restrict__ csucc,
                                       uint8_t* __restrict__ bits, int32_t* __restrict__ iters,
                                       int32_t* __restrict__ rounds, uint8_t* __restrict__ success) {
    const long long rows = *cnt;
    for (long long a = blockIdx.x; a < rows; a += gridDim.x) {
        if (!csucc[a] && !last) continue;
        const long long f = idx[a];
        for (int i = threadIdx.x; i < nb8; i += blockDim.x) bits[f * nb8 + i] = cbits[a * nb8 + i];
        if (threadIdx.x == 0) {
            iters[f] = citers[a];
            success[f] = csucc[a];
            rounds[f] = round;
        }
    }
}

// next round's list: the entries of idx_in[0..*cnt_in) whose decode failed, order kept (one CTA of
// kCompactThreads threads: each takes a contiguous chunk, an exclusive scan of the per-thread counts
// places the chunks)
constexpr int kCompactThreads = 1024;
__global__ void __launch_bounds__(kCompactThreads) compact_failed_kernel(
        const int32_t* __restrict__ idx_in, const long long* __restrict__ cnt_in, const uint8_t* __restrict__ succ,
        int32_t* __restrict__ idx_out, long long* __restrict__ cnt_out) {
    __shared__ long long warp_tot[kCompactThreads / 32];
    const long long n = *cnt_in;
    const long long per = (n + kCompactThreads - 1) / kCompactThreads;
    const long long b = threadIdx.x * per, e = min(n, b + per);
    long long mine = 0;
    for (long long a = b; a < e; ++a) mine += succ[a] ? 0 : 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = mine;                                    // inclusive scan within the warp
    for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {                                           // scan of the warp totals
        long long t = lane < kCompactThreads / 32 ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        if (lane < kCompactThreads / 32) warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    long long out = (wid ? warp_tot[wid - 1] : 0) + incl - mine;
    for (long long a = b; a < e; ++a)
        if (!succ[a]) idx_out[out++] = idx_in[a];
    if (threadIdx.x == kCompactThreads - 1) *cnt_out = out;
}


// --------------------------------------------------------------------------------------
// exact floating-point layered BP (decode_float.cuh): one frame per slot
// --------------------------------------------------------------------------------------
__global__ void build_llr_float_kernel(int n, int nb8, long long F, float Lc, const uint8_t* __restrict__ y,
                                       const uint8_t* __restrict__ known, const uint8_t* __restrict__ kind,
                                       float* __restrict__ llr) {
    const long long total = F * (long long)n;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long f = q / n;
        const int j = (int)(q - f * n);
        const int kd = kind ? kind[j] : 0;
        float v;
        if (kd == 1) v = 0.0f;
        else if (kd == 2) v = ((known[f * nb8 + (j >> 3)] >> (j & 7)) & 1) ? -kLlrKnown : kLlrKnown;
        else v = ((y[f * nb8 + (j >> 3)] >> (j & 7)) & 1) ? -Lc : Lc;
        llr[q] = v;
    }
}

// --------------------------------------------------------------------------------------
// launch planning
// --------------------------------------------------------------------------------------


struct DevInfo {
    int sms = 0, smem_optin = 0;
    bool ok = false;
};

DevInfo dev_info(int dev) {
    static std::mutex mu;
    static DevInfo cache[64];
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return DevInfo{};
    if (!cache[dev].ok) {
        cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&cache[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cache[dev].ok = cache[dev].sms > 0;
    }
    return cache[dev];
}

template <int DMAX, bool ESM, bool POW2, bool SPLIT = false, bool REFILL = false>
const void* kfun() {
    return reinterpret_cast<const void*>(&decode_kernel<DMAX, ESM, POW2, SPLIT, REFILL>);
}

// refill: per-frame lane scheduling (opt-in, QKD_REFILL=1; not for the lane-pair variant)
const void* kernel_of(int variant, bool pow2, bool refill = false) {
    if (refill && variant != 5 && variant < 6) {
        switch (variant) {
            case 1: return pow2 ? kfun<8, true, true, false, true>() : kfun<8, true, false, false, true>();
            case 2: return pow2 ? kfun<20, true, true, false, true>() : kfun<20, true, false, false, true>();
            case 3: return kfun<0, true, false, false, true>();
            default: return kfun<0, false, false, false, true>();
        }
    }
    switch (variant) {
        case 1: return pow2 ? kfun<8, true, true>() : kfun<8, true, false>();
        case 2: return pow2 ? kfun<20, true, true>() : kfun<20, true, false>();
        case 3: return kfun<0, true, false>();
        case 6: return pow2 ? kfun<32, true, true>() : kfun<32, true, false>();
        case 7: return pow2 ? kfun<8, false, true>() : kfun<8, false, false>();
        case 8: return kfun<32, false, false>();
        case 5: return pow2 ? kfun<20, true, true, true>() : kfun<20, true, false, true>();
        default: return kfun<0, false, false>();
    }
}

// 1, 2, -1, -2, -256 as kernel arguments: opaque to ptxas, so a*one + c stays an IMAD (FMA pipe)
Konst runtime_konst() {
    return Konst{1u, 2u, 0xFFFFFFFFu, 0xFFFFFFFEu, 0xFFFFFF00u, 0xFF80FF80u, 0x3F3F3F3Fu, 0x7F7F7F7Fu, 0u, 256u, 0x80000000u, 1u << 26};
}

// Decode variant of a code on a device (fixed at code creation: the split variant has its own
// message layout).  1: degree <= 8, smem E; 2: degree <= 20, smem E, one row per thread;
// 5: degree 9..20, smem E, lane-pair rows; 6: degree 21..32, smem E, one row per thread;
// 7: degree <= 8, E in global memory (frames too long for shared memory), register rows;
// 8: degree 9..32, E in global memory, register rows;
// 3: generic smem E; 4: generic global E.
int choose_variant(int Mb, int64_t n, int64_t m, int nbase, int maxdeg, int smem_optin, bool allow_split) {
    const long long syn_ctl = ((m + 15) & ~15LL) + 64;
    const long long tab1 = (long long)Mb * (sizeof(int4) + sizeof(int)) + (long long)nbase * 2 * sizeof(int2) +
                           (long long)Mb * sizeof(int2);
    const bool fits = 4LL * n + syn_ctl + tab1 <= smem_optin;
    if (fits && maxdeg <= 8) return 1;
    if (fits && maxdeg <= 20) return allow_split ? 5 : 2;
    if (fits && maxdeg <= 32 && !std::getenv("QKD_NO_D32")) return 6;
    if (!fits && maxdeg <= 32 && !std::getenv("QKD_NO_GREG")) return maxdeg <= 8 ? 7 : 8;
    return fits ? 3 : 4;
}

// the kernel's dynamic shared-memory limit, raised once per (kernel, device) to the device maximum
// (a per-call setting to the plan's size could lower it under another thread's launch)
int prepare_kernel(const void* k, int dev, int smem_optin) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({k, dev})) return QKD_OK;
    QKD_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
    done.insert({k, dev});
    return QKD_OK;
}

int make_plan_uncached(const qkd_code* c, long long F, Plan& pl);

// launch plan of (code, F) on the current device, cached in the handle: no attribute calls or
// occupancy queries on the per-call path once a batch size has been seen
int make_plan(const qkd_code* c_, long long F, Plan& pl) {
    qkd_code* c = const_cast<qkd_code*>(c_);
    int dev = 0;
    QKD_CK(cudaGetDevice(&dev));
    const char* e = std::getenv("QKD_TG_MAX");
    const auto key = std::make_tuple(dev, F, e ? atoi(e) : 0);
    {
        std::lock_guard<std::mutex> lk(c->mu);
        auto it = c->plans.find(key);
        if (it != c->plans.end()) {
            pl = it->second;
            return QKD_OK;
        }
    }
    const int rc = make_plan_uncached(c, F, pl);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->plans.size() >= 256) c->plans.clear();
    c->plans[key] = pl;
    return QKD_OK;
}

int make_plan_uncached(const qkd_code* c, long long F, Plan& pl) {
    int dev = 0;
    QKD_CK(cudaGetDevice(&dev));
    DevInfo di = dev_info(dev);
    if (!di.ok) return fail(QKD_ECUDA, "cannot query device attributes");
    pl.ngroups = (F + kFramesPerGroup - 1) / kFramesPerGroup;
    const long long syn_ctl = ((c->m + 15) & ~15LL) + 64;   // syndrome nibbles + control words
    const long long e_bytes = 4LL * c->n;
    pl.variant = choose_variant(c->Mb, c->n, c->m, c->nbase, c->maxdeg, di.smem_optin, c->split);
    if ((pl.variant == 5) != c->split) return fail(QKD_EUNSUP, "code was created for another device geometry");
    // byte-OR addressing: smem E variants, and variant 7 (one slot per CTA, E offsets from the slot's global base)
    pl.pow2 = (pl.variant <= 2 || pl.variant == 5 || pl.variant == 6 || pl.variant == 7) && ((c->Z & (c->Z - 1)) == 0);
    int tg_max = pl.variant == 5 ? 1024 : pl.variant == 1 ? QKD_V1_THREADS
                 : (pl.variant == 2 ? 512 : (pl.variant == 7 ? QKD_G8_THREADS : (pl.variant == 8 ? QKD_G32_THREADS : (pl.variant == 6 ? QKD_D32_THREADS : 256))));
    if (const char* e = std::getenv("QKD_TG_MAX"))   // experiments: fewer threads per frame group
        tg_max = std::max(32, std::min(tg_max, atoi(e) / 32 * 32));
    if (pl.variant == 5)   // two lanes per row, 16 rows per warp
        pl.TG = (int)std::min<long long>(((long long)c->Z + 15) / 16 * 32, tg_max);
    else
        pl.TG = (int)std::min<long long>(((long long)c->Z + 31) / 32 * 32, tg_max);
    const bool gE = pl.variant == 4 || pl.variant >= 7;   // E in the global workspace
    pl.e_bytes = gE ? 0 : (int)e_bytes;
    long long slot = (pl.e_bytes + syn_ctl + 15) & ~15LL;   // 16-byte aligned slots and tables
    if (pl.pow2) {   // slot E bases must be multiples of 4Z for the byte-OR addressing
        const long long al = 4LL * c->Z;
        slot = (slot + al - 1) / al * al;
    }
    pl.slot_bytes = (int)slot;
    int gpc = std::min(15, tg_max / pl.TG);
    const long long per_slot_tab = (long long)(c->nbase + c->nsplit) * sizeof(int2);
    const long long fixed_tab = (long long)c->Mb * (sizeof(int4) + sizeof(int));
    if (slot + per_slot_tab + fixed_tab > di.smem_optin)
        return fail(QKD_EUNSUP, "frame too long for the shared-memory buffers");
    while (gpc > 1 && (long long)gpc * (slot + per_slot_tab) + fixed_tab > (long long)di.smem_optin) --gpc;
    const long long need = (pl.ngroups + di.sms - 1) / di.sms;
    gpc = (int)std::max<long long>(1, std::min<long long>(gpc, need));
    pl.GPC = gpc;
    pl.tab_off = gpc * pl.slot_bytes;
    pl.smem = pl.tab_off + (int)(fixed_tab + gpc * per_slot_tab);
    const void* k = kernel_of(pl.variant, pl.pow2);
    if (int rc = prepare_kernel(k, dev, di.smem_optin)) return rc;
    if (int rc = prepare_kernel(kernel_of(pl.variant, pl.pow2, true), dev, di.smem_optin)) return rc;
    int per_sm = 0;
    QKD_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, pl.TG * pl.GPC, pl.smem));
    if (per_sm < 1) return fail(QKD_EUNSUP, "decode kernel cannot be resident with this geometry");
    const long long ctas = (pl.ngroups + gpc - 1) / gpc;
    pl.grid = (int)std::max<long long>(1, std::min<long long>(ctas, (long long)per_sm * di.sms));
    pl.slots = (long long)pl.grid * gpc;
    // + slack after the last slot: the message prefetch reads up to 32 positions of a thread's next
    // row whatever its degree (decode.cuh row_update), i.e. up to 32 x 32 words past a row chunk
    pl.ws_L = ((size_t)pl.slots * (size_t)c->ws_words + 32 * 32) * 4;
    pl.ws_E = gE ? (size_t)pl.slots * (size_t)c->n * 4 : 0;
    pl.ws_total = 256 + pl.ws_L + pl.ws_E;
    return QKD_OK;
}

}  // namespace

// ======================================================================================
// C ABI
// ======================================================================================
extern "C" {

const char* qkd_last_error(void) { return g_err.c_str(); }

int qkd_code_create(const int32_t* base_shifts, int32_t Mb, int32_t Nb, int32_t Z, const uint8_t* pos_kind,
                    qkd_code** out) {
    if (!out || !base_shifts) return fail(QKD_EINVAL, "null argument");
    *out = nullptr;
    if (Mb < 1 || Nb <= Mb || Z < 1) return fail(QKD_EINVAL, "need Mb >= 1, Nb > Mb, Z >= 1");
    if ((long long)Nb * Z > (1LL << 30)) return fail(QKD_EUNSUP, "n too large");
    qkd_code* c = new qkd_code();
    {   // the decode variant (and with it the message layout) is fixed here, per device
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) { delete c; return fail(QKD_ECUDA, "no CUDA device"); }
        const DevInfo di = dev_info(dev);
        if (!di.ok) { delete c; return fail(QKD_ECUDA, "cannot query device attributes"); }
        int nb = 0, md = 0;
        for (int I = 0; I < Mb; ++I) {
            int d = 0;
            for (int J = 0; J < Nb; ++J) d += base_shifts[(size_t)I * Nb + J] >= 0;
            nb += d;
            md = std::max(md, d);
        }
        // QKD_SPLIT=1 in the environment at code creation selects the lane-pair variant (5) for
        // codes of check degree 9..20; the default is one row per thread (variant 2), which
        // measured ~4% faster on C5a (profiles/r1v4_split_ab.md)
        const char* env = std::getenv("QKD_SPLIT");
        const bool allow = env && env[0] == '1';
        c->split = choose_variant(Mb, (int64_t)Nb * Z, (int64_t)Mb * Z, nb, md, di.smem_optin, allow) == 5;
    }
    c->Mb = Mb;
    c->Nb = Nb;
    c->Z = Z;
    c->n = (int64_t)Nb * Z;
    c->m = (int64_t)Mb * Z;
    for (int I = 0; I < Mb; ++I) {
        int4 li = make_int4(0, (int)c->edge.size(), 0, 0);
        for (int J = 0; J < Nb; ++J) {
            const int s = base_shifts[(size_t)I * Nb + J];
            if (s < -1 || s >= Z) {
                delete c;
                return fail(QKD_ESHIFT, "shift " + std::to_string(s) + " at base block (" + std::to_string(I) +
                                            "," + std::to_string(J) + ") outside [-1, Z)");
            }
            if (s >= 0) {
                c->edge.push_back(make_int2(J * Z, s));
                li.x++;
            }
        }
        if (li.x > 64) {
            delete c;
            return fail(QKD_EUNSUP, "check degree > 64 in block row " + std::to_string(I));
        }
        c->maxdeg = std::max(c->maxdeg, li.x);
        if (c->split) {   // side A words [0, WA), side B words [WA, WA + roundup2(HB))
            const int ha = li.x >> 1, hb = li.x - ha;
            li.w = ((ha + 1) & ~1) + ((hb + 1) & ~1);
            c->soff.push_back(c->nsplit);
            c->nsplit += 2 * hb;
        } else {   // D words per row in emission order, dense regions (decode.cuh msg_word)
            li.w = li.x;
        }
        li.z = (int)c->ws_words;
        // lane-pair layout: Z rows of li.w words; otherwise 32-row chunks of li.w = D words (msg_word)
        c->ws_words += (c->split ? (int64_t)Z : ((int64_t)Z + 31) / 32 * 32) * li.w;
        c->ws_words = (c->ws_words + 3) & ~3LL;   // 16-byte aligned block rows (lane-pair layout: 64-bit moves)
        if (c->ws_words > (1LL << 31) - 1) {
            delete c;
            return fail(QKD_EUNSUP, "code too large for the 32-bit workspace offsets");
        }
        c->layer.push_back(li);
    }
    c->nbase = (int)c->edge.size();
    c->n_edges = (int64_t)c->nbase * Z;
    cudaError_t e = cudaGetDevice(&c->device);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_layer, sizeof(int4) * c->layer.size());
    if (e == cudaSuccess) e = cudaMalloc(&c->d_edge, sizeof(int2) * std::max<size_t>(1, c->edge.size()));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_layer, c->layer.data(), sizeof(int4) * c->layer.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !c->edge.empty())
        e = cudaMemcpy(c->d_edge, c->edge.data(), sizeof(int2) * c->edge.size(), cudaMemcpyHostToDevice);
#ifdef QKD_RACECHECK
    if (e == cudaSuccess && !c->edge.empty()) {
        // delta of base edge (I, J): smallest d in [1, Mb] such that block row (I - d) mod Mb holds J
        std::vector<int> delta(c->edge.size(), Mb);
        for (int I = 0; I < Mb; ++I)
            for (int k = 0; k < c->layer[I].x; ++k) {
                const int J = c->edge[c->layer[I].y + k].x / Z;
                for (int d = 1; d <= Mb; ++d) {
                    const int I2 = ((I - d) % Mb + Mb) % Mb;
                    bool has = false;
                    for (int k2 = 0; k2 < c->layer[I2].x; ++k2) has |= c->edge[c->layer[I2].y + k2].x / Z == J;
                    if (has) { delta[c->layer[I].y + k] = d; break; }
                }
            }
        e = cudaMalloc(&c->d_dbg_delta, sizeof(int) * delta.size());
        if (e == cudaSuccess) e = cudaMemcpy(c->d_dbg_delta, delta.data(), sizeof(int) * delta.size(), cudaMemcpyHostToDevice);
    }
#endif
    if (e == cudaSuccess && c->split) {
        e = cudaMalloc(&c->d_soff, sizeof(int) * c->soff.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(c->d_soff, c->soff.data(), sizeof(int) * c->soff.size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && pos_kind) {
        bool any = false;
        std::vector<uint8_t> pay((size_t)(c->n + 7) / 8, 0);
        for (int64_t j = 0; j < c->n; ++j) {
            if (pos_kind[j] > 2) {
                qkd_code_destroy(c);
                return fail(QKD_EINVAL, "pos_kind values must be 0, 1 or 2");
            }
            if (pos_kind[j] != 0) any = true;
            if (pos_kind[j] == 2) c->has_short = true;
            if (pos_kind[j] == 0) pay[j >> 3] |= (uint8_t)(1u << (j & 7));
        }
        if (any) {
            e = cudaMalloc(&c->d_kind, (size_t)c->n);
            if (e == cudaSuccess) e = cudaMemcpy(c->d_kind, pos_kind, (size_t)c->n, cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_payload, pay.size());
            if (e == cudaSuccess) e = cudaMemcpy(c->d_payload, pay.data(), pay.size(), cudaMemcpyHostToDevice);
        }
    }
    if (e != cudaSuccess) {
        qkd_code_destroy(c);
        return fail(e == cudaErrorMemoryAllocation ? QKD_ENOMEM : QKD_ECUDA,
                    std::string("code tables: ") + cudaGetErrorString(e));
    }
    *out = c;
    return QKD_OK;
}

void qkd_code_destroy(qkd_code* c) {
    if (!c) return;
    for (ReconcileCtx* x : c->ctx_free) delete x;
    if (c->d_layer) cudaFree(c->d_layer);
    if (c->d_edge) cudaFree(c->d_edge);
    if (c->d_kind) cudaFree(c->d_kind);
    if (c->d_payload) cudaFree(c->d_payload);
    if (c->d_soff) cudaFree(c->d_soff);
    if (c->d_dbg_delta) cudaFree(c->d_dbg_delta);
    delete c;
}

int qkd_code_info(const qkd_code* c, int64_t* n, int64_t* m, int64_t* n_edges, int32_t* max_row_deg) {
    if (!c) return fail(QKD_EINVAL, "null code");
    if (n) *n = c->n;
    if (m) *m = c->m;
    if (n_edges) *n_edges = c->n_edges;
    if (max_row_deg) *max_row_deg = c->maxdeg;
    return QKD_OK;
}

int qkd_llr_magnitude(double q) {
    if (!(q > 0.0 && q < 0.5)) return fail(QKD_EINVAL, "qber must lie in (0, 0.5)");
    const double v = std::nearbyint(4.0 * std::log((1.0 - q) / q));   // ties never occur at the configs
    return (int)std::min(127.0, v);
}

int qkd_syndrome(const qkd_code* c, int64_t F, const uint8_t* bits, uint8_t* syn, void* stream) {
    if (!c || F < 0 || (F > 0 && (!bits || !syn))) return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    const int nb8 = (int)((c->n + 7) / 8), mb8 = (int)((c->m + 7) / 8);
    if (nb8 > 160 * 1024) return fail(QKD_EUNSUP, "frame too long for the syndrome kernel");
    int dev = 0;
    QKD_CK(cudaGetDevice(&dev));
    const DevInfo di = dev_info(dev);
    QKD_CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(&syndrome_kernel),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, nb8));
    QKD_CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(&syndrome_qc_kernel),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, nb8));
    const int grid = (int)std::min<long long>(F, (long long)di.sms * 8);
    if (c->Z % 32 == 0 && ((reinterpret_cast<uintptr_t>(bits) | reinterpret_cast<uintptr_t>(syn)) & 3) == 0) {
        // n, m are multiples of 32 here, so frames are whole words
        syndrome_qc_kernel<<<grid, 256, nb8, (cudaStream_t)stream>>>(c->d_layer, c->d_edge, c->Mb, c->Z, nb8 / 4,
                                                                     mb8, F, bits, syn);
    } else {
        syndrome_kernel<<<grid, 256, nb8, (cudaStream_t)stream>>>(c->d_layer, c->d_edge, c->Mb, c->Z, (int)c->n,
                                                                   (int)c->m, nb8, mb8, F, bits, syn);
    }
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

int qkd_build_llr(const qkd_code* c, double qber, int64_t F, const uint8_t* y, const uint8_t* known, int8_t* llr,
                  void* stream) {
    if (!c || F < 0 || (F > 0 && (!y || !llr))) return fail(QKD_EINVAL, "bad argument");
    const int Lq = qkd_llr_magnitude(qber);
    if (Lq < 0) return Lq;
    if (c->has_short && !known) return fail(QKD_EINVAL, "code has shortened positions: known_bits required");
    if (F == 0) return QKD_OK;
    const int nb8 = (int)((c->n + 7) / 8);
    const long long total = F * nb8;
    const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 64);
    build_llr_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((int)c->n, nb8, F, Lq, y, c->d_kind ? known : nullptr,
                                                             c->d_kind, llr);
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

size_t qkd_workspace_bytes(const qkd_code* c, int64_t F) {
    if (!c || F < 0) return 0;
    Plan pl;
    if (make_plan(c, std::max<int64_t>(F, 1), pl) != QKD_OK) return 0;
    return pl.ws_total;
}

int qkd_launch_info(const qkd_code* c, int64_t F, int32_t* info) {
    if (!c || !info || F < 1) return fail(QKD_EINVAL, "bad argument");
    Plan pl;
    const int rc = make_plan(c, F, pl);
    if (rc) return rc;
    info[0] = pl.variant + (pl.pow2 ? 10 : 0);
    info[1] = pl.TG;
    info[2] = pl.GPC;
    info[3] = pl.grid;
    info[4] = pl.smem;
    info[5] = kFramesPerGroup;
    info[6] = (int32_t)pl.ngroups;
    return QKD_OK;
}

// F_dev (internal, interactive rounds): the launch decodes the first *F_dev <= F frames; the plan
// (variant, grid, workspace) is the one for F
static int decode_launch(const qkd_code* c, int64_t F, const long long* F_dev, const int8_t* llr, const uint8_t* syn,
                         int32_t max_iter, int32_t early_stop, void* ws, size_t ws_bytes, uint8_t* bits,
                         int32_t* iters, uint8_t* success, int8_t* fL, int8_t* fE, int64_t* counters, void* stream) {
    if (!c || F < 0 || max_iter < 0) return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    if (!llr || !syn || !ws || !bits || !iters || !success) return fail(QKD_EINVAL, "null buffer");
    Plan pl;
    int rc = make_plan(c, F, pl);
    if (rc) return rc;
    if (ws_bytes < pl.ws_total)
        return fail(QKD_EDIM, "workspace too small: need " + std::to_string(pl.ws_total) + " bytes");
    char* w = static_cast<char*>(ws);
    DecParams p{};
    p.layer = c->d_layer;
    p.edge = c->d_edge;
    p.soff = c->split ? c->d_soff : nullptr;
    p.nsplit = c->nsplit;
    p.Mb = c->Mb;
    p.Z = c->Z;
    p.nbase = c->nbase;
    p.n = (int)c->n;
    p.m = (int)c->m;
    p.mb8 = (int)((c->m + 7) / 8);
    p.nb8 = (int)((c->n + 7) / 8);
    p.n_edges = c->n_edges;
    p.ws_words = c->ws_words;
    p.llr = llr;
    p.syn = syn;
    p.F = F;
    p.ngroups = pl.ngroups;
    p.F_dev = F_dev;
    p.T = max_iter;
    p.early_stop = early_stop ? 1 : 0;
    p.vec_llr = (c->n % 4 == 0) && ((reinterpret_cast<uintptr_t>(llr) & 3) == 0);
    {   // per-frame lane refill: default for variant 1 (degree <= 8; C5b -11%), opt-in elsewhere
        // (QKD_REFILL=1; C5a +9%); QKD_REFILL=0 turns it off everywhere
        const char* env = std::getenv("QKD_REFILL");
        const bool on = env ? env[0] == '1' : pl.variant == 1;
        p.refill = (pl.variant != 5 && pl.variant < 6 && on) ? 1 : 0;
    }
    p.work = reinterpret_cast<int*>(w);
    p.Lws = reinterpret_cast<uint32_t*>(w + 256);
    p.Ews = pl.ws_E ? reinterpret_cast<uint32_t*>(w + 256 + pl.ws_L) : nullptr;
    p.bits = bits;
    p.iters = iters;
    p.success = success;
    p.fL = fL;
    p.fE = fE;
    p.counters = reinterpret_cast<unsigned long long*>(counters);
    p.TG = pl.TG;
    p.GPC = pl.GPC;
    p.slot_bytes = pl.slot_bytes;
    p.e_bytes = pl.e_bytes;
    p.tab_off = pl.tab_off;
    p.K = runtime_konst();
    cudaStream_t st = (cudaStream_t)stream;
    QKD_CK(cudaMemsetAsync(p.work, 0, sizeof(int), st));
    const dim3 grid(pl.grid), block(pl.TG * pl.GPC);
    void* args[] = {&p};
#ifdef QKD_RACECHECK
    // debug build: layer stamps per slot, checked by the kernel (decode_kernel.cuh rc_row); the
    // call synchronises and fails when any E read saw a stale or early stamp
    const size_t dbg_words = 16 + (size_t)pl.grid * pl.GPC * (size_t)c->n;
    QKD_CK(cudaMalloc(&p.dbg, dbg_words * 4));
    QKD_CK(cudaMemsetAsync(p.dbg, 0, dbg_words * 4, st));
    p.dbg_delta = c->d_dbg_delta;
#endif
    QKD_CK(cudaLaunchKernel(kernel_of(pl.variant, pl.pow2, p.refill != 0), grid, block, args, pl.smem, st));
    QKD_CK(cudaGetLastError());
#ifdef QKD_RACECHECK
    {
        unsigned rec[8] = {0};
        QKD_CK(cudaStreamSynchronize(st));
        QKD_CK(cudaMemcpy(rec, p.dbg, sizeof(rec), cudaMemcpyDeviceToHost));
        cudaFree(p.dbg);
        if (rec[0])
            return fail(QKD_ECUDA, "racecheck: " + std::to_string(rec[0]) + " E reads out of layer order; first: layer " +
                                       std::to_string(rec[1]) + " row " + std::to_string(rec[2]) + " base edge " +
                                       std::to_string(rec[3]) + " stamp " + std::to_string((int)rec[4]) + " expected " +
                                       std::to_string((int)rec[5]) + " slot " + std::to_string(rec[6]));
    }
#endif
    return QKD_OK;
}

int qkd_decode_batch(const qkd_code* c, int64_t F, const int8_t* llr, const uint8_t* syn, int32_t max_iter,
                     int32_t early_stop, void* ws, size_t ws_bytes, uint8_t* bits, int32_t* iters,
                     uint8_t* success, int8_t* fL, int8_t* fE, int64_t* counters, void* stream) {
    return decode_launch(c, F, nullptr, llr, syn, max_iter, early_stop, ws, ws_bytes, bits, iters, success, fL, fE,
                         counters, stream);
}

int qkd_score_batch(const qkd_code* c, int64_t F, const uint8_t* bits, const uint8_t* x, const uint8_t* success,
                    int32_t* errors, int64_t* counters, void* stream) {
    if (!c || F < 0 || (F > 0 && (!bits || !x || !success))) return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    const int nb8 = (int)((c->n + 7) / 8);
    const int grid = (int)std::min<long long>(F, 148LL * 16);
    score_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(nb8, F, bits, x, c->d_payload, success, errors,
                                                         reinterpret_cast<unsigned long long*>(counters));
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

size_t qkd_reconcile_device_bytes(const qkd_code* c, int64_t F) {
    if (!c || F < 0) return 0;
    const size_t nb8 = (size_t)((c->n + 7) / 8), mb8 = (size_t)((c->m + 7) / 8);
    size_t s = 0;
    s += align256(F * nb8);                   // Bob's bits
    s += c->has_short ? align256(F * nb8) : 0;   // known bits
    s += align256(F * mb8);                   // syndrome
    s += align256(F * (size_t)c->n);          // llr
    s += align256(F * nb8);                   // bits out
    s += align256(F * 4);                     // iters
    s += align256(F);                         // success
    return s + align256(qkd_workspace_bytes(c, F));
}

int qkd_reconcile_host(const qkd_code* c, double qber, int64_t F, const uint8_t* y_h, const uint8_t* known_h,
                       const uint8_t* syn_h, int32_t max_iter, int32_t early_stop, void* dbuf, size_t dbytes,
                       uint8_t* bits_h, int32_t* iters_h, uint8_t* succ_h, void* stream) {
    if (!c || F < 0) return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    if (!y_h || !syn_h || !bits_h || !iters_h || !succ_h || !dbuf) return fail(QKD_EINVAL, "null buffer");
    if (c->has_short && !known_h) return fail(QKD_EINVAL, "known bits required (shortened positions)");
    const size_t need = qkd_reconcile_device_bytes(c, F);
    if (need == 0 || dbytes < need) return fail(QKD_EDIM, "device buffer too small: need " + std::to_string(need));
    const size_t nb8 = (size_t)((c->n + 7) / 8), mb8 = (size_t)((c->m + 7) / 8);
    char* w = static_cast<char*>(dbuf);
    uint8_t* d_y = (uint8_t*)w; w += align256(F * nb8);
    uint8_t* d_k = nullptr;
    if (c->has_short) { d_k = (uint8_t*)w; w += align256(F * nb8); }
    uint8_t* d_s = (uint8_t*)w; w += align256(F * mb8);
    int8_t* d_llr = (int8_t*)w; w += align256(F * (size_t)c->n);
    uint8_t* d_b = (uint8_t*)w; w += align256(F * nb8);
    int32_t* d_it = (int32_t*)w; w += align256(F * 4);
    uint8_t* d_su = (uint8_t*)w; w += align256(F);
    const size_t wsb = qkd_workspace_bytes(c, F);
    cudaStream_t st = (cudaStream_t)stream;
    // Pipelined in K chunks of frames: copies in on one stream, LLR + decode on the caller's stream,
    // copies out on a third, chained by events, so chunk c's decode overlaps chunk c+1's host->device
    // and chunk c-1's device->host transfers.  Chunks keep >= ~16 waves of frame groups each (tail
    // effect per launch), at most 8 of them.
    Plan pl;
    int rc = make_plan(c, F, pl);
    if (rc) return rc;
    const long long per_wave = std::max<long long>(1, pl.slots) * kFramesPerGroup;
    const int K = (int)std::max<long long>(1, std::min<long long>(ReconcileCtx::kMaxChunks, F / (16 * per_wave)));
    qkd_code* cm = const_cast<qkd_code*>(c);
    ReconcileCtx* x = nullptr;   // a context of this handle not used by a concurrent call
    {
        std::lock_guard<std::mutex> lk(cm->mu);
        if (!cm->ctx_free.empty()) {
            x = cm->ctx_free.back();
            cm->ctx_free.pop_back();
        }
    }
    if (!x) {
        x = new ReconcileCtx();
        if (!x->ok) {
            delete x;
            return fail(QKD_ECUDA, "cannot create the reconcile streams/events");
        }
    }
    auto release = [&]() {
        std::lock_guard<std::mutex> lk(cm->mu);
        cm->ctx_free.push_back(x);
    };
    auto ck = [&](cudaError_t e, const char* what) -> int {
        if (e == cudaSuccess) return QKD_OK;
        release();
        return fail(QKD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    // the copies into dbuf must not overtake work already queued on the caller's stream (it may
    // still be reading a previous use of this buffer): s_in starts behind it
    if ((rc = ck(cudaEventRecord(x->entry, st), "event"))) return rc;
    if ((rc = ck(cudaStreamWaitEvent(x->s_in, x->entry, 0), "wait"))) return rc;
    if ((rc = ck(cudaStreamWaitEvent(x->s_out, x->entry, 0), "wait"))) return rc;
    for (int k = 0; k < K; ++k) {   // all host->device copies, in chunk order
        const long long a = F * k / K, n_k = F * (k + 1) / K - a;
        if ((rc = ck(cudaMemcpyAsync(d_y + a * nb8, y_h + a * nb8, n_k * nb8, cudaMemcpyHostToDevice, x->s_in), "h2d"))) return rc;
        if (d_k && (rc = ck(cudaMemcpyAsync(d_k + a * nb8, known_h + a * nb8, n_k * nb8, cudaMemcpyHostToDevice, x->s_in), "h2d")))
            return rc;
        if ((rc = ck(cudaMemcpyAsync(d_s + a * mb8, syn_h + a * mb8, n_k * mb8, cudaMemcpyHostToDevice, x->s_in), "h2d"))) return rc;
        if ((rc = ck(cudaEventRecord(x->ev[2 * k], x->s_in), "event"))) return rc;
    }
    for (int k = 0; k < K; ++k) {
        const long long a = F * k / K, n_k = F * (k + 1) / K - a;
        if ((rc = ck(cudaStreamWaitEvent(st, x->ev[2 * k], 0), "wait"))) return rc;
        rc = qkd_build_llr(c, qber, n_k, d_y + a * nb8, d_k ? d_k + a * nb8 : nullptr, d_llr + a * (long long)c->n, stream);
        if (!rc)
            rc = qkd_decode_batch(c, n_k, d_llr + a * (long long)c->n, d_s + a * mb8, max_iter, early_stop, w, wsb,
                                  d_b + a * nb8, d_it + a, d_su + a, nullptr, nullptr, nullptr, stream);
        if (rc) { release(); return rc; }
        if ((rc = ck(cudaEventRecord(x->ev[2 * k + 1], st), "event"))) return rc;
        if ((rc = ck(cudaStreamWaitEvent(x->s_out, x->ev[2 * k + 1], 0), "wait"))) return rc;
        if ((rc = ck(cudaMemcpyAsync(bits_h + a * nb8, d_b + a * nb8, n_k * nb8, cudaMemcpyDeviceToHost, x->s_out), "d2h")))
            return rc;
        if ((rc = ck(cudaMemcpyAsync(iters_h + a, d_it + a, n_k * 4, cudaMemcpyDeviceToHost, x->s_out), "d2h"))) return rc;
        if ((rc = ck(cudaMemcpyAsync(succ_h + a, d_su + a, n_k, cudaMemcpyDeviceToHost, x->s_out), "d2h"))) return rc;
    }
    if ((rc = ck(cudaStreamSynchronize(x->s_out), "sync"))) return rc;
    if ((rc = ck(cudaStreamSynchronize(st), "sync"))) return rc;
    release();
    return QKD_OK;
}

size_t qkd_adaptive_work_bytes(const qkd_code* c, int64_t F) {
    if (!c || F < 0) return 0;
    const size_t nb8 = (size_t)((c->n + 7) / 8), mb8 = (size_t)((c->m + 7) / 8), Fs = (size_t)std::max<int64_t>(F, 1);
    const size_t ws = qkd_workspace_bytes(c, Fs);
    if (ws == 0) return 0;
    return align256((size_t)c->n) + 2 * align256(Fs * 4) + 256 + 3 * align256(Fs * nb8) + align256(Fs * mb8) +
           align256(Fs * (size_t)c->n) + align256(Fs * 4) + align256(Fs) + align256(ws);
}

int qkd_reconcile_adaptive(const qkd_code* c, double qber, int64_t F, const int32_t* order, int64_t d, int64_t s0,
                           int64_t delta, int32_t max_rounds, const uint8_t* bob, const uint8_t* alice,
                           const uint8_t* syn, int32_t max_iter, void* work, size_t work_bytes, uint8_t* bits,
                           int32_t* iters, int32_t* rounds, uint8_t* success, void* stream) {
    if (!c || F < 0 || d < 0 || d > c->n || s0 < 0 || s0 > d || delta < 1 || max_rounds < 0 || max_iter < 0)
        return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    if ((d > 0 && !order) || !bob || !alice || !syn || !work || !bits || !iters || !rounds || !success)
        return fail(QKD_EINVAL, "null buffer");
    const int Lq = qkd_llr_magnitude(qber);
    if (Lq < 0) return Lq;
    const size_t need = qkd_adaptive_work_bytes(c, F);
    if (need == 0 || work_bytes < need) return fail(QKD_EDIM, "work buffer too small: need " + std::to_string(need));
    const int nb8 = (int)((c->n + 7) / 8), mb8 = (int)((c->m + 7) / 8);
    char* w = static_cast<char*>(work);
    uint8_t* kind = (uint8_t*)w; w += align256((size_t)c->n);
    int32_t* idx_a = (int32_t*)w; w += align256((size_t)F * 4);   // active frame ids, double-buffered
    int32_t* idx_b = (int32_t*)w; w += align256((size_t)F * 4);
    long long* cnt = (long long*)w; w += 256;                     // cnt[0], cnt[1]: their lengths
    uint8_t* g_bob = (uint8_t*)w; w += align256((size_t)F * nb8);
    uint8_t* g_known = (uint8_t*)w; w += align256((size_t)F * nb8);
    uint8_t* c_bits = (uint8_t*)w; w += align256((size_t)F * nb8);
    uint8_t* g_syn = (uint8_t*)w; w += align256((size_t)F * mb8);
    int8_t* llr = (int8_t*)w; w += align256((size_t)F * (size_t)c->n);
    int32_t* c_iters = (int32_t*)w; w += align256((size_t)F * 4);
    uint8_t* c_succ = (uint8_t*)w; w += align256((size_t)F);
    const size_t wsb = qkd_workspace_bytes(c, F);
    cudaStream_t st = (cudaStream_t)stream;
    // Every round is enqueued without a host synchronisation: the list of still-failed frames and its
    // length stay on the device (compact_failed_kernel), each kernel reads the length there, and the
    // decode launch is planned for F and decodes the first *cnt frames.  A round whose list is empty
    // costs a few empty launches.
    const int g = (int)std::min<long long>(F, 148LL * 16);
    init_active_kernel<<<(int)std::min<long long>((F + 255) / 256, 148LL * 8), 256, 0, st>>>(idx_a, F, cnt);
    QKD_CK(cudaGetLastError());
    int32_t* cur = idx_a;
    int32_t* nxt = idx_b;
    long long* ccur = cnt;
    long long* cnxt = cnt + 1;
    long long s_prev = -1;
    for (int k = 0; k <= max_rounds; ++k) {
        const long long sk = std::min<long long>(s0 + (long long)k * delta, d);
        if (sk == s_prev) break;                               // nothing left to reveal
        const bool last = (k == max_rounds) || (sk == d);
        s_prev = sk;
        QKD_CK(cudaMemsetAsync(kind, 0, (size_t)c->n, st));
        if (d > 0) {
            reveal_kind_kernel<<<(int)std::min<long long>((d + 255) / 256, 148LL * 8), 256, 0, st>>>(order, d, sk,
                                                                                                   (int)c->n, kind);
            QKD_CK(cudaGetLastError());
        }
        gather_rows_kernel<<<g, 256, 0, st>>>(cur, ccur, bob, nb8, g_bob);
        gather_rows_kernel<<<g, 256, 0, st>>>(cur, ccur, alice, nb8, g_known);
        gather_rows_kernel<<<g, 256, 0, st>>>(cur, ccur, syn, mb8, g_syn);
        const long long total = F * (long long)nb8;
        build_llr_kernel<<<(int)std::min<long long>((total + 255) / 256, 148LL * 64), 256, 0, st>>>(
            (int)c->n, nb8, F, Lq, g_bob, g_known, kind, llr, ccur);
        QKD_CK(cudaGetLastError());
        int rc = decode_launch(c, F, ccur, llr, g_syn, max_iter, 1, w, wsb, c_bits, c_iters, c_succ, nullptr,
                               nullptr, nullptr, stream);
        if (rc) return rc;
        scatter_results_kernel<<<g, 256, 0, st>>>(cur, ccur, nb8, k, last ? 1 : 0, c_bits, c_iters, c_succ, bits,
                                                  iters, rounds, success);
        QKD_CK(cudaGetLastError());
        if (last) break;
        compact_failed_kernel<<<1, kCompactThreads, 0, st>>>(cur, ccur, c_succ, nxt, cnxt);
        QKD_CK(cudaGetLastError());
        std::swap(cur, nxt);
        std::swap(ccur, cnxt);
    }
    return QKD_OK;
}

// ---- exact floating-point BP ---------------------------------------
struct FPlan {
    bool esm = false;
    int fd = 20;   // register-array size of the row update: 20 or 32 (kFloatDMax)
    int TG = 0, GPC = 0, grid = 0, smem = 0, slot_bytes = 0, e_bytes = 0, tab_off = 0;
    long long slots = 0;
    size_t ws_total = 0;
};

static const void* fkernel(bool esm, bool flood, int fd) {
    if (fd <= 20)
        return esm ? (flood ? reinterpret_cast<const void*>(&decode_float_kernel<true, true, 20>)
                            : reinterpret_cast<const void*>(&decode_float_kernel<true, false, 20>))
                   : (flood ? reinterpret_cast<const void*>(&decode_float_kernel<false, true, 20>)
                            : reinterpret_cast<const void*>(&decode_float_kernel<false, false, 20>));
    return esm ? (flood ? reinterpret_cast<const void*>(&decode_float_kernel<true, true, kFloatDMax>)
                        : reinterpret_cast<const void*>(&decode_float_kernel<true, false, kFloatDMax>))
               : (flood ? reinterpret_cast<const void*>(&decode_float_kernel<false, true, kFloatDMax>)
                        : reinterpret_cast<const void*>(&decode_float_kernel<false, false, kFloatDMax>));
}

static int make_fplan(const qkd_code* c, long long F, FPlan& pl) {
    if (c->maxdeg > kFloatDMax) return fail(QKD_EUNSUP, "float decoder: check degree > 32");
    int dev = 0;
    QKD_CK(cudaGetDevice(&dev));
    const DevInfo di = dev_info(dev);
    if (!di.ok) return fail(QKD_ECUDA, "cannot query device attributes");
    const long long tab = (long long)c->Mb * sizeof(int4) + (long long)c->nbase * sizeof(int2);
    const long long syn_ctl = ((c->m + 15) & ~15LL) + 16;
    pl.esm = 4LL * c->n + syn_ctl + tab <= di.smem_optin;
    pl.e_bytes = pl.esm ? (int)(4LL * c->n) : 0;
    pl.slot_bytes = (int)((pl.e_bytes + syn_ctl + 15) & ~15LL);
    if (pl.slot_bytes + tab > di.smem_optin) return fail(QKD_EUNSUP, "float decoder: frame too long");
    pl.TG = (int)std::min<long long>(((long long)c->Z + 31) / 32 * 32, 512);
    int gpc = std::max(1, 1024 / pl.TG);
    while (gpc > 1 && (long long)gpc * pl.slot_bytes + tab > di.smem_optin) --gpc;
    gpc = (int)std::max<long long>(1, std::min<long long>(gpc, (F + di.sms - 1) / di.sms));
    pl.GPC = gpc;
    pl.tab_off = gpc * pl.slot_bytes;
    pl.smem = pl.tab_off + (int)tab;
    pl.fd = c->maxdeg <= 20 ? 20 : kFloatDMax;
    for (const void* k : {fkernel(true, false, pl.fd), fkernel(true, true, pl.fd), fkernel(false, false, pl.fd),
                          fkernel(false, true, pl.fd)})
        QKD_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
    const void* k = fkernel(pl.esm, false, pl.fd);
    int per_sm = 0;
    QKD_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, pl.TG * pl.GPC, pl.smem));
    if (per_sm < 1) return fail(QKD_EUNSUP, "float decoder cannot be resident with this geometry");
    const long long ctas = (F + gpc - 1) / gpc;
    pl.grid = (int)std::max<long long>(1, std::min<long long>(ctas, (long long)per_sm * di.sms));
    pl.slots = (long long)pl.grid * gpc;
    pl.ws_total = 256 + (size_t)pl.slots * (size_t)c->ws_words * 4 + (pl.esm ? 0 : (size_t)pl.slots * c->n * 4);
    return QKD_OK;
}

size_t qkd_float_workspace_bytes(const qkd_code* c, int64_t F) {
    if (!c || F < 0) return 0;
    FPlan pl;
    if (make_fplan(c, std::max<int64_t>(F, 1), pl) != QKD_OK) return 0;
    return pl.ws_total;
}

int qkd_build_llr_float(const qkd_code* c, double qber, int64_t F, const uint8_t* y, const uint8_t* known,
                        float* llr, void* stream) {
    if (!c || F < 0 || (F > 0 && (!y || !llr))) return fail(QKD_EINVAL, "bad argument");
    if (!(qber > 0.0 && qber < 0.5)) return fail(QKD_EINVAL, "qber must lie in (0, 0.5)");
    if (c->has_short && !known) return fail(QKD_EINVAL, "code has shortened positions: known_bits required");
    if (F == 0) return QKD_OK;
    const float Lc = (float)std::log((1.0 - qber) / qber);
    const long long total = F * c->n;
    build_llr_float_kernel<<<(int)std::min<long long>((total + 255) / 256, 148LL * 64), 256, 0, (cudaStream_t)stream>>>(
        (int)c->n, (int)((c->n + 7) / 8), F, Lc, y, c->d_kind ? known : nullptr, c->d_kind, llr);
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

int qkd_decode_float_batch(const qkd_code* c, int64_t F, const float* llr, const uint8_t* syn, int32_t max_iter,
                           int32_t early_stop, int32_t schedule, void* ws, size_t ws_bytes, uint8_t* bits,
                           int32_t* iters, uint8_t* success, float* fL, float* fE, void* stream) {
    if (!c || F < 0 || max_iter < 0 || schedule < 0 || schedule > 1) return fail(QKD_EINVAL, "bad argument");
    if (F == 0) return QKD_OK;
    if (!llr || !syn || !ws || !bits || !iters || !success) return fail(QKD_EINVAL, "null buffer");
    FPlan pl;
    int rc = make_fplan(c, F, pl);
    if (rc) return rc;
    if (ws_bytes < pl.ws_total)
        return fail(QKD_EDIM, "workspace too small: need " + std::to_string(pl.ws_total) + " bytes");
    char* w = static_cast<char*>(ws);
    FParams p{};
    p.layer = c->d_layer;
    p.edge = c->d_edge;
    p.Mb = c->Mb;
    p.Z = c->Z;
    p.nbase = c->nbase;
    p.n = (int)c->n;
    p.m = (int)c->m;
    p.mb8 = (int)((c->m + 7) / 8);
    p.nb8 = (int)((c->n + 7) / 8);
    p.n_edges = c->n_edges;
    p.ws_words = c->ws_words;
    p.llr = llr;
    p.syn = syn;
    p.F = F;
    p.T = max_iter;
    p.early_stop = early_stop ? 1 : 0;
    p.work = reinterpret_cast<int*>(w);
    p.Lws = reinterpret_cast<float*>(w + 256);
    p.Ews = pl.esm ? nullptr : reinterpret_cast<float*>(w + 256 + (size_t)pl.slots * (size_t)c->ws_words * 4);
    p.bits = bits;
    p.iters = iters;
    p.success = success;
    p.fL = fL;
    p.fE = fE;
    p.TG = pl.TG;
    p.GPC = pl.GPC;
    p.slot_bytes = pl.slot_bytes;
    p.e_bytes = pl.e_bytes;
    p.tab_off = pl.tab_off;
    cudaStream_t st = (cudaStream_t)stream;
    QKD_CK(cudaMemsetAsync(p.work, 0, sizeof(int), st));
    void* args[] = {&p};
    const void* k = fkernel(pl.esm, schedule != 0, pl.fd);
    QKD_CK(cudaLaunchKernel(k, dim3(pl.grid), dim3(pl.TG * pl.GPC), args, pl.smem, st));
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

int qkd_tau_table(uint8_t* out, void* stream) {
    if (!out) return fail(QKD_EINVAL, "null buffer");
    tau_table_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(out, runtime_konst());
    QKD_CK(cudaGetLastError());
    return QKD_OK;
}

}  // extern "C"
