/*
 * qkd_ldpc.h -- C ABI of the B200-native (sm_100a) batched quantized LDPC syndrome
 * decoder for QKD information reconciliation, after arXiv:1903.10107
 * ("High Throughput and Low Cost LDPC Reconciliation for Quantum Key Distribution").
 *
 * Citations: PAPER.md line numbers as P:<n> (the paper's LaTeX), SPEC.md as S:<n>;
 * R<k> = the reading of the paper recorded in DESIGN.md §3 where the paper is silent.
 *
 * Conventions common to every entry point
 *   - Return value: QKD_OK (0) or a negative QKD_E* code.  qkd_last_error() then returns a
 *     thread-local, human-readable message.  No C++ exception crosses this boundary.
 *   - "_dev" pointers are CUDA device pointers on the current device; "_host" pointers are
 *     host memory (pinned memory gives asynchronous copies).  The caller owns every buffer;
 *     the library allocates only inside qkd_code_create (the code tables).
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).  Device
 *     work is asynchronous on that stream; outputs are valid after the stream completes.
 *   - Bit arrays are packed LSB-first: bit j of a frame is bit (j % 8) of byte j / 8;
 *     a frame of n bits occupies ceil(n/8) bytes and frames are contiguous.
 *   - Frames are independent: every per-frame result depends only on that frame's own
 *     inputs (not on batch size, position in the batch, stream or rank).
 */
#ifndef QKD_LDPC_H
#define QKD_LDPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QKD_OK 0
#define QKD_EINVAL (-1) /* bad argument (NULL pointer, qber outside (0,0.5), max_iter < 0) */
#define QKD_EDIM (-2)   /* dimension mismatch / too small workspace */
#define QKD_ESHIFT (-3) /* base-matrix shift outside [-1, Z) */
#define QKD_ECUDA (-4)  /* a CUDA runtime call failed */
#define QKD_ENOMEM (-5) /* allocation of the code tables failed */
#define QKD_EUNSUP (-6) /* structure beyond the kernels' limits (check degree > 64) */

typedef struct qkd_code qkd_code;

/*
 * Create a QC-LDPC code ("a base matrix of size Mb x Nb. Each element of the base
 * matrix is a sub-matrix with the expansion-factor Z. Each nonzero entry is replaced by a
 * cyclically shifted identity matrix while each zero entry is replaced by a all-zero
 * matrix").  Block (I,J) with shift s contributes the edges (I*Z + r, J*Z + (r+s) mod Z),
 * r = 0..Z-1 (R14).  One circulant per base entry (R15).
 *   base_shifts : host, Mb*Nb int32 row-major; -1 = zero block, else a shift in [0, Z).
 *   pos_kind    : host, n = Nb*Z bytes, or NULL (all payload).  0 = payload, 1 = punctured
 *                 (channel LLR 0), 2 = shortened (LLR +-127 from the known bit).  The
 *                 rate-adaptive positions of P:157.
 *   out         : receives the handle; immutable afterwards and shareable between threads
 *                 and streams.  Tables are uploaded to the current device.
 * Errors: QKD_EINVAL (Mb < 1, Nb <= Mb, Z < 1, NULL), QKD_ESHIFT (names the block in
 * qkd_last_error), QKD_EUNSUP (a block row with more than 64 non-zero blocks), QKD_ECUDA.
 */
int qkd_code_create(const int32_t* base_shifts, int32_t Mb, int32_t Nb, int32_t Z,
                    const uint8_t* pos_kind, qkd_code** out);
void qkd_code_destroy(qkd_code* code);

/* n = Nb*Z variables, m = Mb*Z checks, n_edges = (non-zero base entries)*Z, and the largest
 * check-node degree ("degCN_i"). Any output pointer may be NULL. */
int qkd_code_info(const qkd_code* code, int64_t* n, int64_t* m, int64_t* n_edges,
                  int32_t* max_row_deg);

/* Quantized channel-LLR magnitude of a BSC with crossover qber: min(127, round(4 ln((1-q)/q)))
 * (P:103-112 8-bit quantization; step 1/4 = R1, round-to-nearest = R2; BASELINE configs[0]).
 * Returns the magnitude (0..127) or QKD_EINVAL if qber is not in (0, 0.5). */
int qkd_llr_magnitude(double qber);

/* Alice's syndrome s = H x.  bits_dev [F][ceil(n/8)] -> syn_dev [F][ceil(m/8)]. */
int qkd_syndrome(const qkd_code* code, int64_t n_frames, const uint8_t* bits_dev,
                 uint8_t* syn_dev, void* stream);

/* Bob's int8 channel LLRs: payload bit y -> +Lq (y=0) / -Lq (y=1);
 * punctured -> 0; shortened -> +127 if the known bit is 0 else -127.
 *   bob_bits_dev   [F][ceil(n/8)]  Bob's sifted key bits
 *   known_bits_dev [F][ceil(n/8)]  bits known at shortened positions; may be NULL when the
 *                                  code has no shortened position
 *   llr_dev        [F][n] int8 out */
int qkd_build_llr(const qkd_code* code, double qber, int64_t n_frames,
                  const uint8_t* bob_bits_dev, const uint8_t* known_bits_dev, int8_t* llr_dev,
                  void* stream);

/* Device workspace (bytes) qkd_decode_batch needs for n_frames on the current device: the
 * int8 check-to-variable messages of the frame groups in flight ("only the latest E_j
 * and L_ij are stored") plus a work counter.  Bounded by the number of resident frame
 * groups, not by n_frames. */
size_t qkd_workspace_bytes(const qkd_code* code, int64_t n_frames);

/*
 * Decode a batch with the paper's quantized decoder: layered schedule over block rows in
 * order (R13); check nodes by the improved RCBP rule tau of Algorithm 1
 * with the leave-one-out reduction of Eq.(4)/(7) done by the forward/backward schedule in
 * ascending block column (R6) and the target-syndrome bit folded into the sign of Eq.(1)
 * (R5); variable nodes by Eq.(8)/(9) with the saturation rule of Algorithm 2 (P:138-147,
 * E_max = 127, MSG_max = 63); stopping criterion of P:99 checked before iteration 1 and
 * after every full iteration (R10, R11).
 *   llr_dev      [F][n] int8, |v| <= 127            (channel LLRs, e.g. qkd_build_llr)
 *   syndrome_dev [F][ceil(m/8)]                     (Alice's syndrome)
 *   max_iter     ITER_max >= 0
 *   early_stop   1: stop a frame at its first syndrome match;  0: run exactly max_iter
 *                iterations and report success = (syndrome matched after the last one)
 *   workspace    >= qkd_workspace_bytes(code, F) bytes of device memory (contents ignored)
 * Outputs (device):
 *   bits_dev     [F][ceil(n/8)]  hard decisions, bit = (E_j < 0) (R9)
 *   iters_dev    [F] int32       completed iterations at the stop (0 = matched on input)
 *   success_dev  [F] uint8       1 iff the syndrome matched
 *   final_L_dev  [F][n_edges] int8 or NULL: L_ij at the stop, canonical edge order
 *                (block row I ascending, then block column J ascending, then row r:
 *                index (slot_base(I) + k) * Z + r)
 *   final_E_dev  [F][n] int8 or NULL: E_j at the stop
 *   counters_dev int64[5] or NULL, accumulated (+=): [0] frames, [1] successes,
 *                [4] sum of iterations ([2], [3] are qkd_score_batch's).
 * Errors: QKD_EINVAL, QKD_EDIM (workspace too small), QKD_ECUDA.
 */
int qkd_decode_batch(const qkd_code* code, int64_t n_frames, const int8_t* llr_dev,
                     const uint8_t* syndrome_dev, int32_t max_iter, int32_t early_stop,
                     void* workspace_dev, size_t workspace_bytes, uint8_t* bits_dev,
                     int32_t* iters_dev, uint8_t* success_dev, int8_t* final_L_dev,
                     int8_t* final_E_dev, int64_t* counters_dev, void* stream);

/* Harness scoring against Alice's key ("there may exist undetected errors"): for each
 * frame, bit errors on payload positions (pos_kind == 0) between bits_dev and alice_bits_dev;
 * counters_dev[2] += frames with >= 1 error, counters_dev[3] += successful frames with >= 1
 * error (undetected).  Optional per-frame error counts to errors_dev (int32 [F], may be NULL). */
int qkd_score_batch(const qkd_code* code, int64_t n_frames, const uint8_t* bits_dev,
                    const uint8_t* alice_bits_dev, const uint8_t* success_dev,
                    int32_t* errors_dev, int64_t* counters_dev, void* stream);

/* End-to-end call with HOST buffers: copies Bob's bits, the known (shortened) bits and
 * Alice's syndrome host->device, builds the LLRs, decodes and copies bits/iters/success back
 * (device->host); returns when everything has completed.  The batch is pipelined in chunks: the
 * copies run on two internal streams chained by events to `stream`, which builds and decodes, so
 * transfers overlap decoding (host buffers should be pinned for that).
 * device_buffer must hold qkd_reconcile_device_bytes(code, F) bytes. */
size_t qkd_reconcile_device_bytes(const qkd_code* code, int64_t n_frames);
int qkd_reconcile_host(const qkd_code* code, double qber, int64_t n_frames,
                       const uint8_t* bob_bits_host, const uint8_t* known_bits_host,
                       const uint8_t* syndrome_host, int32_t max_iter, int32_t early_stop,
                       void* device_buffer, size_t device_buffer_bytes, uint8_t* bits_host,
                       int32_t* iters_host, uint8_t* success_host, void* stream);

/* Interactive rate-adaptive reconciliation ("the shortened bits are
 * selected in turn from the puncturing bits when addition information revealing is
 * necessary", "multi-interaction is an essential step"; SPEC bob_attempt /
 * alice_reveal; reading R25 of DESIGN.md).
 *   order_dev  int32 [d]: the reserved positions in reveal order (DESIGN R19: column weight
 *              ascending, seeded ties).  Round k (k = 0..max_rounds) treats order[0, s_k) as
 *              shortened (known, LLR +-127 from alice_bits) and order[s_k, d) as punctured
 *              (LLR 0), s_k = min(s0 + k * delta, d); every other position is payload.
 *   Round 0 decodes all frames; round k > 0 re-decodes, from a fresh state, only the frames
 *   that have not matched their syndrome yet (gathered into a compact batch); the rounds
 *   stop early when every frame matched or nothing is left to reveal.
 *   Per frame outputs: bits/iters/success of the round at which it matched (else of the last
 *   round it ran), rounds_dev = that round index k.  Leakage of a frame that stopped at
 *   round k: m - (d - s_k) syndrome-and-reveal bits (host side: R20 with p = d - s_k).
 *   bob_bits_dev, alice_bits_dev [F][ceil(n/8)], syndrome_dev [F][ceil(m/8)] are read only.
 *   work_dev: qkd_adaptive_work_bytes(code, F) bytes.  The code handle's own pos_kind is
 *   ignored (the rounds set the pattern).  Asynchronous: the list of still-failed frames is
 *   compacted on the device and every round is enqueued on `stream` without a host
 *   synchronisation (rounds after all frames matched cost a few empty launches).
 * Errors: QKD_EINVAL (d < 0, s0 outside [0, d], delta < 1, max_rounds < 0, NULL), QKD_EDIM
 * (work buffer too small), QKD_ECUDA. */
size_t qkd_adaptive_work_bytes(const qkd_code* code, int64_t n_frames);
int qkd_reconcile_adaptive(const qkd_code* code, double qber, int64_t n_frames,
                           const int32_t* order_dev, int64_t d, int64_t s0, int64_t delta,
                           int32_t max_rounds, const uint8_t* bob_bits_dev, const uint8_t* alice_bits_dev,
                           const uint8_t* syndrome_dev, int32_t max_iter, void* work_dev,
                           size_t work_bytes, uint8_t* bits_dev, int32_t* iters_dev,
                           int32_t* rounds_dev, uint8_t* success_dev, void* stream);

/* Exact floating-point layered BP (R26): the reference decoder the
 * quantized path is compared with ("maintain the high efficiency as the floating-point
 * version").  Check node Eq.(1) + Eq.(2)/(4) with the box-plus of Eq.(6)/(7) (forward/backward
 * schedule of R6, beta in R26's stable form), variable node Eq.(8)/(9) without saturation, the
 * same layered schedule and stopping rule as qkd_decode_batch; fp32 throughout.
 * qkd_build_llr_float: llr_dev float [F][n] = +-ln((1-q)/q) by Bob's bit, 0 punctured, +-1000 for
 *   shortened positions (known_bits required when the code has them).
 * qkd_decode_float_batch: like qkd_decode_batch with float LLRs; final_L_dev (float [F][n_edges],
 *   canonical order) and final_E_dev (float [F][n]) optional.  Check degrees <= 32.
 *   schedule 0 = layered (the paper's); 1 = flooding: every iteration all
 *   check nodes from the previous state, then E_j = LLR_j + sum_i L_ij (float atomics, so the
 *   summation order -- and the last bits of E -- vary from run to run).
 * Errors: QKD_EINVAL, QKD_EDIM (workspace too small), QKD_EUNSUP (check degree > 32), QKD_ECUDA. */
int qkd_build_llr_float(const qkd_code* code, double qber, int64_t n_frames, const uint8_t* bob_bits_dev,
                        const uint8_t* known_bits_dev, float* llr_dev, void* stream);
size_t qkd_float_workspace_bytes(const qkd_code* code, int64_t n_frames);
int qkd_decode_float_batch(const qkd_code* code, int64_t n_frames, const float* llr_dev,
                           const uint8_t* syndrome_dev, int32_t max_iter, int32_t early_stop, int32_t schedule,
                           void* workspace_dev, size_t workspace_bytes, uint8_t* bits_dev, int32_t* iters_dev,
                           uint8_t* success_dev, float* final_L_dev, float* final_E_dev, void* stream);

/* Launch geometry chosen for (code, F) on the current device:
 * info[0] kernel variant (1: degree<=8 smem, 2: degree<=20 smem, 3: generic smem,
 * 4: generic with E in global memory, 5: degree 9..20 lane-pair rows (QKD_SPLIT=1 at
 * code creation), 6: degree 21..32 smem, one row per thread, 7: degree <= 8 with E in global memory,
 * register rows, 8: degree 9..32 with E in global memory, register rows; +10 when Z is a power of two), [1] threads per frame group, [2] frame groups per
 * CTA, [3] grid, [4] dynamic shared bytes per CTA, [5] frames per group (4), [6] groups. */
int qkd_launch_info(const qkd_code* code, int64_t n_frames, int32_t* info);

/* Self-test of the device tau arithmetic: out_dev[64*64] = tau(p, q) for p, q in [0, 63]
 * computed by the decode kernels' packed-byte implementation of Algorithm 1. */
int qkd_tau_table(uint8_t* out_dev, void* stream);

const char* qkd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* QKD_LDPC_H */
