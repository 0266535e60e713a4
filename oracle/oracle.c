/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  A plain, slow, scalar CPU implementation of the
 * quantized layered RCBP syndrome decoder of arXiv:1903.10107 (PAPER.md = "P:<line>").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or constant with the CUDA path
 * (paper_1903_10107_b200/csrc); its only inputs are the base matrix, LLR/bit arrays and
 * syndromes.  Every function cites the passage it follows.  Readings of the paper where it
 * is silent are DESIGN.md §3 (R1..R21, = SURVEY.md §8(c) Q1..Q21).
 *
 * Integer arithmetic throughout (the method is integer-only once the channel LLR is
 * quantized); the only floating point is the one-off LLR magnitude log (R1, R2) and the
 * efficiency report (R20).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MSG_MAX 63   /* P:118 "if the input p and q are 6-bit input, MSG_max is set as 63" (R3) */
#define E_MAX 127    /* P:137 "the value of E_max is set as 127" */

/* ------------------------------------------------------------------------- */
/* Code: QC expansion ("Each nonzero entry is replaced by a cyclically shifted    */
/* identity matrix"; circulant convention column = J*Z + (r+s) mod Z, R14).              */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t Mb, Nb, Z;
    int64_t n, m, n_edges;
    int32_t* deg;        /* [Mb] number of non-zero blocks in block row I */
    int32_t* bJ;         /* [base edges] block column, block-row major, ascending J */
    int32_t* bS;         /* [base edges] shift */
    int32_t* slot_base;  /* [Mb+1] prefix sum of deg */
} orc_code;

void orc_code_destroy(orc_code* c);

/* returns NULL on invalid input (shift out of range, Nb <= Mb, Z < 1) */
orc_code* orc_code_create(const int32_t* shifts, int32_t Mb, int32_t Nb, int32_t Z) {
    if (Mb < 1 || Nb <= Mb || Z < 1) return NULL;
    for (int64_t i = 0; i < (int64_t)Mb * Nb; i++)
        if (shifts[i] < -1 || shifts[i] >= Z) return NULL;
    orc_code* c = (orc_code*)calloc(1, sizeof(orc_code));
    c->Mb = Mb; c->Nb = Nb; c->Z = Z;
    c->n = (int64_t)Nb * Z; c->m = (int64_t)Mb * Z;
    c->deg = (int32_t*)calloc(Mb, sizeof(int32_t));
    c->slot_base = (int32_t*)calloc(Mb + 1, sizeof(int32_t));
    int nb = 0;
    for (int I = 0; I < Mb; I++) for (int J = 0; J < Nb; J++) if (shifts[I * Nb + J] >= 0) nb++;
    c->bJ = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    c->bS = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
    int e = 0;
    for (int I = 0; I < Mb; I++) {
        c->slot_base[I] = e;
        for (int J = 0; J < Nb; J++) {
            int s = shifts[I * Nb + J];
            if (s >= 0) { c->bJ[e] = J; c->bS[e] = s; e++; c->deg[I]++; }
        }
    }
    c->slot_base[Mb] = e;
    c->n_edges = (int64_t)e * Z;
    for (int I = 0; I < Mb; I++) if (c->deg[I] > 256) { orc_code_destroy(c); return NULL; }
    return c;
}

void orc_code_destroy(orc_code* c) {
    if (!c) return;
    free(c->deg); free(c->bJ); free(c->bS); free(c->slot_base); free(c);
}

int64_t orc_code_n(const orc_code* c) { return c->n; }
int64_t orc_code_m(const orc_code* c) { return c->m; }
int64_t orc_code_edges(const orc_code* c) { return c->n_edges; }

/* column of the k-th edge of check row i (k in ascending block column) */
static inline int64_t col_of(const orc_code* c, int I, int r, int k) {
    int b = c->slot_base[I] + k;
    return (int64_t)c->bJ[b] * c->Z + (r + c->bS[b]) % c->Z;
}

/* canonical edge index: (slot_base(I) + k) * Z + r */
static inline int64_t edge_of(const orc_code* c, int I, int r, int k) {
    return (int64_t)(c->slot_base[I] + k) * c->Z + r;
}

/* H as an explicit edge list in canonical order: rows_out/cols_out [n_edges] */
void orc_expand(const orc_code* c, int64_t* rows_out, int64_t* cols_out) {
    for (int I = 0; I < c->Mb; I++)
        for (int k = 0; k < c->deg[I]; k++)
            for (int r = 0; r < c->Z; r++) {
                int64_t e = edge_of(c, I, r, k);
                rows_out[e] = (int64_t)I * c->Z + r;
                cols_out[e] = col_of(c, I, r, k);
            }
}

/* ------------------------------------------------------------------------- */
/* Quantization (R1 step 1/4, R2 round-to-nearest; BASELINE configs[0]). */
/* ------------------------------------------------------------------------- */
/* Lq = min(127, round(4 * ln((1-q)/q))); -1 if q not in (0, 0.5) */
int orc_llr_magnitude(double q) {
    if (!(q > 0.0 && q < 0.5)) return -1;
    double v = round(4.0 * log((1.0 - q) / q));
    if (v > E_MAX) v = E_MAX;
    return (int)v;
}

/* Bob's channel LLR: payload y=0 -> +Lq, y=1 -> -Lq; punctured -> 0; shortened -> +-127
 * by the known bit (R19).  kind may be NULL (all payload). */
void orc_build_llr(int64_t n, int Lq, const uint8_t* y_bits, const uint8_t* kind,
                   const uint8_t* known_bits, int8_t* llr) {
    for (int64_t j = 0; j < n; j++) {
        int y = (y_bits[j >> 3] >> (j & 7)) & 1;
        int k = kind ? kind[j] : 0;
        if (k == 1) llr[j] = 0;
        else if (k == 2) llr[j] = ((known_bits[j >> 3] >> (j & 7)) & 1) ? -E_MAX : E_MAX;
        else llr[j] = (int8_t)(y ? -Lq : Lq);
    }
}

/* ------------------------------------------------------------------------- */
/* Syndrome ("parity check constraints are tested")             */
/* ------------------------------------------------------------------------- */
void orc_syndrome(const orc_code* c, const uint8_t* bits, uint8_t* syn) {
    memset(syn, 0, (size_t)((c->m + 7) / 8));
    for (int I = 0; I < c->Mb; I++)
        for (int r = 0; r < c->Z; r++) {
            int p = 0;
            for (int k = 0; k < c->deg[I]; k++) {
                int64_t j = col_of(c, I, r, k);
                p ^= (bits[j >> 3] >> (j & 7)) & 1;
            }
            int64_t i = (int64_t)I * c->Z + r;
            if (p) syn[i >> 3] |= (uint8_t)(1u << (i & 7));
        }
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1, verbatim.                                           */
/* ------------------------------------------------------------------------- */
int orc_tau(int p, int q) {
    int a = p < MSG_MAX ? p : MSG_MAX;         /* a <- MIN(p, MSG_max) */
    int b = q < MSG_MAX ? q : MSG_MAX;         /* b <- MIN(q, MSG_max) */
    int g = a > b ? a : b;                     /* g <- MAX(a, b) */
    int l = a < b ? a : b;                     /* l <- MIN(a, b) */
    int d = g - l;                             /* d <- g - l */
    int t;
    if (l > 2) t = l - (d < 2) - (d < 6);      /* tau <- l - (d<2) - (d<6) */
    else { t = l - (d < 4); if (t < 0) t = 0; }/* tau <- MAX(l - (d<4), 0) */
    return t;
}

/* ------------------------------------------------------------------------- */
/* Check node, one row (Eq.(1) sign product, Eq.(4)/(7) box-plus replaced by   */
/* tau; syndrome bit folded into the sign (R5); leave-one-out by the forward/  */
/* backward schedule in ascending block column (R6)).                                  */
/*   x[k] : exact L_ji = E_j' - L_ij^{t-1} (Eq.(8)),  s_i : target syndrome bit        */
/*   Lnew[k] : L_ij^t                                                                  */
/* ------------------------------------------------------------------------- */
void orc_check_node(int d, const int* x, int s_i, int* Lnew) {
    int sgn[256], mag[256], F[256], B[256], o[256];
    int S = s_i;
    for (int k = 0; k < d; k++) {
        sgn[k] = x[k] < 0;                                    /* sign(L_ji) */
        int a = x[k] < 0 ? -x[k] : x[k];
        mag[k] = a < MSG_MAX ? a : MSG_MAX;                   /* 6-bit magnitude (R3) */
        S ^= sgn[k];                                          /* Eq.(1) incl. s_i */
    }
    if (d == 1) {
        o[0] = MSG_MAX;                                       /* empty box-plus: R6 */
    } else if (d == 2) {
        o[0] = mag[1]; o[1] = mag[0];                         /* single operand */
    } else {
        F[0] = mag[0];
        for (int k = 1; k <= d - 2; k++) F[k] = orc_tau(F[k - 1], mag[k]);       /* forward */
        B[d - 1] = mag[d - 1];
        for (int k = d - 2; k >= 1; k--) B[k] = orc_tau(mag[k], B[k + 1]);      /* backward */
        o[0] = B[1];
        o[d - 1] = F[d - 2];
        for (int k = 1; k <= d - 2; k++) o[k] = orc_tau(F[k - 1], B[k + 1]);
    }
    for (int k = 0; k < d; k++) Lnew[k] = (S ^ sgn[k]) ? -o[k] : o[k];   /* Eq.(1) leave-one-out sign */
}

/* Algorithm 2 with Eq.(9): update only if |E_j| != E_max; the guard reads the
 * value before this layer's update (R8); saturate to [-127,127] (R4). */
int orc_vn_update(int E_before, int x, int Lnew) {
    int a = E_before < 0 ? -E_before : E_before;
    if (a == E_MAX) return E_before;                          /* ABS(E_j) != E_max guard */
    int v = x + Lnew;                                         /* E_j <- L_ji^t + L_ij^t */
    if (v > E_MAX) v = E_MAX;
    if (v < -E_MAX) v = -E_MAX;
    return v;
}

/* ------------------------------------------------------------------------- */
/* Decoder (P:62 layered schedule, Algorithm 2 loop; R10-R13).          */
/* ------------------------------------------------------------------------- */
static int syndrome_ok(const orc_code* c, const int* E, const uint8_t* syn) {
    for (int I = 0; I < c->Mb; I++)
        for (int r = 0; r < c->Z; r++) {
            int64_t i = (int64_t)I * c->Z + r;
            int p = (syn[i >> 3] >> (i & 7)) & 1;
            for (int k = 0; k < c->deg[I]; k++) p ^= E[col_of(c, I, r, k)] < 0;   /* bit = (E<0), R9 */
            if (p) return 0;
        }
    return 1;
}

/* small LCG used only to permute row order inside a block row (test hook for R13/F7) */
static uint64_t lcg(uint64_t* s) { *s = *s * 6364136223846793005ULL + 1442695040888963407ULL; return *s >> 33; }

/*
 * Decode one frame.  llr[n], syn[ceil(m/8)].  Outputs: bits[ceil(n/8)] (bit = E<0),
 * *iters, *success; L_out[n_edges] and E_out[n] optional (final state).  perm_seed != 0
 * processes the rows of each block row in a seeded random order (must not change anything).
 */
int orc_decode(const orc_code* c, const int8_t* llr, const uint8_t* syn, int T, int early_stop,
               uint64_t perm_seed, uint8_t* bits, int32_t* iters, uint8_t* success,
               int8_t* L_out, int8_t* E_out) {
    int64_t n = c->n;
    int* E = (int*)malloc(sizeof(int) * n);
    int* L = (int*)calloc((size_t)c->n_edges, sizeof(int));        /* R16: L = 0 */
    int* rord = (int*)malloc(sizeof(int) * c->Z);
    int x[256], Ln[256];
    int64_t jk[256];
    uint64_t ps = perm_seed;
    for (int64_t j = 0; j < n; j++) E[j] = llr[j];                  /* E <- channel LLR */
    int t_done = 0, ok = 0;
    if (early_stop && syndrome_ok(c, E, syn)) { ok = 1; t_done = 0; goto finish; }   /* R10 */
    for (int t = 1; t <= T; t++) {
        for (int I = 0; I < c->Mb; I++) {                           /* layers in order (R13) */
            int d = c->deg[I];
            for (int r = 0; r < c->Z; r++) rord[r] = r;
            if (perm_seed)
                for (int r = c->Z - 1; r > 0; r--) { int q = (int)(lcg(&ps) % (uint64_t)(r + 1)); int tmp = rord[r]; rord[r] = rord[q]; rord[q] = tmp; }
            for (int rr = 0; rr < c->Z; rr++) {
                int r = rord[rr];
                int64_t i = (int64_t)I * c->Z + r;
                int s_i = (syn[i >> 3] >> (i & 7)) & 1;
                for (int k = 0; k < d; k++) {
                    jk[k] = col_of(c, I, r, k);
                    x[k] = E[jk[k]] - L[edge_of(c, I, r, k)];        /* Eq.(8), exact (R7) */
                }
                orc_check_node(d, x, s_i, Ln);
                for (int k = 0; k < d; k++) {
                    L[edge_of(c, I, r, k)] = Ln[k];                  /* L always stored (R8) */
                    E[jk[k]] = orc_vn_update(E[jk[k]], x[k], Ln[k]);
                }
            }
        }
        t_done = t;
        if (early_stop && syndrome_ok(c, E, syn)) { ok = 1; goto finish; }   /* P:99, R11 */
    }
    ok = early_stop ? 0 : syndrome_ok(c, E, syn);                  /* R12 */
finish:
    memset(bits, 0, (size_t)((n + 7) / 8));
    for (int64_t j = 0; j < n; j++) if (E[j] < 0) bits[j >> 3] |= (uint8_t)(1u << (j & 7));
    *iters = t_done;
    *success = (uint8_t)ok;
    if (L_out) for (int64_t e = 0; e < c->n_edges; e++) L_out[e] = (int8_t)L[e];
    if (E_out) for (int64_t j = 0; j < n; j++) E_out[j] = (int8_t)E[j];
    free(E); free(L); free(rord);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Frame-parallel driver: one frame per thread at a time (S:336 inter-frame only). */
/* ------------------------------------------------------------------------- */
typedef struct {
    const orc_code* c; const int8_t* llr; const uint8_t* syn; int T, es;
    uint8_t* bits; int32_t* iters; uint8_t* succ; int8_t* L; int8_t* E;
    int64_t F; int64_t next; pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* p) {
    batch_job* b = (batch_job*)p;
    const orc_code* c = b->c;
    int64_t nb = (c->n + 7) / 8, sb = (c->m + 7) / 8;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int64_t f = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (f >= b->F) break;
        orc_decode(c, b->llr + f * c->n, b->syn + f * sb, b->T, b->es, 0, b->bits + f * nb,
                   b->iters + f, b->succ + f, b->L ? b->L + f * c->n_edges : NULL,
                   b->E ? b->E + f * c->n : NULL);
    }
    return NULL;
}

int orc_decode_batch(const orc_code* c, int64_t F, const int8_t* llr, const uint8_t* syn, int T,
                     int early_stop, uint8_t* bits, int32_t* iters, uint8_t* success,
                     int8_t* L_out, int8_t* E_out, int nthreads) {
    batch_job b = { c, llr, syn, T, early_stop, bits, iters, success, L_out, E_out, F, 0 };
    pthread_mutex_init(&b.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    pthread_t th[512];
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, batch_worker, &b);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&b.mu);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Efficiency (R20): f = (m - p) / ((n - p - s) * h2(q)); leaked bits over the payload's */
/* Shannon limit.  P:41/P:54 use f without defining it.                                 */
/* ------------------------------------------------------------------------- */
double orc_efficiency(int64_t m, int64_t n, int64_t p, int64_t s, double q) {
    double h = -q * log2(q) - (1.0 - q) * log2(1.0 - q);
    return (double)(m - p) / ((double)(n - p - s) * h);
}

/* ========================================================================= */
/* Exact floating-point layered BP, fp64, step by step.    */
/* The reference the quantized decoder is measured against ("maintain the   */
/* high efficiency as the floating-point version").                  */
/* ========================================================================= */

#define ORC_LLR_KNOWN 1000.0   /* R26: stand-in for an infinite LLR (shortened bit, degree-1 check) */

/* Eq.(6): L1 [+] L2 = beta(L1, L2) = 2 atanh(tanh(L1/2) tanh(L2/2)), written literally.  Exact in
 * exact arithmetic; in fp64 tanh(x/2) rounds to 1 for x > ~38, so the decoder uses orc_beta. */
double orc_beta_eq6(double a, double b) { return 2.0 * atanh(tanh(a / 2.0) * tanh(b / 2.0)); }

/* The same function for magnitudes a, b >= 0 in its numerically stable textbook form (reading
 * R26): 2 atanh(tanh(a/2) tanh(b/2)) = min(a,b) + ln(1 + e^{-(a+b)}) - ln(1 + e^{-|a-b|}). */
double orc_beta(double a, double b) {
    double m = a < b ? a : b;
    return m + log1p(exp(-(a + b))) - log1p(exp(-fabs(a - b)));
}

/* Check node, exact: Eq.(1) sign (syndrome bit folded in, R5), Eq.(2)/(4) magnitude as the box-plus
 * of the other inputs by the forward/backward schedule of R6 (Eq.(7) nesting; box-plus is
 * associative, so the schedule only changes rounding).  x: L_ji, out: L_ij. */
void orc_check_node_float(int d, const double* x, int s_i, double* Lnew) {
    double mag[256], F[256], B[256];
    int sg = s_i, neg[256];
    for (int k = 0; k < d; k++) {
        neg[k] = x[k] < 0.0;
        mag[k] = fabs(x[k]);
        sg ^= neg[k];
    }
    double o[256];
    if (d == 1) {
        o[0] = ORC_LLR_KNOWN;            /* empty box-plus = +inf, R26's finite stand-in (no inf - inf) */
    } else {
        F[0] = mag[0];
        for (int k = 1; k < d; k++) F[k] = orc_beta(F[k - 1], mag[k]);
        B[d - 1] = mag[d - 1];
        for (int k = d - 2; k >= 0; k--) B[k] = orc_beta(mag[k], B[k + 1]);
        o[0] = B[1];
        o[d - 1] = F[d - 2];
        for (int k = 1; k < d - 1; k++) o[k] = orc_beta(F[k - 1], B[k + 1]);
    }
    for (int k = 0; k < d; k++) Lnew[k] = (sg ^ neg[k]) ? -o[k] : o[k];
}

static int syndrome_ok_f(const orc_code* c, const double* E, const uint8_t* syn) {
    for (int I = 0; I < c->Mb; I++)
        for (int r = 0; r < c->Z; r++) {
            int64_t i = (int64_t)I * c->Z + r;
            int p = (syn[i >> 3] >> (i & 7)) & 1;
            for (int k = 0; k < c->deg[I]; k++) p ^= E[col_of(c, I, r, k)] < 0.0;   /* bit = (E<0), R9 */
            if (p) return 0;
        }
    return 1;
}

/* Channel LLR, exact (P:103-104 before quantization): ln((1-q)/q) by Bob's bit; punctured 0;
 * shortened +-known_llr (reading R26: a finite stand-in for +-infinity). */
void orc_build_llr_float(int64_t n, double q, double known_llr, const uint8_t* y_bits, const uint8_t* kind,
                         const uint8_t* known_bits, double* llr) {
    double Lc = log((1.0 - q) / q);
    for (int64_t j = 0; j < n; j++) {
        int yb = (y_bits[j >> 3] >> (j & 7)) & 1;
        int kd = kind ? kind[j] : 0;
        if (kd == 1) llr[j] = 0.0;
        else if (kd == 2) llr[j] = ((known_bits[j >> 3] >> (j & 7)) & 1) ? -known_llr : known_llr;
        else llr[j] = yb ? -Lc : Lc;
    }
}

/* Layered BP decode of one frame (P:91-97 with Eq.(8) L_ji = E_j - L_ij, Eq.(9) E_j = L_ji + L_ij,
 * no saturation); same schedule, stopping rule and outputs as orc_decode (R10-R13, R16). */
int orc_decode_float(const orc_code* c, const double* llr, const uint8_t* syn, int T, int early_stop,
                     uint8_t* bits, int32_t* iters, uint8_t* success, double* L_out, double* E_out) {
    int64_t n = c->n;
    double* E = (double*)malloc(sizeof(double) * n);
    double* L = (double*)calloc((size_t)c->n_edges, sizeof(double));
    double x[256], Ln[256];
    int64_t jk[256];
    for (int64_t j = 0; j < n; j++) E[j] = llr[j];
    int t_done = 0, ok = 0;
    if (early_stop && syndrome_ok_f(c, E, syn)) { ok = 1; goto finish; }
    for (int t = 1; t <= T; t++) {
        for (int I = 0; I < c->Mb; I++) {
            int d = c->deg[I];
            for (int r = 0; r < c->Z; r++) {
                int64_t i = (int64_t)I * c->Z + r;
                int s_i = (syn[i >> 3] >> (i & 7)) & 1;
                for (int k = 0; k < d; k++) {
                    jk[k] = col_of(c, I, r, k);
                    x[k] = E[jk[k]] - L[edge_of(c, I, r, k)];        /* Eq.(8) */
                }
                orc_check_node_float(d, x, s_i, Ln);
                for (int k = 0; k < d; k++) {
                    L[edge_of(c, I, r, k)] = Ln[k];
                    E[jk[k]] = x[k] + Ln[k];                          /* Eq.(9) */
                }
            }
        }
        t_done = t;
        if (early_stop && syndrome_ok_f(c, E, syn)) { ok = 1; goto finish; }
    }
    ok = early_stop ? 0 : syndrome_ok_f(c, E, syn);
finish:
    memset(bits, 0, (size_t)((n + 7) / 8));
    for (int64_t j = 0; j < n; j++) if (E[j] < 0.0) bits[j >> 3] |= (uint8_t)(1u << (j & 7));
    *iters = t_done;
    *success = (uint8_t)ok;
    if (L_out) memcpy(L_out, L, sizeof(double) * (size_t)c->n_edges);
    if (E_out) memcpy(E_out, E, sizeof(double) * (size_t)n);
    free(E); free(L);
    return 0;
}

typedef struct {
    const orc_code* c; const double* llr; const uint8_t* syn; int T, es;
    uint8_t* bits; int32_t* iters; uint8_t* succ; double* L; double* E;
    int64_t F; int64_t next; pthread_mutex_t mu; int flooding;
} batch_job_f;

int orc_decode_float_flooding(const orc_code* c, const double* llr, const uint8_t* syn, int T, int early_stop,
                              uint8_t* bits, int32_t* iters, uint8_t* success, double* L_out, double* E_out);

static void* batch_worker_f(void* p) {
    batch_job_f* b = (batch_job_f*)p;
    const orc_code* c = b->c;
    int64_t nb = (c->n + 7) / 8, sb = (c->m + 7) / 8;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int64_t f = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (f >= b->F) break;
        (b->flooding ? orc_decode_float_flooding : orc_decode_float)(
            c, b->llr + f * c->n, b->syn + f * sb, b->T, b->es, b->bits + f * nb, b->iters + f, b->succ + f,
            b->L ? b->L + f * c->n_edges : NULL, b->E ? b->E + f * c->n : NULL);
    }
    return NULL;
}

int orc_decode_float_batch(const orc_code* c, int64_t F, const double* llr, const uint8_t* syn, int T,
                           int early_stop, uint8_t* bits, int32_t* iters, uint8_t* success, double* L_out,
                           double* E_out, int nthreads, int flooding) {
    batch_job_f b = { c, llr, syn, T, early_stop, bits, iters, success, L_out, E_out, F, 0 };
    b.flooding = flooding;
    pthread_mutex_init(&b.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    pthread_t th[512];
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, batch_worker_f, &b);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&b.mu);
    return 0;
}

/* Flooding schedule of the same exact BP ("layered scheduling ... enables the
 * decoding convergence to speed-up by a factor of two" over "original flooding scheduling").  Every
 * iteration: all check nodes from the previous iteration's state, x_ij = E_j - L_ij (Eq.(8)), then
 * E_j = channel LLR_j + sum_i L_ij (Eq.(9) over all of VN_j's checks at once), summed in ascending
 * check order.  Same stopping rule and outputs as orc_decode_float. */
int orc_decode_float_flooding(const orc_code* c, const double* llr, const uint8_t* syn, int T, int early_stop,
                              uint8_t* bits, int32_t* iters, uint8_t* success, double* L_out, double* E_out) {
    int64_t n = c->n;
    double* E = (double*)malloc(sizeof(double) * n);
    double* L = (double*)calloc((size_t)c->n_edges, sizeof(double));
    double x[256], Ln[256];
    for (int64_t j = 0; j < n; j++) E[j] = llr[j];
    int t_done = 0, ok = 0;
    if (early_stop && syndrome_ok_f(c, E, syn)) { ok = 1; goto finish; }
    for (int t = 1; t <= T; t++) {
        for (int I = 0; I < c->Mb; I++)                       /* all check nodes, old E and L */
            for (int r = 0; r < c->Z; r++) {
                int d = c->deg[I];
                int64_t i = (int64_t)I * c->Z + r;
                int s_i = (syn[i >> 3] >> (i & 7)) & 1;
                for (int k = 0; k < d; k++) x[k] = E[col_of(c, I, r, k)] - L[edge_of(c, I, r, k)];
                orc_check_node_float(d, x, s_i, Ln);
                for (int k = 0; k < d; k++) L[edge_of(c, I, r, k)] = Ln[k];   /* E untouched in this pass */
            }
        for (int64_t j = 0; j < n; j++) E[j] = llr[j];         /* all variable nodes */
        for (int I = 0; I < c->Mb; I++)
            for (int r = 0; r < c->Z; r++)
                for (int k = 0; k < c->deg[I]; k++) E[col_of(c, I, r, k)] += L[edge_of(c, I, r, k)];
        t_done = t;
        if (early_stop && syndrome_ok_f(c, E, syn)) { ok = 1; goto finish; }
    }
    ok = early_stop ? 0 : syndrome_ok_f(c, E, syn);
finish:
    memset(bits, 0, (size_t)((n + 7) / 8));
    for (int64_t j = 0; j < n; j++) if (E[j] < 0.0) bits[j >> 3] |= (uint8_t)(1u << (j & 7));
    *iters = t_done;
    *success = (uint8_t)ok;
    if (L_out) memcpy(L_out, L, sizeof(double) * (size_t)c->n_edges);
    if (E_out) memcpy(E_out, E, sizeof(double) * (size_t)n);
    free(E); free(L);
    return 0;
}
