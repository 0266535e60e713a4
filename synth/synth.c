/*
 * synth.c -- seeded, synthetic INPUT generators shared by the oracle tests and the
 * CUDA path's tests/bench.  This file holds none of the decoder's arithmetic: it
 * builds the workload (a QC base matrix, a reserved puncture/shorten order, and
 * binary-symmetric-channel frames), nothing else.  Both sides receive its outputs
 * as plain inputs; neither side's arithmetic lives here.
 *
 * Recipe ("base matrix of size Mb x Nb",
 * P:157 "positions with low column weights are chosen as puncturing bits first"):
 *   code:   column-degree counts by largest remainder of f_k*Nb (ties -> lower degree),
 *           columns sorted by descending degree, each column takes its d least-loaded
 *           rows (ties by the seeded RNG), then shifts uniform in [0,Z) in row-major
 *           order over non-zero entries.  RNG = sequential SplitMix64 from the seed.
 *   order:  variables sorted by (column weight ascending, seeded random key).
 *   frames: counter-based: x uniform, e_j ~ Bernoulli(q) as (hash < floor(q*2^64)),
 *           y = x XOR e.  Frame ids are global, so any shard of a batch is bit-identical
 *           to the same slice of the full batch.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
    z += GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* sequential SplitMix64 stream */
typedef struct { uint64_t s; } sm64;
static inline uint64_t sm64_next(sm64* r) { uint64_t v = mix64(r->s); r->s += GOLDEN; return v; }

uint64_t synth_mix64(uint64_t z) { return mix64(z); }

/*
 * Degree counts by largest remainder.  frac_e4[k] are fractions in units of 1e-4
 * (exact integers, so remainder ties are decided exactly, not by float noise).
 * Returns 0 on success, -1 on bad input.
 */
int synth_degree_counts(int32_t Nb, int32_t nd, const int32_t* degs, const int32_t* frac_e4,
                        int32_t* counts_out) {
    int64_t total = 0, rem[64];
    if (nd < 1 || nd > 64) return -1;
    for (int k = 0; k < nd; k++) total += frac_e4[k];
    if (total != 10000) return -1;
    int32_t assigned = 0;
    for (int k = 0; k < nd; k++) {
        int64_t num = (int64_t)frac_e4[k] * Nb;
        counts_out[k] = (int32_t)(num / 10000);
        rem[k] = num % 10000;
        assigned += counts_out[k];
    }
    while (assigned < Nb) {
        int best = -1;
        for (int k = 0; k < nd; k++) {
            if (best < 0 || rem[k] > rem[best] || (rem[k] == rem[best] && degs[k] < degs[best])) best = k;
        }
        counts_out[best] += 1;
        rem[best] = -1;
        assigned++;
    }
    return 0;
}

/*
 * Build a QC base matrix: shifts_out[Mb*Nb] row-major, -1 = zero block.
 */
int synth_qc_code(int32_t Mb, int32_t Nb, int32_t Z, int32_t nd, const int32_t* degs,
                  const int32_t* frac_e4, uint64_t seed, int32_t* shifts_out) {
    int32_t counts[64];
    if (Mb < 1 || Nb <= Mb || Z < 1) return -1;
    if (synth_degree_counts(Nb, nd, degs, frac_e4, counts)) return -1;
    for (int k = 0; k < nd; k++) if (degs[k] < 1 || degs[k] > Mb) return -1;
    /* column degrees in descending order */
    int32_t* coldeg = (int32_t*)malloc(sizeof(int32_t) * Nb);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * nd);
    for (int k = 0; k < nd; k++) order[k] = k;
    for (int a = 0; a < nd; a++)
        for (int b = a + 1; b < nd; b++)
            if (degs[order[b]] > degs[order[a]]) { int t = order[a]; order[a] = order[b]; order[b] = t; }
    int c = 0;
    for (int a = 0; a < nd; a++)
        for (int q = 0; q < counts[order[a]]; q++) coldeg[c++] = degs[order[a]];
    sm64 rng = { seed };
    int32_t* load = (int32_t*)calloc(Mb, sizeof(int32_t));
    uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * Mb);
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * Mb);
    for (int i = 0; i < Mb * Nb; i++) shifts_out[i] = -1;
    for (int J = 0; J < Nb; J++) {
        for (int I = 0; I < Mb; I++) { key[I] = sm64_next(&rng); idx[I] = I; }
        /* sort rows by (load, key) ascending -- insertion sort, Mb is small */
        for (int a = 1; a < Mb; a++) {
            int v = idx[a], b = a - 1;
            while (b >= 0 && (load[idx[b]] > load[v] || (load[idx[b]] == load[v] && key[idx[b]] > key[v]))) {
                idx[b + 1] = idx[b]; b--;
            }
            idx[b + 1] = v;
        }
        for (int q = 0; q < coldeg[J]; q++) { shifts_out[idx[q] * Nb + J] = 0; load[idx[q]]++; }
    }
    for (int I = 0; I < Mb; I++)
        for (int J = 0; J < Nb; J++)
            if (shifts_out[I * Nb + J] >= 0) shifts_out[I * Nb + J] = (int32_t)(sm64_next(&rng) % (uint64_t)Z);
    free(coldeg); free(order); free(load); free(key); free(idx);
    return 0;
}

/*
 * Reserved (rate-adaptive) order: all n variables sorted by (column weight ascending,
 * seeded random key).  Column weight of variable j = number of non-zero entries in
 * base column j / Z.  P:157.
 */
int synth_reserved_order(const int32_t* shifts, int32_t Mb, int32_t Nb, int32_t Z, uint64_t seed,
                         int64_t* order_out) {
    int64_t n = (int64_t)Nb * Z;
    int32_t* w = (int32_t*)calloc(Nb, sizeof(int32_t));
    for (int I = 0; I < Mb; I++) for (int J = 0; J < Nb; J++) if (shifts[I * Nb + J] >= 0) w[J]++;
    /* counting sort by weight, then within a weight class sort by random key */
    uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * n);
    sm64 rng = { seed };
    for (int64_t j = 0; j < n; j++) key[j] = sm64_next(&rng);
    int64_t pos = 0;
    for (int wt = 0; wt <= Mb; wt++) {
        int64_t start = pos;
        for (int64_t j = 0; j < n; j++) if (w[j / Z] == wt) order_out[pos++] = j;
        /* shell sort the class by key (deterministic) */
        int64_t len = pos - start;
        for (int64_t gap = len / 2; gap > 0; gap /= 2)
            for (int64_t a = start + gap; a < pos; a++) {
                int64_t v = order_out[a], b = a;
                while (b - gap >= start && key[order_out[b - gap]] > key[v]) { order_out[b] = order_out[b - gap]; b -= gap; }
                order_out[b] = v;
            }
    }
    free(w); free(key);
    return pos == n ? 0 : -1;
}

/* ---------------- frames ---------------- */
typedef struct {
    int64_t n, f0, f1, nbytes;
    uint64_t thr, kseed;
    uint8_t *x, *y;
    int32_t* nerr;
    int64_t base;           /* global id of row 0 of the output arrays */
} frame_job;

static void gen_one(const frame_job* jb, int64_t fid) {
    int64_t row = fid - jb->base;
    uint8_t* xr = jb->x + row * jb->nbytes;
    uint8_t* yr = jb->y ? jb->y + row * jb->nbytes : NULL;
    uint64_t kx = mix64(jb->kseed ^ mix64(2 * (uint64_t)fid));
    uint64_t ke = mix64(jb->kseed ^ mix64(2 * (uint64_t)fid + 1));
    int32_t ne = 0;
    int64_t nw = (jb->n + 63) / 64;
    for (int64_t w = 0; w < nw; w++) {
        uint64_t xv = mix64(kx + (uint64_t)w);
        uint64_t ev = 0;
        int64_t lim = jb->n - w * 64; if (lim > 64) lim = 64;
        if (lim < 64) xv &= ((1ULL << lim) - 1);
        for (int b = 0; b < lim; b++)
            if (mix64(ke + (uint64_t)(w * 64 + b)) < jb->thr) ev |= 1ULL << b;
        ne += __builtin_popcountll(ev);
        uint64_t yv = xv ^ ev;
        for (int q = 0; q < 8 && w * 8 + q < jb->nbytes; q++) {
            xr[w * 8 + q] = (uint8_t)(xv >> (8 * q));
            if (yr) yr[w * 8 + q] = (uint8_t)(yv >> (8 * q));
        }
    }
    if (jb->nerr) jb->nerr[row] = ne;
}

typedef struct { frame_job* jb; int64_t a, b; } frame_chunk;
static void* frame_worker(void* p) {
    frame_chunk* c = (frame_chunk*)p;
    for (int64_t f = c->a; f < c->b; f++) gen_one(c->jb, f);
    return NULL;
}

/*
 * Generate frames [f0, f0+F) of a BSC(q) workload.  x_out/y_out are [F][ceil(n/8)] bytes,
 * LSB-first (bit j of a frame is bit j%8 of byte j/8).  nerr_out[F] = true error weight.
 * q is given as the exact threshold thr = floor(q * 2^64) computed by the caller.
 */
int synth_frames(int64_t n, uint64_t thr, uint64_t seed, int64_t f0, int64_t F,
                 uint8_t* x_out, uint8_t* y_out, int32_t* nerr_out, int32_t nthreads) {
    if (n < 1 || F < 0) return -1;
    frame_job jb = { n, f0, f0 + F, (n + 7) / 8, thr, mix64(seed), x_out, y_out, nerr_out, f0 };
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (F < nthreads) nthreads = (int32_t)(F > 0 ? F : 1);
    pthread_t th[256];
    frame_chunk ch[256];
    for (int t = 0; t < nthreads; t++) {
        ch[t].jb = &jb;
        ch[t].a = f0 + F * t / nthreads;
        ch[t].b = f0 + F * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, frame_worker, &ch[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    return 0;
}
