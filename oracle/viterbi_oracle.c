/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference soft/hard-decision Viterbi decoder
 * (vitertile 0.1.0, /root/reference/pkg/src/vitertile).  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load this
 * library, and only as the checker / the timed CPU baseline.  The product
 * path (paper_2011_13579_b200) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function below against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py,
 * which imports /root/reference/pkg/src in the build container).
 *
 * All arithmetic is exact int64 on integer-valued LLRs, which equals the
 * reference's float64 arithmetic for the integer inputs the parity contract
 * is defined on.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define VTO_MAX_B 8

typedef struct {
    int K;                    /* constraint length */
    int B;                    /* outputs per input bit (len(generators)) */
    uint32_t gens[VTO_MAX_B]; /* generator polynomials, bit K-1 taps the input */
} vto_code;

static int parity32(uint32_t x) { return __builtin_popcount(x) & 1; }

/* codes.py:183-193 branch_output: register = (u << (K-1)) | state;
 * output bit b = parity(g_b & register); to_state = (u << (K-2)) | (state >> 1). */
static void branch_output(const vto_code* c, uint32_t state, uint32_t u, uint32_t* to, int* bits) {
    uint32_t reg = (u << (c->K - 1)) | state;
    for (int b = 0; b < c->B; ++b) bits[b] = parity32(c->gens[b] & reg);
    *to = (u << (c->K - 2)) | (state >> 1);
}

/* reference.py:60-83 predecessors/_acs_tables: predecessors of j are
 * i0 = 2*(j mod 2^(K-2)), i1 = i0 + 1; input bit u = j >> (K-2); signs are
 * 1 - 2*branch_output bits. */
typedef struct {
    int S;
    int32_t* pred0;
    int32_t* pred1;
    int8_t* sgn0; /* S x B */
    int8_t* sgn1;
} acs_tables;

static int tables_build(const vto_code* c, acs_tables* t) {
    int S = 1 << (c->K - 1);
    t->S = S;
    t->pred0 = (int32_t*)malloc(sizeof(int32_t) * S);
    t->pred1 = (int32_t*)malloc(sizeof(int32_t) * S);
    t->sgn0 = (int8_t*)malloc((size_t)S * c->B);
    t->sgn1 = (int8_t*)malloc((size_t)S * c->B);
    if (!t->pred0 || !t->pred1 || !t->sgn0 || !t->sgn1) return -1;
    for (int j = 0; j < S; ++j) {
        uint32_t beta = (uint32_t)j & ((1u << (c->K - 2)) - 1);
        uint32_t i0 = 2 * beta, i1 = i0 + 1, u = (uint32_t)j >> (c->K - 2), to;
        int bits[VTO_MAX_B];
        t->pred0[j] = (int32_t)i0;
        t->pred1[j] = (int32_t)i1;
        branch_output(c, i0, u, &to, bits);
        for (int b = 0; b < c->B; ++b) t->sgn0[j * c->B + b] = (int8_t)(1 - 2 * bits[b]);
        branch_output(c, i1, u, &to, bits);
        for (int b = 0; b < c->B; ++b) t->sgn1[j * c->B + b] = (int8_t)(1 - 2 * bits[b]);
    }
    return 0;
}

static void tables_free(acs_tables* t) {
    free(t->pred0); free(t->pred1); free(t->sgn0); free(t->sgn1);
}

/*
 * reference.py:95-128 forward_batch (one frame) + reference.py:131-144
 * traceback_batch + reference.py:194-206 decode_batch.
 *   llr:   B x N, element (b, t) at llr[b * ld + t]   (the reference's (B, N) layout)
 *   init:  optional S initial metrics (reference.py:111-112; NULL = all zero)
 *   renorm: subtract max metric after every stage (reference.py:124-125)
 *   bits:  N decoded bits (uint8)
 *   final_metric: max path metric at the end (reference.py:206)
 * Tie rule: take1 = cand1 >= cand0 (reference.py:121); final state = argmax,
 * lowest index on ties (np.argmax, reference.py:138).
 * surv: caller scratch of N*S bytes, or NULL to allocate.
 */
static int forward_traceback(const vto_code* c, const acs_tables* t, const int64_t* llr, int64_t ld,
                             int64_t N, const int64_t* init, int renorm, uint8_t* bits,
                             int64_t* final_metric, uint8_t* surv, int64_t* lam, int64_t* nxt) {
    int S = t->S, B = c->B;
    for (int j = 0; j < S; ++j) lam[j] = init ? init[j] : 0;
    for (int64_t n = 0; n < N; ++n) {
        int64_t l[VTO_MAX_B];
        for (int b = 0; b < B; ++b) l[b] = llr[b * ld + n];
        uint8_t* sv = surv + n * S;
        for (int j = 0; j < S; ++j) {
            int64_t d0 = 0, d1 = 0;
            for (int b = 0; b < B; ++b) {
                d0 += t->sgn0[j * B + b] * l[b];
                d1 += t->sgn1[j * B + b] * l[b];
            }
            int64_t c0 = lam[t->pred0[j]] + d0;
            int64_t c1 = lam[t->pred1[j]] + d1;
            int take1 = c1 >= c0;
            nxt[j] = take1 ? c1 : c0;
            sv[j] = (uint8_t)take1;
        }
        if (renorm) {
            int64_t mx = nxt[0];
            for (int j = 1; j < S; ++j) if (nxt[j] > mx) mx = nxt[j];
            for (int j = 0; j < S; ++j) nxt[j] -= mx;
        }
        memcpy(lam, nxt, sizeof(int64_t) * S);
    }
    int best = 0;
    for (int j = 1; j < S; ++j) if (lam[j] > lam[best]) best = j;
    if (final_metric) *final_metric = lam[best];
    uint32_t mask = (1u << (c->K - 2)) - 1, shift = (uint32_t)(c->K - 2);
    uint32_t j = (uint32_t)best;
    for (int64_t n = N - 1; n >= 0; --n) {
        bits[n] = (uint8_t)(j >> shift);
        j = 2 * (j & mask) + surv[n * S + j];
    }
    return 0;
}

static int code_ok(const vto_code* c) {
    if (c->K < 3 || c->K > 16 || c->B < 1 || c->B > VTO_MAX_B) return 0;
    return 1;
}

/* Decode one (B, N) frame; llr row-major (B, N) int64. */
int vto_decode_frame(const vto_code* c, const int64_t* llr, int64_t N, const int64_t* init,
                     int renorm, uint8_t* bits, int64_t* final_metric) {
    if (!code_ok(c) || N < 1) return -1;
    acs_tables t;
    if (tables_build(c, &t)) return -2;
    uint8_t* surv = (uint8_t*)malloc((size_t)N * t.S);
    int64_t* lam = (int64_t*)malloc(sizeof(int64_t) * t.S * 2);
    int rc = (surv && lam) ? forward_traceback(c, &t, llr, N, N, init, renorm, bits, final_metric,
                                               surv, lam, lam + t.S) : -2;
    free(surv); free(lam); tables_free(&t);
    return rc;
}

/* reference.py:194-206 decode_batch over F frames stored (F, B, N) int64. */
int vto_decode_batch(const vto_code* c, const int64_t* llrs, int64_t F, int64_t N, int renorm,
                     uint8_t* bits, int64_t* final_metric) {
    if (!code_ok(c) || N < 1) return -1;
    acs_tables t;
    if (tables_build(c, &t)) return -2;
    uint8_t* surv = (uint8_t*)malloc((size_t)N * t.S);
    int64_t* lam = (int64_t*)malloc(sizeof(int64_t) * t.S * 2);
    int rc = 0;
    if (!surv || !lam) rc = -2;
    for (int64_t f = 0; f < F && rc == 0; ++f)
        rc = forward_traceback(c, &t, llrs + f * c->B * N, N, N, NULL, renorm, bits + f * N,
                               final_metric ? final_metric + f : NULL, surv, lam, lam + t.S);
    free(surv); free(lam); tables_free(&t);
    return rc;
}

/* ---------------------------------------------------------------------------
 * framing.py:68-141 plan_frames + decode_stream on an int8 stream stored
 * stage-major (N, B) (the CLI/LLR-file layout, cli.py:136-140).  Windows:
 * emit [kF, min((k+1)F, N)), window [max(0, emit_start - V), min(N, emit_stop + V));
 * each window decoded from all-zero metrics; only the emit range is kept.
 * ------------------------------------------------------------------------- */
typedef struct {
    const vto_code* c;
    const acs_tables* t;
    const int8_t* llr;
    int64_t N, F, V;
    uint8_t* out;
    int64_t w_begin, w_end;
    int rc;
} stream_job;

static void* stream_worker(void* arg) {
    stream_job* j = (stream_job*)arg;
    int64_t Lmax = j->F + 2 * j->V;
    if (Lmax > j->N) Lmax = j->N;
    int B = j->c->B, S = j->t->S;
    int64_t* wl = (int64_t*)malloc(sizeof(int64_t) * B * Lmax);
    uint8_t* surv = (uint8_t*)malloc((size_t)Lmax * S);
    uint8_t* bits = (uint8_t*)malloc((size_t)Lmax);
    int64_t* lam = (int64_t*)malloc(sizeof(int64_t) * S * 2);
    if (!wl || !surv || !bits || !lam) { j->rc = -2; goto done; }
    for (int64_t w = j->w_begin; w < j->w_end; ++w) {
        int64_t e0 = w * j->F, e1 = e0 + j->F < j->N ? e0 + j->F : j->N;
        int64_t s = e0 - j->V > 0 ? e0 - j->V : 0;
        int64_t stop = e1 + j->V < j->N ? e1 + j->V : j->N;
        int64_t L = stop - s;
        for (int64_t n = 0; n < L; ++n)
            for (int b = 0; b < B; ++b) wl[b * L + n] = j->llr[(s + n) * B + b];
        forward_traceback(j->c, j->t, wl, L, L, NULL, 0, bits, NULL, surv, lam, lam + S);
        memcpy(j->out + e0, bits + (e0 - s), (size_t)(e1 - e0));
    }
done:
    free(wl); free(surv); free(bits); free(lam);
    return NULL;
}

int vto_num_windows(int64_t N, int64_t F) { return (int)((N + F - 1) / F); }

/* Decode windows [w_begin, w_end) of the plan (all windows: 0, ceil(N/F)).
 * out is the full N-byte stream output; only emit ranges of the given windows
 * are written.  nthreads <= 1 runs serially. */
int vto_decode_stream_range(const vto_code* c, const int8_t* llr, int64_t N, int64_t F, int64_t V,
                            int64_t w_begin, int64_t w_end, uint8_t* out, int nthreads) {
    if (!code_ok(c) || N < 1 || F < 1 || V < 0) return -1;
    acs_tables t;
    if (tables_build(c, &t)) return -2;
    if (nthreads < 1) nthreads = 1;
    int64_t nw = w_end - w_begin;
    if (nthreads > nw) nthreads = (int)(nw > 0 ? nw : 1);
    stream_job* jobs = (stream_job*)calloc((size_t)nthreads, sizeof(stream_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    int rc = 0;
    for (int i = 0; i < nthreads; ++i) {
        jobs[i].c = c; jobs[i].t = &t; jobs[i].llr = llr; jobs[i].N = N; jobs[i].F = F; jobs[i].V = V;
        jobs[i].out = out;
        jobs[i].w_begin = w_begin + nw * i / nthreads;
        jobs[i].w_end = w_begin + nw * (i + 1) / nthreads;
        if (nthreads == 1) stream_worker(&jobs[i]);
        else pthread_create(&th[i], NULL, stream_worker, &jobs[i]);
    }
    for (int i = 0; i < nthreads; ++i) {
        if (nthreads > 1) pthread_join(th[i], NULL);
        if (jobs[i].rc) rc = jobs[i].rc;
    }
    free(jobs); free(th); tables_free(&t);
    return rc;
}

int vto_decode_stream(const vto_code* c, const int8_t* llr, int64_t N, int64_t F, int64_t V,
                      uint8_t* out, int nthreads) {
    return vto_decode_stream_range(c, llr, N, F, V, 0, (N + F - 1) / F, out, nthreads);
}

/* codes.py:216-230 encode_batch: frames (F, N) -> coded (F, N, B), zero initial state. */
int vto_encode_batch(const vto_code* c, const uint8_t* bits, int64_t F, int64_t N, uint8_t* coded) {
    if (!code_ok(c)) return -1;
    for (int64_t f = 0; f < F; ++f) {
        uint32_t state = 0;
        for (int64_t n = 0; n < N; ++n) {
            uint32_t to;
            int ob[VTO_MAX_B];
            branch_output(c, state, bits[f * N + n] & 1u, &to, ob);
            for (int b = 0; b < c->B; ++b) coded[(f * N + n) * c->B + b] = (uint8_t)ob[b];
            state = to;
        }
    }
    return 0;
}
