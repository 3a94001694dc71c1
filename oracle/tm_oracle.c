/*
 * tm_oracle.c -- plain, slow, fp64 CPU oracle for the TalkingMachines
 * sparse-causal chunk-attention hot path (arXiv 2506.03099).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2506_03099_b200/csrc) and neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n.
 *
 * Every function is the plain definition written out, in fp64, with no
 * blocking, fusion, online softmax or reordering:
 *   - orc_allowed_key_chunks   P:137-143 (Sec 4.2 attend set)
 *   - orc_window_attention     P:147-151 (Eq 7) over the full-window sparse
 *                              causal mask
 *   - orc_stream_attention     P:151 + P:187 (KV cache of c0, c_{t-1}):
 *                              softmax over the literal concatenation
 *                              [K_ref | K_prev | K_cur] (c2)
 *   - orc_interpolate          P:60 (Eq 1)
 *   - orc_velocity_target      P:65 (Eq 2)
 *   - orc_euler                P:55 (ODE integration, x <- x + dt*v)
 *   - orc_sampler_step         few-step student update:
 *                              x1_hat = x + (1 - t) u; re-noise by Eq 1
 *   - orc_audio_window         5-latent-frame audio window, edges
 *                              clamped by repeating the boundary frame
 *   - orc_audio_cross_attention audio cross-attention of the face-region query
 *                              tokens of each latent frame
 *
 * Tensor layout (all fp64, row-major, token-major as the API's
 * [L][H][d]):  element (token i, head h, dim c) at ((i*H)+h)*d + c.
 * Output of attention: out[r][h][c] for the r-th requested query row.
 *
 * Masked keys are EXCLUDED from the softmax (not penalised).
 * Return codes: 0 ok; -1 dimension error; -2 degenerate mask (an
 * all-false row); -3 negative chunk index; -4 bad argument.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_DIM (-1)
#define ORC_ERR_DEGENERATE (-2)
#define ORC_ERR_NEG_CHUNK (-3)
#define ORC_ERR_ARG (-4)

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Sec 4.2: a token of chunk c_t attends all tokens of c_t, of
 * c_{t-1} and of c_0.  As a SET: t=0 -> {0}; t=1 -> {0,1}.
 * Writes the distinct allowed chunk indices in increasing order. */
int orc_allowed_key_chunks(int64_t t, int64_t out[3]) {
    if (t < 0) return ORC_ERR_NEG_CHUNK;
    int n = 0;
    out[n++] = 0;                       /* c_0, the starting chunk */
    if (t - 1 > 0) out[n++] = t - 1;    /* c_{t-1}, if distinct from c_0 */
    if (t > 0) out[n++] = t;            /* c_t itself */
    return n;
}

static int chunk_allowed(int64_t qc, int64_t kc) {
    int64_t a[3];
    int n = orc_allowed_key_chunks(qc, a);
    for (int i = 0; i < n; ++i)
        if (a[i] == kc) return 1;
    return 0;
}

/* One query row, one head: the two-pass softmax of Eq 7 over the keys listed
 * in idx[0..n): s_j = (q . k_j) * scale; m = max s; p_j = exp(s_j - m);
 * l = sum p; o = sum_j (p_j / l) v_j.  k_row/v_row give the address of key
 * j's (head h) vector. */
static void attend_row(const double* qv, int d, const double* const* krow,
                       const double* const* vrow, int64_t n, double scale,
                       double* s, double* o) {
    double m = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int c = 0; c < d; ++c) dot += qv[c] * krow[j][c];
        s[j] = dot * scale;
        if (s[j] > m) m = s[j];
    }
    double l = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        s[j] = exp(s[j] - m);
        l += s[j];
    }
    for (int c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        double w = s[j] / l;
        for (int c = 0; c < d; ++c) o[c] += w * vrow[j][c];
    }
}

/* c1: full-window form.  The sequence is [c_0 | c_1 | ... | c_{N-1}] with
 * chunk_len[c] tokens in chunk c.  For each requested query token rows[r]
 * and head h, attend over keys j with chunk(j) in allowed(chunk(i)).
 * rows == NULL means all L rows in order. */
int orc_window_attention(const double* q, const double* k, const double* v,
                         int H, int d, const int64_t* chunk_len, int n_chunks,
                         double scale, const int64_t* rows, int64_t n_rows,
                         double* out) {
    if (H <= 0 || d <= 0 || n_chunks <= 0 || !q || !k || !v || !out || !chunk_len)
        return ORC_ERR_DIM;
    int64_t L = 0;
    for (int c = 0; c < n_chunks; ++c) {
        if (chunk_len[c] < 0) return ORC_ERR_DIM;
        L += chunk_len[c];
    }
    if (L == 0) return ORC_ERR_DIM;
    int64_t* chunk_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)L);
    if (!chunk_of) return ORC_ERR_ARG;
    {
        int64_t i = 0;
        for (int c = 0; c < n_chunks; ++c)
            for (int64_t t = 0; t < chunk_len[c]; ++t) chunk_of[i++] = c;
    }
    if (!rows) n_rows = L;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t i = rows ? rows[r] : r;
        if (i < 0 || i >= L) { free(chunk_of); return ORC_ERR_DIM; }
    }
    int status = ORC_OK;
#pragma omp parallel
    {
        const double** kr = (const double**)malloc(sizeof(double*) * (size_t)L);
        const double** vr = (const double**)malloc(sizeof(double*) * (size_t)L);
        double* s = (double*)malloc(sizeof(double) * (size_t)L);
#pragma omp for schedule(dynamic, 4) collapse(2)
        for (int64_t r = 0; r < n_rows; ++r) {
            for (int h = 0; h < H; ++h) {
                int64_t i = rows ? rows[r] : r;
                int64_t n = 0;
                for (int64_t j = 0; j < L; ++j) {
                    if (chunk_allowed(chunk_of[i], chunk_of[j])) {
                        kr[n] = k + ((j * H) + h) * (int64_t)d;
                        vr[n] = v + ((j * H) + h) * (int64_t)d;
                        ++n;
                    }
                }
                if (n == 0) {
#pragma omp atomic write
                    status = ORC_ERR_DEGENERATE;
                    continue;
                }
                attend_row(q + ((i * H) + h) * (int64_t)d, d, kr, vr, n, scale, s,
                           out + ((r * H) + h) * (int64_t)d);
            }
        }
        free(kr); free(vr); free(s);
    }
    free(chunk_of);
    return status;
}

/* c2: streaming form for chunk t >= 1 at one (layer, step).  Keys/values
 * are the literal concatenation [ref (Lr) | prev (Lp, 0 when t == 1) |
 * cur (Lc)], all [len][H][d]; queries are the Lc current tokens. */
int orc_stream_attention(const double* q, int64_t Lc, int H, int d,
                         const double* k_ref, const double* v_ref, int64_t Lr,
                         const double* k_prev, const double* v_prev, int64_t Lp,
                         const double* k_cur, const double* v_cur, double scale,
                         const int64_t* rows, int64_t n_rows, double* out) {
    if (Lc <= 0 || H <= 0 || d <= 0 || Lr < 0 || Lp < 0 || !q || !out) return ORC_ERR_DIM;
    if ((Lr > 0 && (!k_ref || !v_ref)) || (Lp > 0 && (!k_prev || !v_prev)) || !k_cur || !v_cur)
        return ORC_ERR_ARG;
    const int64_t Lk = Lr + Lp + Lc;
    const int64_t row = (int64_t)H * d;
    /* The concatenation, materialised (plain, obviously correct). */
    double* K = (double*)malloc(sizeof(double) * (size_t)(Lk * row));
    double* V = (double*)malloc(sizeof(double) * (size_t)(Lk * row));
    if (!K || !V) { free(K); free(V); return ORC_ERR_ARG; }
    if (Lr) { memcpy(K, k_ref, sizeof(double) * Lr * row); memcpy(V, v_ref, sizeof(double) * Lr * row); }
    if (Lp) { memcpy(K + Lr * row, k_prev, sizeof(double) * Lp * row); memcpy(V + Lr * row, v_prev, sizeof(double) * Lp * row); }
    memcpy(K + (Lr + Lp) * row, k_cur, sizeof(double) * Lc * row);
    memcpy(V + (Lr + Lp) * row, v_cur, sizeof(double) * Lc * row);
    if (!rows) n_rows = Lc;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t i = rows ? rows[r] : r;
        if (i < 0 || i >= Lc) { free(K); free(V); return ORC_ERR_DIM; }
    }
#pragma omp parallel
    {
        const double** kr = (const double**)malloc(sizeof(double*) * (size_t)Lk);
        const double** vr = (const double**)malloc(sizeof(double*) * (size_t)Lk);
        double* s = (double*)malloc(sizeof(double) * (size_t)Lk);
#pragma omp for schedule(dynamic, 4) collapse(2)
        for (int64_t r = 0; r < n_rows; ++r) {
            for (int h = 0; h < H; ++h) {
                int64_t i = rows ? rows[r] : r;
                for (int64_t j = 0; j < Lk; ++j) {
                    kr[j] = K + j * row + (int64_t)h * d;
                    vr[j] = V + j * row + (int64_t)h * d;
                }
                attend_row(q + i * row + (int64_t)h * d, d, kr, vr, Lk, scale, s,
                           out + (r * H + h) * (int64_t)d);
            }
        }
        free(kr); free(vr); free(s);
    }
    free(K); free(V);
    return ORC_OK;
}

/* Eq 1: x_t = t x_1 + (1 - t) x_0. */
int orc_interpolate(const double* x0, const double* x1, double t, int64_t n, double* out) {
    if (n < 0 || (n > 0 && (!x0 || !x1 || !out))) return ORC_ERR_DIM;
    for (int64_t i = 0; i < n; ++i) out[i] = t * x1[i] + (1.0 - t) * x0[i];
    return ORC_OK;
}

/* Eq 2: v_t = dx_t/dt = x_1 - x_0. */
int orc_velocity_target(const double* x0, const double* x1, int64_t n, double* out) {
    if (n < 0 || (n > 0 && (!x0 || !x1 || !out))) return ORC_ERR_DIM;
    for (int64_t i = 0; i < n; ++i) out[i] = x1[i] - x0[i];
    return ORC_OK;
}

/* P:55 ODE integration with an Euler step: x' = x + dt * v. */
int orc_euler(const double* x, const double* v, int64_t n, double dt, double* out) {
    if (n < 0 || (n > 0 && (!x || !v || !out))) return ORC_ERR_DIM;
    for (int64_t i = 0; i < n; ++i) out[i] = x[i] + dt * v[i];
    return ORC_OK;
}

/* Few-step generator update (student with 2 NFE), one
 * schedule entry: given the state x at time t_cur (Eq 1 convention: t = 0
 * noise, t = 1 data) and the predicted velocity u,
 *   x1_hat = x + (1 - t_cur) * u                     (the implied clean sample)
 *   x_next = t_next * x1_hat + (1 - t_next) * eps     (Eq 1 re-noise to t_next)
 * and for the final entry (t_next >= 1) x_next = x1_hat.  eps may be NULL
 * only when t_next >= 1. */
int orc_sampler_step(const double* x, const double* u, const double* eps, int64_t n, double t_cur,
                     double t_next, double* x_next) {
    if (n < 0 || (n > 0 && (!x || !u || !x_next))) return ORC_ERR_DIM;
    if (t_next < 1.0 && n > 0 && !eps) return ORC_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) {
        const double x1_hat = x[i] + (1.0 - t_cur) * u[i];
        x_next[i] = t_next >= 1.0 ? x1_hat : t_next * x1_hat + (1.0 - t_next) * eps[i];
    }
    return ORC_OK;
}

/* "each latent frame will attend only to the audio tokens within a
 * window of five latent frames centered around itself"; SPEC S:116-118 and its
 * design decision: frames [f - W/2, f + W/2] clamped to [0, frames - 1] by
 * repeating the boundary frame (f = 0 -> {0, 0, 0, 1, 2}).  Writes W frame
 * indices. */
int orc_audio_window(int64_t frames, int64_t f, int window, int64_t* out) {
    if (frames <= 0 || f < 0 || f >= frames || window <= 0 || window % 2 == 0) return ORC_ERR_ARG;
    for (int i = 0; i < window; ++i) {
        int64_t g = f - window / 2 + i;
        if (g < 0) g = 0;
        if (g > frames - 1) g = frames - 1;
        out[i] = g;
    }
    return ORC_OK;
}

/* P:123 (audio cross attention restricted to facial-region queries) with the
 * P:125 window: q [frames][T][H][d] latent-frame tokens, k/v [frames][A][H][d]
 * audio tokens; for every frame f and face token t (face_ids, a subset of
 * [0, T)) the keys/values are the concatenation of the audio tokens of the
 * window frames of f (orc_audio_window), softmax(q k^T * scale) v (Eq 7's
 * form).  Non-face rows of out are 0 (no residual update). */
int orc_audio_cross_attention(const double* q, const double* k, const double* v, int64_t frames,
                              int64_t T, int64_t A, int H, int d, const int64_t* face_ids,
                              int64_t n_face, int window, double scale, double* out) {
    if (frames <= 0 || T <= 0 || A <= 0 || H <= 0 || d <= 0 || !q || !k || !v || !out) return ORC_ERR_DIM;
    if (n_face <= 0 || !face_ids) return ORC_ERR_DEGENERATE;      /* empty face mask */
    for (int64_t i = 0; i < n_face; ++i)
        if (face_ids[i] < 0 || face_ids[i] >= T) return ORC_ERR_DIM;
    const int64_t row = (int64_t)H * d;
    memset(out, 0, sizeof(double) * (size_t)(frames * T * row));
    int64_t* win = (int64_t*)malloc(sizeof(int64_t) * (size_t)window);
    if (!win) return ORC_ERR_ARG;
    int status = ORC_OK;
    for (int64_t f = 0; f < frames && status == ORC_OK; ++f) {
        status = orc_audio_window(frames, f, window, win);
        if (status) break;
        const int64_t Lk = (int64_t)window * A;
#pragma omp parallel
        {
            const double** kr = (const double**)malloc(sizeof(double*) * (size_t)Lk);
            const double** vr = (const double**)malloc(sizeof(double*) * (size_t)Lk);
            double* s = (double*)malloc(sizeof(double) * (size_t)Lk);
#pragma omp for collapse(2)
            for (int64_t i = 0; i < n_face; ++i) {
                for (int h = 0; h < H; ++h) {
                    for (int w = 0; w < window; ++w)
                        for (int64_t a = 0; a < A; ++a) {
                            const int64_t tok = win[w] * A + a;
                            kr[w * A + a] = k + tok * row + (int64_t)h * d;
                            vr[w * A + a] = v + tok * row + (int64_t)h * d;
                        }
                    const int64_t t = face_ids[i];
                    attend_row(q + (f * T + t) * row + (int64_t)h * d, d, kr, vr, Lk, scale, s,
                               out + (f * T + t) * row + (int64_t)h * d);
                }
            }
            free(kr); free(vr); free(s);
        }
    }
    free(win);
    return status;
}
