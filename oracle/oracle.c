/*
 * oracle.c -- plain, slow, fp64 reference for PackMamba's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked into the product.
 *
 * Each function is the plain definition written out, in the paper's order
 * and notation, with no blocking, fusion or reordering:
 *   - packing: FIFO seal (sec 5) and scatter (sec 3.1);
 *   - conv1d_pack fwd: Alg 1 -- causal depthwise conv whose taps
 *     are dropped when they would reach before the sequence start
 *     ("terminated early");
 *   - conv1d_pack bwd: the adjoint, masked with reverse indices read from the
 *     position indices of the next K-1 slots (reading Q7);
 *   - ScanOp_pack fwd: Eq 1a/1b/2a with Euler B (reading Q1),
 *     skip term D (Q3), delta = softplus(dt + dt_bias) (Q4), and the reset
 *     "Set A-bar[i] to zero when indices[i] is zero" (Alg 2);
 *   - ScanOp_pack bwd: reverse recurrence with A-bar -> 0 at heads;
 *   - Eq 3 brute force.
 * "Parity pins" for every function live in tests/test_oracle_*.py.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int pmo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void pmo_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------------ */
/* packing                                                                   */
/* ------------------------------------------------------------------------ */

/* P:273 "sequentially packing sequences in the received order, sealing the
 * pack when it cannot fit the next sequence".  A sequence that
 * exactly fills the remaining space fits (reading Q17).  Lengths > cap are
 * an error: "no instances of sequences spanning across packed sequences"
 * (reading Q18). */
int pmo_plan_fifo(const int32_t* lens, int64_t n, int64_t cap,
                  int64_t* seq_row, int64_t* seq_off, int64_t* n_rows) {
    int64_t row = -1, used = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (lens[i] < 1 || lens[i] > cap) return 2;
        if (row < 0 || used + lens[i] > cap) { /* seal, open a new pack */
            row += 1;
            used = 0;
        }
        seq_row[i] = row;
        seq_off[i] = used;
        used += lens[i];
    }
    *n_rows = row + 1;
    return 0;
}

/* P:273 "a local greedy algorithm that sorts some of the sequences before
 * packing"; sort by length descending (ties: id ascending), then
 * first-fit into the earliest pack with room. */
int pmo_plan_ffd(const int32_t* lens, int64_t n, int64_t cap,
                 int64_t* seq_row, int64_t* seq_off, int64_t* n_rows) {
    for (int64_t i = 0; i < n; ++i)
        if (lens[i] < 1 || lens[i] > cap) return 2;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t* used = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    /* insertion sort: plain and stable enough to be checked by eye */
    for (int64_t i = 1; i < n; ++i) {
        int64_t k = order[i], j = i - 1;
        while (j >= 0 && (lens[order[j]] < lens[k] ||
                          (lens[order[j]] == lens[k] && order[j] > k))) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = k;
    }
    int64_t rows = 0;
    for (int64_t s = 0; s < n; ++s) {
        int64_t i = order[s], r = 0;
        while (r < rows && used[r] + lens[i] > cap) ++r;
        if (r == rows) { used[rows] = 0; rows += 1; }
        seq_row[i] = r;
        seq_off[i] = used[r];
        used[r] += lens[i];
    }
    *n_rows = rows;
    free(order);
    free(used);
    return 0;
}

/* P:120 "concatenating the input tensor along the sequence dimension to
 * obtain a packed_sequence and the auxiliary structure position_indices";
 * S:44-50 invariants: pos runs 0..len-1, 0 at heads and padding, padding
 * data is 0 (reading Q8). */
void pmo_pack(const int32_t* lens, int64_t n, int64_t cap,
              const int64_t* seq_row, const int64_t* seq_off,
              const uint8_t* src, int64_t rec_bytes,
              uint8_t* dst, int32_t* pos, int64_t n_rows) {
    memset(dst, 0, (size_t)(n_rows * cap * rec_bytes));
    memset(pos, 0, sizeof(int32_t) * (size_t)(n_rows * cap));
    int64_t src_tok = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t p = 0; p < lens[i]; ++p) {
            int64_t slot = seq_row[i] * cap + seq_off[i] + p;
            memcpy(dst + slot * rec_bytes, src + (src_tok + p) * rec_bytes,
                   (size_t)rec_bytes);
            pos[slot] = (int32_t)p;
        }
        src_tok += lens[i];
    }
}

/* ------------------------------------------------------------------------ */
/* conv1d_pack                                                               */
/* ------------------------------------------------------------------------ */

static double sigmoid_d(double v) { return 1.0 / (1.0 + exp(-v)); }

/* tap predicate of Alg 1 (reading Q6): tap j reaches o = K-1-j
 * back and is kept iff it stays inside the current sequence. */
static int tap_ok(const int32_t* pos_row, int64_t t, int64_t o) {
    return t - o >= 0 && o <= (int64_t)pos_row[t];
}

void pmo_conv_fwd(const double* x, const double* w, const double* bias,
                  const int32_t* pos, double* out,
                  int64_t R, int64_t Dn, int64_t L, int32_t K, int32_t silu) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t r = 0; r < R; ++r)
        for (int64_t d = 0; d < Dn; ++d) {
            const double* xr = x + (r * Dn + d) * L;
            const int32_t* pr = pos + r * L;
            double* orow = out + (r * Dn + d) * L;
            for (int64_t t = 0; t < L; ++t) {
                double pre = bias ? bias[d] : 0.0;
                for (int32_t j = 0; j < K; ++j) {
                    int64_t o = K - 1 - j;
                    if (tap_ok(pr, t, o)) pre += w[d * K + j] * xr[t - o];
                }
                orow[t] = silu ? pre * sigmoid_d(pre) : pre;
            }
        }
}

/* Adjoint of pmo_conv_fwd.  dx[s] gathers the outputs t = s + o that read
 * x[s] through tap j = K-1-o; the same predicate o <= pos[s+o] is the
 * paper's "reverse indices ... from the position indices of the last
 * conv_width elements" (reading Q7). */
void pmo_conv_bwd(const double* x, const double* w, const double* bias,
                  const int32_t* pos, const double* dout,
                  double* dx, double* dw, double* dbias,
                  int64_t R, int64_t Dn, int64_t L, int32_t K, int32_t silu) {
#pragma omp parallel for schedule(static)
    for (int64_t d = 0; d < Dn; ++d) {
        for (int32_t j = 0; j < K; ++j) dw[d * K + j] = 0.0;
        if (dbias) dbias[d] = 0.0;
        double* dpre = (double*)malloc(sizeof(double) * (size_t)L);
        for (int64_t r = 0; r < R; ++r) {
            const double* xr = x + (r * Dn + d) * L;
            const double* gr = dout + (r * Dn + d) * L;
            const int32_t* pr = pos + r * L;
            /* recompute pre and form dpre = dout * d(out)/d(pre) */
            for (int64_t t = 0; t < L; ++t) {
                double pre = bias ? bias[d] : 0.0;
                for (int32_t j = 0; j < K; ++j) {
                    int64_t o = K - 1 - j;
                    if (tap_ok(pr, t, o)) pre += w[d * K + j] * xr[t - o];
                }
                double g = 1.0;
                if (silu) {
                    double s = sigmoid_d(pre);
                    g = s * (1.0 + pre * (1.0 - s));
                }
                dpre[t] = gr[t] * g;
            }
            double* dxr = dx + (r * Dn + d) * L;
            for (int64_t s = 0; s < L; ++s) {
                double acc = 0.0;
                for (int64_t o = 0; o < K; ++o) {
                    int64_t t = s + o;
                    if (t < L && tap_ok(pr, t, o))
                        acc += w[d * K + (K - 1 - o)] * dpre[t];
                }
                dxr[s] = acc;
            }
            for (int64_t t = 0; t < L; ++t) {
                for (int32_t j = 0; j < K; ++j) {
                    int64_t o = K - 1 - j;
                    if (tap_ok(pr, t, o)) dw[d * K + j] += dpre[t] * xr[t - o];
                }
                if (dbias) dbias[d] += dpre[t];
            }
        }
        free(dpre);
    }
}

/* ------------------------------------------------------------------------ */
/* ScanOp_pack                                                               */
/* ------------------------------------------------------------------------ */

/* softplus(v) = log(1 + exp(v)), written in the overflow-free but
 * mathematically identical form (reading Q4). */
static double softplus_d(double v) {
    return v > 0.0 ? v + log1p(exp(-v)) : log1p(exp(v));
}

static int is_head(const int32_t* pos_row, int64_t t) {
    return t == 0 || pos_row[t] == 0;
}

/* Eq 1a/1b/2a:  h_t = A-bar_t h_{t-1} + B-bar_t x_t,
 * y_t = C_t h_t (+ D x_t, reading Q3), A-bar = exp(delta A) and, per
 * north_star / reading Q1, B-bar x = delta B x (Euler).  At heads
 * A-bar := 0 (Alg 2), i.e. the state restarts from B-bar x. */
void pmo_scan_fwd(const double* u, const double* dt, const double* A,
                  const double* B, const double* C, const double* D,
                  const double* dt_bias, int32_t softplus, const int32_t* pos,
                  double* y, double* h_out,
                  int64_t R, int64_t Dn, int64_t L, int32_t N) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t r = 0; r < R; ++r)
        for (int64_t d = 0; d < Dn; ++d) {
            double* h = (double*)calloc((size_t)N, sizeof(double));
            const int64_t lane = (r * Dn + d) * L;
            for (int64_t t = 0; t < L; ++t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                double x = u[lane + t];
                double yt = 0.0;
                for (int32_t n = 0; n < N; ++n) {
                    double abar = is_head(pos + r * L, t) ? 0.0
                                                          : exp(delta * A[d * N + n]);
                    double bx = delta * B[(r * N + n) * L + t] * x;
                    h[n] = is_head(pos + r * L, t) ? bx : abar * h[n] + bx;
                    yt += C[(r * N + n) * L + t] * h[n];
                    if (h_out) h_out[(lane + t) * N + n] = h[n];
                }
                if (y) y[lane + t] = yt + (D ? D[d] : 0.0) * x;
            }
            free(h);
        }
}

/* Reverse-mode adjoint of pmo_scan_fwd for rows [r0, r1) ("another two scan
 * operators, where modifications only require setting A-bar -> 0"):
 *   g_t = C_t dy_t + A-bar_{t+1} g_{t+1}        (A-bar = 0 at heads)
 *   dA  += delta_t * g_t * A-bar_t * h_{t-1}    (post-reset A-bar, Q16)
 *   dB_t = sum_d g_t delta_t x_t,  dC_t = sum_d dy_t h_t,  dD = sum dy x
 *   d delta_t = x_t sum_n g B + sum_n A g A-bar_t h_{t-1}
 *   ddt = d delta * softplus'(v) = d delta * sigmoid(v). */
void pmo_scan_bwd_rows(const double* u, const double* dt, const double* A,
                       const double* B, const double* C, const double* D,
                       const double* dt_bias, int32_t softplus,
                       const int32_t* pos, const double* dy,
                       double* du, double* ddt, double* dA, double* dB,
                       double* dC, double* dD, double* ddt_bias,
                       int64_t R, int64_t Dn, int64_t L, int32_t N,
                       int64_t r0, int64_t r1) {
    (void)R;
    const int nth = pmo_num_threads();
    /* thread-private partials for the cross-channel sums, reduced in a
     * fixed order afterwards */
    const size_t bc = (size_t)(r1 - r0) * (size_t)N * (size_t)L;
    double* pB = (double*)calloc((size_t)nth * bc, sizeof(double));
    double* pC = (double*)calloc((size_t)nth * bc, sizeof(double));
    for (int64_t i = 0; i < Dn * N; ++i) dA[i] = 0.0;
    for (int64_t d = 0; d < Dn; ++d) {
        if (dD) dD[d] = 0.0;
        if (ddt_bias) ddt_bias[d] = 0.0;
    }
#pragma omp parallel for schedule(static)
    for (int64_t d = 0; d < Dn; ++d) {
#ifdef _OPENMP
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
        double* hs = (double*)malloc(sizeof(double) * (size_t)(L * N));
        double* as = (double*)malloc(sizeof(double) * (size_t)(L * N));
        double* g = (double*)malloc(sizeof(double) * (size_t)N);
        double* carry = (double*)malloc(sizeof(double) * (size_t)N);
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t lane = (r * Dn + d) * L;
            const int32_t* pr = pos + r * L;
            double* myB = pB + (size_t)tid * bc + (size_t)(r - r0) * N * L;
            double* myC = pC + (size_t)tid * bc + (size_t)(r - r0) * N * L;
            /* forward: keep h_t and post-reset A-bar_t for this lane */
            for (int32_t n = 0; n < N; ++n) g[n] = 0.0;
            for (int64_t t = 0; t < L; ++t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                for (int32_t n = 0; n < N; ++n) {
                    double abar = is_head(pr, t) ? 0.0 : exp(delta * A[d * N + n]);
                    double bx = delta * B[(r * N + n) * L + t] * u[lane + t];
                    double hprev = t > 0 ? hs[(t - 1) * N + n] : 0.0;
                    hs[t * N + n] = is_head(pr, t) ? bx : abar * hprev + bx;
                    as[t * N + n] = abar;
                }
            }
            /* reverse */
            for (int32_t n = 0; n < N; ++n) carry[n] = 0.0;
            for (int64_t t = L - 1; t >= 0; --t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                double x = u[lane + t], gy = dy[lane + t];
                double S = 0.0, dq = 0.0;
                for (int32_t n = 0; n < N; ++n) {
                    g[n] = C[(r * N + n) * L + t] * gy + carry[n];
                    S += g[n] * B[(r * N + n) * L + t];
                    double hprev = t > 0 ? hs[(t - 1) * N + n] : 0.0;
                    double q = g[n] * as[t * N + n] * hprev;
                    dq += A[d * N + n] * q;
                    dA[d * N + n] += delta * q; /* lane d is owned by one thread */
                    myB[n * L + t] += g[n] * delta * x;
                    myC[n * L + t] += gy * hs[t * N + n];
                    carry[n] = as[t * N + n] * g[n];
                }
                du[lane + t] = (D ? D[d] : 0.0) * gy + delta * S;
                double ddelta = x * S + dq;
                double gd = ddelta * (softplus ? sigmoid_d(v) : 1.0);
                ddt[lane + t] = gd;
                if (dD) dD[d] += gy * x;
                if (ddt_bias) ddt_bias[d] += gd;
            }
        }
        free(hs); free(as); free(g); free(carry);
    }
    for (int64_t r = r0; r < r1; ++r)
        for (int32_t n = 0; n < N; ++n)
            for (int64_t t = 0; t < L; ++t) {
                double sb = 0.0, sc = 0.0;
                for (int k = 0; k < nth; ++k) {
                    sb += pB[(size_t)k * bc + ((size_t)(r - r0) * N + n) * L + t];
                    sc += pC[(size_t)k * bc + ((size_t)(r - r0) * N + n) * L + t];
                }
                dB[(r * N + n) * L + t] = sb;
                dC[(r * N + n) * L + t] = sc;
            }
    free(pB);
    free(pC);
}

void pmo_scan_bwd(const double* u, const double* dt, const double* A,
                  const double* B, const double* C, const double* D,
                  const double* dt_bias, int32_t softplus, const int32_t* pos,
                  const double* dy,
                  double* du, double* ddt, double* dA, double* dB, double* dC,
                  double* dD, double* ddt_bias,
                  int64_t R, int64_t Dn, int64_t L, int32_t N) {
    pmo_scan_bwd_rows(u, dt, A, B, C, D, dt_bias, softplus, pos, dy, du, ddt,
                      dA, dB, dC, dD, ddt_bias, R, Dn, L, N, 0, R);
}

/* Eq 3, with x_k read as B-bar_k x_k (reading Q2) and the sum
 * starting at the segment head s(t) (the reset makes every product that
 * spans a head vanish):
 *   h_t = sum_{k=s(t)}^{t} (prod_{i=k+1}^{t} A-bar_i) delta_k B_k x_k. */
void pmo_scan_fwd_eq3(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus,
                      const int32_t* pos, double* y,
                      int64_t R, int64_t Dn, int64_t L, int32_t N) {
    for (int64_t r = 0; r < R; ++r)
        for (int64_t d = 0; d < Dn; ++d) {
            const int64_t lane = (r * Dn + d) * L;
            for (int64_t t = 0; t < L; ++t) {
                int64_t s = t;
                while (!is_head(pos + r * L, s)) --s;
                double yt = 0.0;
                for (int32_t n = 0; n < N; ++n) {
                    double h = 0.0;
                    for (int64_t k = s; k <= t; ++k) {
                        double prod = 1.0;
                        for (int64_t i = k + 1; i <= t; ++i) {
                            double vi = dt[lane + i] + (dt_bias ? dt_bias[d] : 0.0);
                            double di = softplus ? softplus_d(vi) : vi;
                            prod *= exp(di * A[d * N + n]);
                        }
                        double vk = dt[lane + k] + (dt_bias ? dt_bias[d] : 0.0);
                        double dk = softplus ? softplus_d(vk) : vk;
                        h += prod * dk * B[(r * N + n) * L + k] * u[lane + k];
                    }
                    yt += C[(r * N + n) * L + t] * h;
                }
                y[lane + t] = yt + (D ? D[d] : 0.0) * u[lane + t];
            }
        }
}

/* ------------------------------------------------------------------------ */
/* O2: the unpacked, per-sequence textbook operators (no position indices).  */
/* Used by the PUI pin f(S) = unpack(f(pack(S))).               */
/* One sequence: x,u,dt,y,... (Dn, Ls); B, C (N, Ls).                        */
/* ------------------------------------------------------------------------ */

/* causal depthwise conv with zero left padding (the unmodified operator the
 * paper starts from, "the convolution kernel sliding"). */
void pmo_seq_conv_fwd(const double* x, const double* w, const double* bias,
                      double* out, int64_t Dn, int64_t Ls, int32_t K,
                      int32_t silu) {
    for (int64_t d = 0; d < Dn; ++d)
        for (int64_t t = 0; t < Ls; ++t) {
            double pre = bias ? bias[d] : 0.0;
            for (int32_t j = 0; j < K; ++j) {
                int64_t src = t - (K - 1 - j);
                double xv = src >= 0 ? x[d * Ls + src] : 0.0; /* zero pad */
                pre += w[d * K + j] * xv;
            }
            out[d * Ls + t] = silu ? pre * sigmoid_d(pre) : pre;
        }
}

/* its adjoint; dw, dbias ACCUMULATE (callers sum over sequences) */
void pmo_seq_conv_bwd(const double* x, const double* w, const double* bias,
                      const double* dout, double* dx, double* dw,
                      double* dbias, int64_t Dn, int64_t Ls, int32_t K,
                      int32_t silu) {
    double* dpre = (double*)malloc(sizeof(double) * (size_t)(Ls > 0 ? Ls : 1));
    for (int64_t d = 0; d < Dn; ++d) {
        for (int64_t t = 0; t < Ls; ++t) {
            double pre = bias ? bias[d] : 0.0;
            for (int32_t j = 0; j < K; ++j) {
                int64_t src = t - (K - 1 - j);
                pre += w[d * K + j] * (src >= 0 ? x[d * Ls + src] : 0.0);
            }
            double g = 1.0;
            if (silu) {
                double s = sigmoid_d(pre);
                g = s * (1.0 + pre * (1.0 - s));
            }
            dpre[t] = dout[d * Ls + t] * g;
        }
        for (int64_t s = 0; s < Ls; ++s) {
            double acc = 0.0;
            for (int32_t o = 0; o < K; ++o) { /* output t = s + o via tap K-1-o */
                int64_t t = s + o;
                if (t < Ls) acc += w[d * K + (K - 1 - o)] * dpre[t];
            }
            dx[d * Ls + s] = acc;
        }
        for (int64_t t = 0; t < Ls; ++t) {
            for (int32_t j = 0; j < K; ++j) {
                int64_t src = t - (K - 1 - j);
                if (src >= 0) dw[d * K + j] += dpre[t] * x[d * Ls + src];
            }
            if (dbias) dbias[d] += dpre[t];
        }
    }
    free(dpre);
}

/* Eq 1a/1b/2a for one sequence, h_{-1} = 0, no reset. */
void pmo_seq_scan_fwd(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, double* y,
                      int64_t Dn, int64_t Ls, int32_t N) {
    double* h = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t d = 0; d < Dn; ++d) {
        for (int32_t n = 0; n < N; ++n) h[n] = 0.0;
        for (int64_t t = 0; t < Ls; ++t) {
            double v = dt[d * Ls + t] + (dt_bias ? dt_bias[d] : 0.0);
            double delta = softplus ? softplus_d(v) : v;
            double x = u[d * Ls + t], yt = 0.0;
            for (int32_t n = 0; n < N; ++n) {
                h[n] = exp(delta * A[d * N + n]) * h[n] + delta * B[n * Ls + t] * x;
                yt += C[n * Ls + t] * h[n];
            }
            y[d * Ls + t] = yt + (D ? D[d] : 0.0) * x;
        }
    }
    free(h);
}

/* adjoint of pmo_seq_scan_fwd; dA, dD, ddt_bias ACCUMULATE, dB/dC overwrite */
void pmo_seq_scan_bwd(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus,
                      const double* dy, double* du, double* ddt, double* dA,
                      double* dB, double* dC, double* dD, double* ddt_bias,
                      int64_t Dn, int64_t Ls, int32_t N) {
    double* hs = (double*)malloc(sizeof(double) * (size_t)((Ls + 1) * N));
    double* g = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t i = 0; i < N * Ls; ++i) { dB[i] = 0.0; dC[i] = 0.0; }
    for (int64_t d = 0; d < Dn; ++d) {
        /* hs[(t+1)*N + n] = h_t, hs[n] = h_{-1} = 0 */
        for (int32_t n = 0; n < N; ++n) hs[n] = 0.0;
        for (int64_t t = 0; t < Ls; ++t) {
            double v = dt[d * Ls + t] + (dt_bias ? dt_bias[d] : 0.0);
            double delta = softplus ? softplus_d(v) : v;
            for (int32_t n = 0; n < N; ++n)
                hs[(t + 1) * N + n] = exp(delta * A[d * N + n]) * hs[t * N + n] +
                                      delta * B[n * Ls + t] * u[d * Ls + t];
        }
        for (int32_t n = 0; n < N; ++n) g[n] = 0.0;
        for (int64_t t = Ls - 1; t >= 0; --t) {
            double v = dt[d * Ls + t] + (dt_bias ? dt_bias[d] : 0.0);
            double delta = softplus ? softplus_d(v) : v;
            double x = u[d * Ls + t], gy = dy[d * Ls + t];
            double S = 0.0, dq = 0.0;
            for (int32_t n = 0; n < N; ++n) {
                /* g currently holds dL/dh_{t+1} * abar_{t+1}; add C_t dy_t */
                g[n] += C[n * Ls + t] * gy;
                double abar = exp(delta * A[d * N + n]);
                double q = g[n] * abar * hs[t * N + n];
                S += g[n] * B[n * Ls + t];
                dq += A[d * N + n] * q;
                dA[d * N + n] += delta * q;
                dB[n * Ls + t] += g[n] * delta * x;
                dC[n * Ls + t] += gy * hs[(t + 1) * N + n];
                g[n] = abar * g[n];
            }
            du[d * Ls + t] = (D ? D[d] : 0.0) * gy + delta * S;
            double gd = (x * S + dq) * (softplus ? sigmoid_d(v) : 1.0);
            ddt[d * Ls + t] = gd;
            if (dD) dD[d] += gy * x;
            if (ddt_bias) ddt_bias[d] += gd;
        }
    }
    free(hs);
    free(g);
}

/* ------------------------------------------------------------------------ */
/* NEXT-1 / NEXT-2: the full selective-scan signature.        */
/*   z (R,Dn,L) or NULL : gate, out = y * silu(z) (the paper's element-wise   */
/*                        sigmoid op; Fig 1)                          */
/*   h0 (R,Dn,N) or NULL: state entering t = 0 of each row when that slot is  */
/*                        NOT a sequence start (pos[r,0] != 0) -- the state   */
/*                        passing between cut parts of a long sequence that   */
/*                        the paper plans as future work             */
/*   h_last (R,Dn,N) or NULL: state after step L-1 of each row               */
/* head(r,t) := pos[r,t] == 0 || (t == 0 && h0 == NULL).                     */
/* ------------------------------------------------------------------------ */

static int is_head_ext(const int32_t* pos_row, int64_t t, const double* h0) {
    return pos_row[t] == 0 || (t == 0 && h0 == NULL);
}

/* Eq 2b: f(z) = (e^z - 1)/z, the factor with bbar = f(delta A) delta B;
 * Taylor 1 + z/2 + z^2/6 below |z| = 1e-4. */
static double zoh_f(double z) {
    return fabs(z) < 1e-4 ? 1.0 + z / 2.0 + z * z / 6.0 : expm1(z) / z;
}
/* f'(z) = (e^z - f(z)) / z = (z e^z - e^z + 1) / z^2; Taylor below 1e-3 */
static double zoh_df(double z) {
    return fabs(z) < 1e-3 ? 0.5 + z / 3.0 + z * z / 8.0 + z * z * z / 30.0
                          : (exp(z) - zoh_f(z)) / z;
}

void pmo_scan_fwd_ext(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, int32_t zoh,
                      const int32_t* pos, const double* z, const double* h0,
                      double* out, double* h_last, double* decay,
                      int64_t R, int64_t Dn, int64_t L, int32_t N) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t r = 0; r < R; ++r)
        for (int64_t d = 0; d < Dn; ++d) {
            double* h = (double*)calloc((size_t)N, sizeof(double));
            /* P = d h_last / d h0 = product of the recurrence multipliers */
            double* P = (double*)malloc(sizeof(double) * (size_t)N);
            for (int32_t n = 0; n < N; ++n) P[n] = 1.0;
            const int64_t lane = (r * Dn + d) * L;
            if (h0)
                for (int32_t n = 0; n < N; ++n) h[n] = h0[(r * Dn + d) * N + n];
            for (int64_t t = 0; t < L; ++t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                double x = u[lane + t];
                double yt = 0.0;
                const int head = is_head_ext(pos + r * L, t, h0);
                for (int32_t n = 0; n < N; ++n) {
                    /* Euler (Q1): bbar = delta B;  ZOH (Eq 2b): bbar = f(delta A) delta B */
                    double bfac = zoh ? zoh_f(delta * A[d * N + n]) * delta : delta;
                    double bx = bfac * B[(r * N + n) * L + t] * x;
                    h[n] = head ? bx : exp(delta * A[d * N + n]) * h[n] + bx;
                    P[n] = head ? 0.0 : exp(delta * A[d * N + n]) * P[n];
                    yt += C[(r * N + n) * L + t] * h[n];
                }
                yt += (D ? D[d] : 0.0) * x;
                if (z) {
                    double zz = z[lane + t];
                    yt = yt * zz * sigmoid_d(zz);
                }
                out[lane + t] = yt;
            }
            if (h_last)
                for (int32_t n = 0; n < N; ++n) h_last[(r * Dn + d) * N + n] = h[n];
            if (decay)
                for (int32_t n = 0; n < N; ++n) decay[(r * Dn + d) * N + n] = P[n];
            free(h);
            free(P);
        }
}

/* Adjoint of pmo_scan_fwd_ext.  dout is the cotangent of `out`; dh_last
 * (or NULL) the cotangent of h_last.  Extra outputs: dz (if z), dh0 (if h0).
 * Param grads (dA, dD, ddt_bias) and dB, dC are overwritten sums. */
void pmo_scan_bwd_ext(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, int32_t zoh,
                      const int32_t* pos, const double* z, const double* h0,
                      const double* dout, const double* dh_last,
                      double* du, double* ddt, double* dA, double* dB,
                      double* dC, double* dD, double* ddt_bias, double* dz,
                      double* dh0, int64_t R, int64_t Dn, int64_t L, int32_t N) {
    const int nth = pmo_num_threads();
    const size_t bc = (size_t)R * (size_t)N * (size_t)L;
    double* pB = (double*)calloc((size_t)nth * bc, sizeof(double));
    double* pC = (double*)calloc((size_t)nth * bc, sizeof(double));
    for (int64_t i = 0; i < Dn * N; ++i) dA[i] = 0.0;
    for (int64_t d = 0; d < Dn; ++d) {
        if (dD) dD[d] = 0.0;
        if (ddt_bias) ddt_bias[d] = 0.0;
    }
#pragma omp parallel for schedule(static)
    for (int64_t d = 0; d < Dn; ++d) {
#ifdef _OPENMP
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
        double* hs = (double*)malloc(sizeof(double) * (size_t)((L + 1) * N));
        double* as = (double*)malloc(sizeof(double) * (size_t)(L * N));
        double* g = (double*)malloc(sizeof(double) * (size_t)N);
        double* carry = (double*)malloc(sizeof(double) * (size_t)N);
        for (int64_t r = 0; r < R; ++r) {
            const int64_t lane = (r * Dn + d) * L;
            const int32_t* pr = pos + r * L;
            double* myB = pB + (size_t)tid * bc + (size_t)r * N * L;
            double* myC = pC + (size_t)tid * bc + (size_t)r * N * L;
            /* forward: hs[(t+1)N + n] = h_t, hs[n] = h_{-1} (h0 or 0) */
            for (int32_t n = 0; n < N; ++n) hs[n] = h0 ? h0[(r * Dn + d) * N + n] : 0.0;
            for (int64_t t = 0; t < L; ++t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                const int head = is_head_ext(pr, t, h0);
                for (int32_t n = 0; n < N; ++n) {
                    double abar = head ? 0.0 : exp(delta * A[d * N + n]);
                    double bfac = zoh ? zoh_f(delta * A[d * N + n]) * delta : delta;
                    double bx = bfac * B[(r * N + n) * L + t] * u[lane + t];
                    hs[(t + 1) * N + n] = head ? bx : abar * hs[t * N + n] + bx;
                    as[t * N + n] = abar;
                }
            }
            for (int32_t n = 0; n < N; ++n) carry[n] = dh_last ? dh_last[(r * Dn + d) * N + n] : 0.0;
            for (int64_t t = L - 1; t >= 0; --t) {
                double v = dt[lane + t] + (dt_bias ? dt_bias[d] : 0.0);
                double delta = softplus ? softplus_d(v) : v;
                double x = u[lane + t];
                /* y_t (pre-gate) and the gate's chain rule */
                double yt = (D ? D[d] : 0.0) * x;
                for (int32_t n = 0; n < N; ++n)
                    yt += C[(r * N + n) * L + t] * hs[(t + 1) * N + n];
                double gy = dout[lane + t];
                if (z) {
                    double zz = z[lane + t], s = sigmoid_d(zz);
                    dz[lane + t] = gy * yt * s * (1.0 + zz * (1.0 - s));
                    gy = gy * zz * s;
                }
                /* du = D gy + sum_n g B bfac (Euler: delta * sum_n g B);
                 * Sd = sum_n g B d(bfac)/d(delta) */
                double Sb = 0.0, Sd = 0.0, dq = 0.0;
                for (int32_t n = 0; n < N; ++n) {
                    const double Bn = B[(r * N + n) * L + t];
                    const double zn = delta * A[d * N + n];
                    /* bfac = delta (Euler) or f(z) delta = (e^z - 1)/A (ZOH):
                     * d bfac/d delta = 1 or e^z;  d bfac/dA = 0 or delta^2 f'(z) */
                    const double bfac = zoh ? zoh_f(zn) * delta : delta;
                    const double dbdd = zoh ? exp(zn) : 1.0;
                    g[n] = C[(r * N + n) * L + t] * gy + carry[n];
                    Sb += zoh ? g[n] * Bn * bfac : g[n] * Bn;
                    Sd += g[n] * Bn * dbdd;
                    double q = g[n] * as[t * N + n] * hs[t * N + n];
                    dq += A[d * N + n] * q;
                    dA[d * N + n] += delta * q;
                    if (zoh) dA[d * N + n] += g[n] * Bn * x * delta * delta * zoh_df(zn);
                    myB[n * L + t] += g[n] * bfac * x;
                    myC[n * L + t] += gy * hs[(t + 1) * N + n];
                    carry[n] = as[t * N + n] * g[n];
                }
                du[lane + t] = (D ? D[d] : 0.0) * gy + (zoh ? Sb : delta * Sb);
                double gd = (x * Sd + dq) * (softplus ? sigmoid_d(v) : 1.0);
                ddt[lane + t] = gd;
                if (dD) dD[d] += gy * x;
                if (ddt_bias) ddt_bias[d] += gd;
            }
            /* carry now holds abar_0 * g_0 = dL/dh_{-1} (0 when t = 0 is a head) */
            if (dh0)
                for (int32_t n = 0; n < N; ++n) dh0[(r * Dn + d) * N + n] = carry[n];
        }
        free(hs); free(as); free(g); free(carry);
    }
    for (int64_t r = 0; r < R; ++r)
        for (int32_t n = 0; n < N; ++n)
            for (int64_t t = 0; t < L; ++t) {
                double sb = 0.0, sc = 0.0;
                for (int k = 0; k < nth; ++k) {
                    sb += pB[(size_t)k * bc + ((size_t)r * N + n) * L + t];
                    sc += pC[(size_t)k * bc + ((size_t)r * N + n) * L + t];
                }
                dB[(r * N + n) * L + t] = sb;
                dC[(r * N + n) * L + t] = sc;
            }
    free(pB);
    free(pC);
}
