/*
 * oracle.h -- fp64 CPU oracle for PackMamba's packed conv1d + selective scan.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2408_03865_b200/csrc); neither includes or links the other.
 *
 * Citations: "P:n" = PAPER.md line n (arXiv 2408.03865 LaTeX source),
 *            "S:n" = SPEC.md line n.  Readings of ambiguous passages are the
 *            ones listed in DESIGN.md section "Readings of the paper".
 *
 * Conventions (all arrays dense, row-major, caller-owned, host memory):
 *   x, u, dt, y, dy, du, ddt, dx : (R, Dn, L)   -- channel-major, L innermost
 *   B, C, dB, dC                 : (R, N, L)    -- shared by all channels
 *   pos                          : (R, L) int32 -- position_indices
 *   A, dA                        : (Dn, N)
 *   D, dt_bias, bias, dD, ...    : (Dn)
 *   w, dw                        : (Dn, K)
 * head(r,t) := pos[r,t] == 0 || t == 0                 (Alg 2, Q9)
 * conv tap j (0..K-1) reaches o = K-1-j slots back and is kept iff
 *   o <= pos[r,t] && t - o >= 0                          (Alg 1, Q6)
 *
 * Every function is sequential per (row, channel) lane; OpenMP (if enabled)
 * only distributes independent lanes.  No fast-math.
 */
#ifndef PM_ORACLE_H
#define PM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- packing (sec 3.1, sec 5) ------------- */
/* FIFO seal plan.  Returns 0 on success, 2 if a length is > cap or < 1.    */
int pmo_plan_fifo(const int32_t* lens, int64_t n, int64_t cap,
                  int64_t* seq_row, int64_t* seq_off, int64_t* n_rows);
/* First-fit-decreasing plan ("local greedy" P:273).  Same errors.
 * Rows are filled in first-fit order; within a row, sequences are laid out
 * in the order they were placed (descending length, ties by id).           */
int pmo_plan_ffd(const int32_t* lens, int64_t n, int64_t cap,
                 int64_t* seq_row, int64_t* seq_off, int64_t* n_rows);
/* Scatter token-major records into (n_rows, cap, rec_bytes); padding = 0,
 * pos = 0..len-1 within each sequence, 0 at padding.      */
void pmo_pack(const int32_t* lens, int64_t n, int64_t cap,
              const int64_t* seq_row, const int64_t* seq_off,
              const uint8_t* src, int64_t rec_bytes,
              uint8_t* dst, int32_t* pos, int64_t n_rows);

/* ---- conv1d_pack (Alg 1; sec 3.3) ------------------- */
void pmo_conv_fwd(const double* x, const double* w, const double* bias,
                  const int32_t* pos, double* out,
                  int64_t R, int64_t Dn, int64_t L, int32_t K, int32_t silu);
/* dw, dbias are overwritten (sum over rows and time).  bias may be NULL. */
void pmo_conv_bwd(const double* x, const double* w, const double* bias,
                  const int32_t* pos, const double* dout,
                  double* dx, double* dw, double* dbias,
                  int64_t R, int64_t Dn, int64_t L, int32_t K, int32_t silu);

/* ---- ScanOp_pack (Alg 2; Eqs 1a/1b/2a P:202-205; sec 3.4) ----- */
/* D, dt_bias may be NULL (treated as 0).  y may be NULL.
 * If h_out != NULL it receives h_t for every (r, d, t, n) as (R,Dn,L,N).   */
void pmo_scan_fwd(const double* u, const double* dt, const double* A,
                  const double* B, const double* C, const double* D,
                  const double* dt_bias, int32_t softplus, const int32_t* pos,
                  double* y, double* h_out,
                  int64_t R, int64_t Dn, int64_t L, int32_t N);
/* Adjoint of pmo_scan_fwd.  dA, dD, ddt_bias overwritten with sums
 * over (r, t); dB, dC overwritten with sums over channels.  Any of dD,
 * ddt_bias may be NULL.                                                     */
void pmo_scan_bwd(const double* u, const double* dt, const double* A,
                  const double* B, const double* C, const double* D,
                  const double* dt_bias, int32_t softplus, const int32_t* pos,
                  const double* dy,
                  double* du, double* ddt, double* dA, double* dB, double* dC,
                  double* dD, double* ddt_bias,
                  int64_t R, int64_t Dn, int64_t L, int32_t N);
/* Row-subset variants for large workloads: identical arithmetic, computed
 * only for rows [r0, r1) of the (R, ...) arrays; param grads summed over
 * those rows only.                                                          */
void pmo_scan_bwd_rows(const double* u, const double* dt, const double* A,
                       const double* B, const double* C, const double* D,
                       const double* dt_bias, int32_t softplus,
                       const int32_t* pos, const double* dy,
                       double* du, double* ddt, double* dA, double* dB,
                       double* dC, double* dD, double* ddt_bias,
                       int64_t R, int64_t Dn, int64_t L, int32_t N,
                       int64_t r0, int64_t r1);

/* ---- O3: Eq 3 brute force, O(L^2) (reading Q2) --------------- */
void pmo_scan_fwd_eq3(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus,
                      const int32_t* pos, double* y,
                      int64_t R, int64_t Dn, int64_t L, int32_t N);

/* ---- O2: unpacked per-sequence textbook operators (P:122-127 PUI) ------ */
/* One sequence: x,u,dt,y,dy,... (Dn, Ls); B, C, dB, dC (N, Ls).  No pos.
 * Conv uses zero left padding; scan starts from h_{-1} = 0.
 * Param grads (dw, dbias, dA, dD, ddt_bias) ACCUMULATE into the outputs so
 * callers can sum over sequences; dB, dC are overwritten.                  */
void pmo_seq_conv_fwd(const double* x, const double* w, const double* bias,
                      double* out, int64_t Dn, int64_t Ls, int32_t K,
                      int32_t silu);
void pmo_seq_conv_bwd(const double* x, const double* w, const double* bias,
                      const double* dout, double* dx, double* dw,
                      double* dbias, int64_t Dn, int64_t Ls, int32_t K,
                      int32_t silu);
void pmo_seq_scan_fwd(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, double* y,
                      int64_t Dn, int64_t Ls, int32_t N);
void pmo_seq_scan_bwd(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus,
                      const double* dy, double* du, double* ddt, double* dA,
                      double* dB, double* dC, double* dD, double* ddt_bias,
                      int64_t Dn, int64_t Ls, int32_t N);

/* ---- NEXT-1 / NEXT-2: gate z, state passing h0 / h_last; NEXT-4: ZOH ----- */
/* zoh != 0 selects Eq 2b for B-bar instead of the Euler reading Q1:
 *   bbar = f(z) * delta * B,  z = delta * A[d,n],  f(z) = (e^z - 1) / z,
 * with f(z) = 1 + z/2 + z^2/6 for |z| < 1e-4 (removable
 * singularity); f is evaluated with expm1 elsewhere.                       */
/* out = y * silu(z) if z != NULL (else y); h0 (R,Dn,N): state entering t=0
 * of a row whose slot 0 is not a sequence start (P:275 future work);
 * head(r,t) := pos[r,t]==0 || (t==0 && h0==NULL).  h_last (R,Dn,N): state
 * after step L-1.  Backward: dout = cotangent of out, dh_last (or NULL) of
 * h_last; outputs dz (if z) and dh0 (if h0) in addition.                    */
void pmo_scan_fwd_ext(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, int32_t zoh,
                      const int32_t* pos, const double* z, const double* h0,
                      double* out, double* h_last, double* decay,
                      int64_t R, int64_t Dn, int64_t L, int32_t N);
void pmo_scan_bwd_ext(const double* u, const double* dt, const double* A,
                      const double* B, const double* C, const double* D,
                      const double* dt_bias, int32_t softplus, int32_t zoh,
                      const int32_t* pos, const double* z, const double* h0,
                      const double* dout, const double* dh_last,
                      double* du, double* ddt, double* dA, double* dB,
                      double* dC, double* dD, double* ddt_bias, double* dz,
                      double* dh0, int64_t R, int64_t Dn, int64_t L, int32_t N);

/* number of OpenMP threads the oracle would use (1 if built without OpenMP) */
int pmo_num_threads(void);
void pmo_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif /* PM_ORACLE_H */
