/*
 * pm.h -- C ABI of libpm: PackMamba's packed causal conv1d + selective scan
 * (arXiv 2408.03865) for NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source,
 *            "S:n" = line n of SPEC.md.  Readings "Qn" are listed in
 *            DESIGN.md ("Readings of the paper").
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ---------------------------------------------------------------------------
 * Layout (reading Q13; the paper's "(B, D, L)"):
 *   x, u, dt, y, dy, du, ddt, dx, out, dout : (R, Dn, L)  L innermost
 *   B, C (inputs, dtype io), dB, dC (fp32)  : (R, N, L)   shared by channels
 *   pos  (position_indices, int32)          : (R, L)
 *   A, dA (fp32)                            : (Dn, N)
 *   Dskip, dt_bias, bias, dD, ddt_bias, dbias (fp32) : (Dn)
 *   w, dw (fp32)                            : (Dn, K)
 * R = number of packed rows ("packs"), L = pack length, Dn = d_inner,
 * N = d_state, K = conv width.
 *
 * Segment heads: head(r,t) := pos[r,t] == 0 || t == 0.  Both operators reset
 * there (Alg 1, Alg 2, reading Q9).  pos contents are NOT
 * validated; the semantics hold for any int32 array.
 *
 * I/O dtype (pm_dtype) applies to the per-token tensors x,u,dt,B,C,y,dy,du,
 * ddt,dx,out,dout.  All arithmetic is fp32; parameters and parameter
 * gradients (A, Dskip, dt_bias, w, bias, dA, dD, ddt_bias, dw, dbias) and
 * dB, dC are fp32 (reading Q12).  bf16 outputs are rounded to nearest even.
 *
 * Ownership: every pointer is caller-owned device memory (except *_host),
 * contiguous, element-aligned; the library never allocates or frees device
 * memory and keeps no pointer after the call returns.  Parameter-gradient
 * outputs are OVERWRITTEN, not accumulated.
 *
 * Execution: all device work is enqueued on `stream` (a cudaStream_t; NULL =
 * legacy default stream) without host synchronisation, except pm_pack which
 * copies its host plan with kernel parameters (no sync either).  Arguments
 * are validated before anything is enqueued: on error nothing is written.
 * Launch failures return PM_ERR_CUDA; faults inside kernels surface at the
 * caller's next synchronisation.  The library has no mutable global state and
 * is reentrant.
 *
 * Limits: K in [1, 4]; N in {4, 8, 16}; R, Dn, L >= 1; R*L < 2^31;
 * R*Dn*L < 2^62.  The vector fast path is taken when L*isz % 16 == 0 and the
 * per-token pointers are 16-byte aligned; otherwise a scalar path runs.
 */
#ifndef PM_H
#define PM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PM_API __attribute__((visibility("default")))
#else
#define PM_API
#endif

typedef struct CUstream_st* pm_stream_t; /* == cudaStream_t */

typedef enum {
    PM_OK = 0,
    PM_ERR_INVALID_ARG = 1, /* NULL pointer, non-positive size            */
    PM_ERR_CAPACITY = 2,    /* sequence longer than the pack */
    PM_ERR_SHAPE = 3,       /* inconsistent sizes    */
    PM_ERR_DTYPE = 4,       /* unknown pm_dtype                           */
    PM_ERR_ALIGN = 5,       /* pointer not aligned to its element size    */
    PM_ERR_UNSUPPORTED = 6, /* K or N outside the supported set           */
    PM_ERR_CUDA = 7,        /* a CUDA launch failed                       */
    PM_ERR_WORKSPACE = 8    /* workspace missing or smaller than queried  */
} pm_status;

typedef enum { PM_F32 = 0, PM_BF16 = 1 } pm_dtype;

PM_API const char* pm_status_string(pm_status s);
PM_API const char* pm_version(void);

/* ===========================================================================
 * Packing  (sec 3.1; sec 5)
 * ===========================================================================
 * pm_plan_fifo -- host only.  "sequentially packing sequences in the received
 * order, sealing the pack when it cannot fit the next sequence".  A
 * sequence that exactly fills the remaining space fits (Q17).
 *   seq_lens_host[n_seqs]   lengths, each in [1, pack_len] else
 *                           PM_ERR_CAPACITY ("no instances of
 *                           sequences spanning across packed sequences").
 *   seq_row_host/seq_off_host[n_seqs] (out, may be NULL): row and slot offset.
 *   n_rows_out (out): number of rows.
 * pm_plan_greedy -- host only.  The paper's "local greedy algorithm that
 * sorts ... before packing" as first-fit-decreasing over the whole
 * batch, ties by id.  Same arguments and errors.
 */
PM_API pm_status pm_plan_fifo(const int32_t* seq_lens_host, int64_t n_seqs,
                       int64_t pack_len, int64_t* seq_row_host,
                       int64_t* seq_off_host, int64_t* n_rows_out);
PM_API pm_status pm_plan_greedy(const int32_t* seq_lens_host, int64_t n_seqs,
                         int64_t pack_len, int64_t* seq_row_host,
                         int64_t* seq_off_host, int64_t* n_rows_out);

/* pm_pack -- "concatenating the input tensor along the sequence dimension to
 * obtain a packed_sequence and the auxiliary structure position_indices"
 * (P:120).  FIFO plan on the host, then a device scatter:
 *   src_dev      (sum(len), record_bytes) token-major records, sequences
 *                concatenated in id order (e.g. token ids, record_bytes=4).
 *   dst_dev      (n_rows, pack_len, record_bytes): sequence data laid out
 *                contiguously per row in plan order, padding bytes = 0.
 *   pos_dev      (n_rows, pack_len) int32: 0..len-1 per sequence, 0 on
 *                padding (padding convention Q8).
 *   max_rows     capacity of dst_dev/pos_dev in rows; PM_ERR_CAPACITY if the
 *                plan needs more.
 * Query mode: dst_dev == NULL && pos_dev == NULL computes only *n_rows_out
 * (and the optional seq_row/seq_off) without touching the device.
 * Output is bit-exact (integer/byte work). */
PM_API pm_status pm_pack(const int32_t* seq_lens_host, int64_t n_seqs,
                  int64_t pack_len, const void* src_dev, int64_t record_bytes,
                  void* dst_dev, int32_t* pos_dev, int64_t max_rows,
                  int64_t* n_rows_out, int64_t* seq_row_host,
                  int64_t* seq_off_host, pm_stream_t stream);

/* Same scatter for a caller-supplied plan (e.g. from pm_plan_greedy):
 * seq_row_host/seq_off_host must describe non-overlapping in-range slots. */
PM_API pm_status pm_pack_planned(const int32_t* seq_lens_host, int64_t n_seqs,
                          int64_t pack_len, const int64_t* seq_row_host,
                          const int64_t* seq_off_host, int64_t n_rows,
                          const void* src_dev, int64_t record_bytes,
                          void* dst_dev, int32_t* pos_dev, pm_stream_t stream);

/* ===========================================================================
 * conv1d_pack  (Alg 1; sec 3.3)
 * ===========================================================================
 * Forward:  pre[r,d,t] = bias[d] + sum_{j=0}^{K-1} w[d,j] * x[r,d,t-o]
 *           over taps o = K-1-j with  o <= pos[r,t]  and  t-o >= 0  (the
 *           "terminated early" boundary taps of Alg 1, reading Q6);
 *           out = silu ? pre * sigmoid(pre) : pre.
 *   bias may be NULL (0).  out may not alias x. */
PM_API pm_status pm_causal_conv1d_fwd(const void* x, const float* w,
                               const float* bias, const int32_t* pos,
                               void* out, int64_t R, int64_t Dn, int64_t L,
                               int32_t K, pm_dtype io, int32_t silu,
                               pm_stream_t stream);

/* Backward ("additional modifications ... to calculate dx and dweight
 * ... require reverse indices", read from the position indices of the next
 * K-1 slots, reading Q7):
 *   dpre = dout * d(out)/d(pre);
 *   dx[r,d,s] = sum_{o: s+o<L, o<=pos[r,s+o]} w[d,K-1-o] * dpre[r,d,s+o];
 *   dw[d,j]   = sum_{r,t, tap valid} dpre[r,d,t] * x[r,d,t-(K-1-j)];
 *   dbias[d]  = sum_{r,t} dpre[r,d,t]      (dbias may be NULL).
 * dw/dbias are overwritten.  workspace: >= pm_causal_conv1d_bwd_workspace()
 * bytes of device memory (16-byte aligned), contents undefined on return. */
PM_API size_t pm_causal_conv1d_bwd_workspace(int64_t R, int64_t Dn, int64_t L,
                                      int32_t K);
PM_API pm_status pm_causal_conv1d_bwd(const void* x, const float* w,
                               const float* bias, const int32_t* pos,
                               const void* dout, void* dx, float* dw,
                               float* dbias, int64_t R, int64_t Dn, int64_t L,
                               int32_t K, pm_dtype io, int32_t silu,
                               void* workspace, size_t ws_bytes,
                               pm_stream_t stream);

/* ===========================================================================
 * ScanOp_pack  (Alg 2; Eq 1a/1b/2a P:202-205; sec 3.4)
 * ===========================================================================
 * Forward, per (r, d) lane and state n:
 *   v = dt[r,d,t] + dt_bias[d];  delta = dt_softplus ? softplus(v) : v  (Q4)
 *   abar = head(r,t) ? 0 : exp(delta * A[d,n])        (Eq 2a; Alg 2)
 *   h_n  = head(r,t) ? delta*B[r,n,t]*u : abar*h_n + delta*B[r,n,t]*u
 *                                                   (Eq 1a; Euler B, Q1)
 *   y[r,d,t] = sum_n C[r,n,t]*h_n + Dskip[d]*u[r,d,t] (Eq 1b + skip, Q3)
 * The reset makes the recurrence a segmented associative scan.
 *   Dskip, dt_bias may be NULL (0).
 *   states (optional, may be NULL): pm_selective_scan_state_bytes() bytes,
 *     16-byte aligned: the fp32 chunk-boundary states written for the
 *     backward pass ("reused Mamba's structure for handling hidden_state",
 *     P:234) plus the length-sorted segment schedule that lets both passes
 *     run persistent, longest-first.  Layout is private to the library; pass
 *     the same buffer to the backward pass.  With states == NULL the forward
 *     runs a plain grid (no schedule). */
PM_API size_t pm_selective_scan_state_bytes(int64_t R, int64_t Dn, int64_t L,
                                     int32_t N);
PM_API pm_status pm_selective_scan_fwd(const void* u, const void* dt,
                                const float* A, const void* B, const void* C,
                                const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos,
                                void* y, float* states, int64_t R, int64_t Dn,
                                int64_t L, int32_t N, pm_dtype io,
                                pm_stream_t stream);

/* Backward ("another two scan operators, where modifications only require
 * setting A-bar_{position_indices=0} -> 0"):
 *   g_t  = C_t dy_t + abar_{t+1} g_{t+1}       (abar = 0 at heads)
 *   du   = Dskip*dy + delta * sum_n g B
 *   ddt  = (u * sum_n g B + sum_n A g abar_t h_{t-1}) * softplus'(v)
 *   dA[d,n] = sum_{r,t} delta g abar_t h_{t-1}  (post-reset abar, Q16)
 *   dB[r,n,t] = sum_d g delta u,  dC[r,n,t] = sum_d dy h_t
 *   dD[d] = sum_{r,t} dy u,  ddt_bias[d] = sum_{r,t} ddt
 * dA, dB, dC are required; dD, ddt_bias may be NULL.  All are overwritten.
 * states: the buffer filled by pm_selective_scan_fwd on the SAME inputs, or
 *   NULL to recompute it (then the workspace must also hold the states).
 *   The chunk states are only read; the backward claims its work items
 *   through the schedule counters kept in the same buffer (zeroed by the
 *   forward, reset by the backward's last CTA), so one states buffer must
 *   not be used by two backward calls running concurrently.  This entry
 *   point launches the backward in plain stream order (it never overlaps
 *   whatever kernel precedes it); pm_selective_scan_fwd_bwd below runs the
 *   forward and the backward as one call and overlaps them.  With
 *   states == NULL the library runs the forward itself right before the
 *   backward and overlaps the two the same way.  A states buffer whose
 *   forward did not complete makes the backward trap (sticky CUDA error at
 *   the next synchronisation) instead of reading unwritten states.
 * workspace: >= pm_selective_scan_bwd_workspace(R, Dn, L, N, states==NULL)
 *   bytes of 16-byte aligned device memory. */
PM_API size_t pm_selective_scan_bwd_workspace(int64_t R, int64_t Dn, int64_t L,
                                       int32_t N, int32_t recompute_states);
PM_API pm_status pm_selective_scan_bwd(const void* u, const void* dt,
                                const float* A, const void* B, const void* C,
                                const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos,
                                float* states, const void* dy, void* du,
                                void* ddt, float* dA, float* dB, float* dC,
                                float* dD, float* ddt_bias, void* workspace,
                                size_t ws_bytes, int64_t R, int64_t Dn,
                                int64_t L, int32_t N, pm_dtype io,
                                pm_stream_t stream);

/* ===========================================================================
 * Extended scan: the fused gate and cross-row state passing
 *   (the element-wise sigmoid/silu gate of the Mamba
 *    block, P:135 and Fig 1; NEXT-2: "cut long sequences and pass the hidden
 *    state between the parts", the paper's future work)
 * ===========================================================================
 * Same recurrence as pm_selective_scan_fwd, with:
 *   zoh: 0 = Euler B-bar = delta*B (north_star, reading
 *     Q1); 1 = zero-order hold, Eq 2b:
 *       B-bar = f(z)*delta*B,  z = delta*A[d,n],  f(z) = (e^z - 1)/z
 *     (f evaluated as (abar - 1)/A for |z| >= 0.1 and by its Taylor series
 *     below, so f(0) = 1 and A = 0 is allowed).  The reset still selects
 *     h = B-bar*u at heads.
 *   z (optional, (R,Dn,L) io dtype):  out[r,d,t] = y[r,d,t] * silu(z[r,d,t]),
 *     silu(z) = z / (1 + exp(-z)); with z == NULL, out = y.
 *   h0 (optional, (R,Dn,N) fp32): the state entering slot 0 of each row.
 *     With h0 != NULL slot 0 is a head only when pos[r,0] == 0; otherwise it
 *     continues h0[r] (abar_0 = exp(delta_0 A)).  With h0 == NULL slot 0 is
 *     always a head (the base ABI).
 *   h_last (optional, (R,Dn,N) fp32): written with the state after slot L-1
 *     (the input of the next part of a cut sequence).
 *   decay (optional, (R,Dn,N) fp32): d h_last / d h0 = prod_t abar_t over the
 *     row -- exp(A[d,n] * sum_t delta_t) when no slot of the row is a head
 *     (under the h0 rule above), else 0.  With (decay, h_last) of a local
 *     pass (h0 = 0) the rows of a cut sequence compose as
 *     h_last = decay * h0 + h_last_local (the "(prod abar, h) row summaries"
 *     of a context-parallel scan).
 * At least one of out, states, h_last, decay must be non-NULL.  Pointers are device
 * memory owned by the caller; h0/h_last must not alias. */
PM_API pm_status pm_selective_scan_fwd_ex(const void* u, const void* dt,
                                   const float* A, const void* B,
                                   const void* C, const float* Dskip,
                                   const float* dt_bias, int32_t dt_softplus,
                                   int32_t zoh, const int32_t* pos,
                                   const void* z, const float* h0, void* out,
                                   float* states, float* h_last, float* decay,
                                   int64_t R, int64_t Dn,
                                   int64_t L, int32_t N, pm_dtype io,
                                   pm_stream_t stream);

/* Backward of pm_selective_scan_fwd_ex (same zoh), given dout = dLoss/d(out) and
 * dh_last = dLoss/d(h_last) (optional, (R,Dn,N) fp32; NULL = 0):
 *   dy  = dout * silu(z)                (dy = dout when z == NULL)
 *   dz  = dout * y * silu'(z),  silu'(z) = s (1 + z (1 - s)), s = sigmoid(z)
 *   the carry into slot L-1 starts at dh_last instead of 0;
 *   dh0 (optional, (R,Dn,N) fp32) = dLoss/dh0 = abar_0 g_0 (0 when slot 0 is
 *     a head);
 * the other outputs as pm_selective_scan_bwd.  dz is required iff z != NULL
 * (io dtype, (R,Dn,L)).  states: the buffer filled by the forward pass on
 * the SAME inputs (incl. h0), or NULL to recompute.  Workspace as
 * pm_selective_scan_bwd_workspace(). */
PM_API pm_status pm_selective_scan_bwd_ex(const void* u, const void* dt,
                                   const float* A, const void* B,
                                   const void* C, const float* Dskip,
                                   const float* dt_bias, int32_t dt_softplus,
                                   int32_t zoh, const int32_t* pos,
                                   const void* z, const float* h0,
                                   float* states,
                                   const void* dout, const float* dh_last,
                                   void* du, void* ddt, float* dA, float* dB,
                                   float* dC, float* dD, float* ddt_bias,
                                   void* dz, float* dh0, void* workspace,
                                   size_t ws_bytes, int64_t R, int64_t Dn,
                                   int64_t L, int32_t N, pm_dtype io,
                                   pm_stream_t stream);

/* Forward + backward in one call (activation recompute in training: the
 * forward is re-run for its chunk states right before the backward):
 * exactly pm_selective_scan_fwd_ex(u, ..., out, states, h_last, decay)
 * followed by pm_selective_scan_bwd_ex(u, ..., states, dout, dh_last, ...) on
 * the same stream, with the same arguments and results.  Because the library
 * enqueues the backward directly behind its own forward, the backward is
 * launched programmatically (programmatic dependent launch) when the forward
 * is throughput-bound: backward CTAs start on the SMs the forward's last CTAs
 * leave and wait per segment until the forward has released that segment's
 * states.  Every input of the backward other than the states was written
 * before the forward started, and the backward's outputs (du, ddt, dA, dB,
 * dC, dD, ddt_bias, dz, dh0, workspace) must not overlap the forward's
 * outputs (out, h_last, decay) or any input: overlapping buffers return
 * PM_ERR_INVALID_ARG.  states is required (pm_selective_scan_state_bytes);
 * out, h_last, decay may be NULL.  PM_NO_PDL=1 in the environment serializes
 * the two launches (A/B measurements). */
PM_API pm_status pm_selective_scan_fwd_bwd(const void* u, const void* dt,
                                    const float* A, const void* B,
                                    const void* C, const float* Dskip,
                                    const float* dt_bias, int32_t dt_softplus,
                                    int32_t zoh, const int32_t* pos,
                                    const void* z, const float* h0, void* out,
                                    float* states, float* h_last, float* decay,
                                    const void* dout, const float* dh_last,
                                    void* du, void* ddt, float* dA, float* dB,
                                    float* dC, float* dD, float* ddt_bias,
                                    void* dz, float* dh0, void* workspace,
                                    size_t ws_bytes, int64_t R, int64_t Dn,
                                    int64_t L, int32_t N, pm_dtype io,
                                    pm_stream_t stream);

/* ===========================================================================
 * Context-parallel scan over cut sequences (the paper's
 * future work: "cut long sequences into multiple parts and pass the
 * hidden state between these parts ... parallel strategies for infinitely
 * long sequences")
 * ===========================================================================
 * A sequence longer than a pack is laid out over consecutive rows; row r
 * continues row r-1 iff pos[r,0] != 0 (its position indices keep counting:
 * with h0 given, slot 0 is a head only when pos[r,0] == 0), or as `cont[r]`
 * says when cont != NULL (cont[0]: row 0 continues the external state h_init).
 * The recurrence is linear in the state entering a row, so
 *   1. pm_selective_scan_fwd_ex with h0 = 0 (zeros, not NULL), states, h_last
 *      and decay gives every row's LOCAL pass and its summary (decay, h_last);
 *   2. pm_scan_chain_fwd composes the summaries along the chains into the
 *      true state entering every row, h_in[r] = decay[r-1] h_in[r-1] +
 *      h_last_local[r-1] (h_in[0] = h_init or 0), and the true h_last;
 *   3. pm_selective_scan_fwd_fixup adds C_t . (prod_{i<=t} abar_i) h_in to
 *      out over each continuing row's PREFIX (the slots before its first
 *      head) and the same state correction to the prefix's chunk states --
 *      no other slot changes, since a head resets the state.
 * Backward: pm_selective_scan_dh0 gives each row's local dLoss/dh0 from its
 * own outputs (reverse walk over the prefix), pm_scan_chain_bwd composes the
 * cotangent of every row's h_last, G[r] = dh_last_ext[r] + dh0_local[r+1] +
 * decay[r+1] G[r+1] when row r+1 continues row r, and
 * pm_selective_scan_bwd_ex(h0 = h_in, states = the fixed-up states,
 * dh_last = G) gives every gradient of the cut sequence.
 * Across GPUs the same two composition kernels run on one summary per rank
 * (cont != NULL, one "row" per rank): (chain_decay, h_last of its last row)
 * forward, (chain_decay, dh_init) backward -- exchanged by one all_gather.
 * All buffers (R,Dn,N) / (Dn,N) fp32, device memory, caller-owned. */

/* h_in[r] (state entering row r), h_last[r] (true state after row r, or
 * NULL) and chain_decay (Dn,N) = d h_last[R-1] / d h_init (or NULL) from the
 * local summaries decay, h_last_local (R,Dn,N).  h_init (Dn,N) or NULL = 0.
 * pos (R,L) is read only when cont == NULL (then L is its row length). */
PM_API pm_status pm_scan_chain_fwd(const int32_t* pos, const int32_t* cont,
                                   const float* decay, const float* h_last_local,
                                   const float* h_init, float* h_in, float* h_last,
                                   float* chain_decay, int64_t R, int64_t Dn,
                                   int64_t L, int32_t N, pm_stream_t stream);
/* dh_last[r] (R,Dn,N) = G[r], the cotangent of h_last[r] for the backward,
 * from the rows' local dh0 (pm_selective_scan_dh0), the external cotangents
 * dh_last_ext (R,Dn,N) or NULL, and g_end (Dn,N) or NULL: the cotangent of
 * h_last[R-1] from beyond the last row (the next rank).  dh_init (Dn,N) or
 * NULL receives dLoss/dh_init. */
PM_API pm_status pm_scan_chain_bwd(const int32_t* pos, const int32_t* cont,
                                   const float* decay, const float* dh0_local,
                                   const float* dh_last_ext, const float* g_end,
                                   float* dh_last, float* dh_init, int64_t R,
                                   int64_t Dn, int64_t L, int32_t N,
                                   pm_stream_t stream);
/* In place on out (R,Dn,L, io dtype; out = y or y*silu(z)) and states (the
 * forward's buffer or NULL): for every row with pos[r,0] != 0, every slot t
 * before its first head gets out += C_t . (prod_{i<=t} abar_i) h_in[r]
 * (x silu(z_t) with z != NULL) and every chunk checkpoint of that prefix the
 * state correction.  Rows with pos[r,0] == 0 are not touched.  Arguments as
 * pm_selective_scan_fwd_ex (same dt_softplus, A, dt_bias, z). */
PM_API pm_status pm_selective_scan_fwd_fixup(const void* dt, const float* A,
                                             const void* C, const float* dt_bias,
                                             int32_t dt_softplus, const int32_t* pos,
                                             const void* z, const float* h_in,
                                             void* out, float* states, int64_t R,
                                             int64_t Dn, int64_t L, int32_t N,
                                             pm_dtype io, pm_stream_t stream);
/* dh0_local (R,Dn,N) = dLoss/dh0 of each row through its own outputs only:
 * sum over the slots t before the row's first head of
 * prod_{i<=t} abar_i * C_t * dy_t, dy = dout (* silu(z) with z != NULL);
 * 0 for rows with pos[r,0] == 0. */
PM_API pm_status pm_selective_scan_dh0(const void* dt, const float* A, const void* C,
                                       const float* dt_bias, int32_t dt_softplus,
                                       const int32_t* pos, const void* z,
                                       const void* dout, float* dh0_local, int64_t R,
                                       int64_t Dn, int64_t L, int32_t N, pm_dtype io,
                                       pm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PM_H */
