// scan_impl.cuh -- shared declarations of the ScanOp_pack kernels (Alg 2
// P:172-185, Eq 1a/1b/2a P:202-205, sec 3.4 P:199-224 of arXiv 2408.03865).
//
// Design:
//  * forward: one thread = one (row, channel) lane holding all N states in
//    registers, sequential in time; a CTA = 128 consecutive channels of one
//    row, so the head predicate is CTA-uniform (no divergence) and B/C/pos
//    tiles are staged once in shared memory (fp32) and broadcast;
//  * time parallelism comes from the packing itself: a row is split at
//    sequence heads into independent segments (sequences never span
//    rows, and the reset cuts every carry), so no carry fix-up and no
//    redundant exponentials are needed; segments are scheduled
//    longest-first on persistent CTAs;
//  * the reset is a select on the CTA-uniform head flag (h = b), never a
//    multiply by 0, so NaN/Inf and -0 cannot cross a boundary;
//  * forward saves the state every kChunk steps ("reused Mamba's structure
//    for handling hidden_state"); backward walks chunks in reverse,
//    parks every step's state of the chunk in TMEM, runs the reverse
//    recurrence g_t = C_t dy_t + abar_{t+1} g_{t+1} (abar = 0 at heads,
//    P:224) and reduces dB/dC over channels with a warp transpose through
//    shared memory, then over warps, into per-channel-block partials that a
//    finalize kernel sums in a fixed order (deterministic).
//  * scan_fwd.cu holds the forward + schedule kernels, scan_bwd.cu the
//    backward, scan.cu the C ABI (validation, workspace layout).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <type_traits>

#include "common.cuh"

namespace pm {

#ifndef PM_FWD_THREADS
#define PM_FWD_THREADS 128
#endif
#ifndef PM_FWD_MINB
#define PM_FWD_MINB 4
#endif
constexpr int kScanThreads = PM_FWD_THREADS;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kTile = 64;   // fwd staging tile (time steps)
constexpr int kChunk = 16;  // checkpoint interval (time steps)
constexpr int kFwdMinB = PM_FWD_MINB;  // resident fwd CTAs per SM (register cap 128)
#ifndef PM_BWD_MINB
#define PM_BWD_MINB 4
#endif
constexpr int kBwdMinB = PM_BWD_MINB;  // resident bwd CTAs per SM (register cap 128; smem fits 4)

#ifndef PM_BWD_CH
#define PM_BWD_CH 64
#endif
constexpr int kBwdCh = PM_BWD_CH;            // channels per CTA
constexpr int kBwdThreads = 2 * kBwdCh;      // lane pair per channel
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr int kRedStride = 32;               // float4 per transpose row (no padding)
constexpr int kBSub = 2;                     // bwd register sub-chunk (= one reduction round)
constexpr int kBNSub = kChunk / kBSub;
static_assert(kChunk == 16, "phase 1 maps 8 steps to each thread of a pair");

struct ScanFwdArgs {
  const void* u;
  const void* dt;
  const float* A;
  const void* B;
  const void* C;
  const float* Dskip;
  const float* dt_bias;
  const int32_t* pos;
  void* y;
  float* states;
  const int4* items;  // length-sorted segment list {r, k, s0, s1} (NULL: grid mode)
  int* counter;       // work counter for the persistent loop
  int* done;          // per-segment finished channel blocks (persistent mode)
  int n_items;
  int R, Dn, L, nseg, nchunk, softplus;
  const void* z;      // NEXT-1 gate (R,Dn,L) or NULL: y <- y * silu(z)
  const float* h0;    // NEXT-2 state entering t=0 (R,Dn,N) or NULL
  float* h_last;      // state after step L-1 (R,Dn,N) or NULL
  float* decay;       // d h_last / d h0 (R,Dn,N) or NULL (NEXT-2 row summary)
  int zoh;             // NEXT-4: Eq 2b discretisation of B-bar (else Euler, Q1)
};

struct ScanBwdArgs {
  const void* u;
  const void* dt;
  const float* A;
  const void* B;
  const void* C;
  const float* Dskip;
  const float* dt_bias;
  const int32_t* pos;
  const float* states;
  const void* dy;
  void* du;
  void* ddt;
  float* ws_bc;     // (nDblk, R, L, 2N)
  float* ws_param;  // (R*nseg, N+2, Dn)
  const int4* items;  // length-sorted segment list {r, k, s0, s1} (NULL: grid mode)
  int* counter;       // counters[1] of the schedule: work counter; counter[1]: CTAs exited
  const int* done;    // the fwd's per-segment released channel counts (complete at Dn)
  int n_items;
  int R, Dn, L, nseg, nchunk, softplus;
  const void* z;        // NEXT-1 gate (R,Dn,L) or NULL; dy is then d(out)
  const float* h0;      // NEXT-2 state entering t=0 (R,Dn,N) or NULL
  const float* dh_last; // cotangent of the state after step L-1 or NULL
  void* dz;             // (R,Dn,L) when z != NULL
  float* dh0;           // (R,Dn,N) when h0 != NULL
  int zoh;              // NEXT-4: Eq 2b discretisation of B-bar (else Euler, Q1)
  const float* psum;    // time split: part summaries (R*nseg, 2, N, Dn) or NULL
  int nparts;           // parts per segment (1: no time split)
  // TMA descriptors of the per-chunk inputs (vector path; use_tma = 0 falls
  // back to cp.async): (L, Dn, R) u/dt/dy/z, (L, N, R) B/C, (L, R) pos,
  // (Dn, N, nchunk, R) states
  int use_tma;
  int pdl;  // launched programmatically behind the library's own forward (pm.h)
  int wide; // scan_bwd2.cu's two-channels-per-thread kernel (TMA maps boxed for kWideCh)
  CUtensorMap tm_u, tm_dt, tm_dy, tm_z, tm_B, tm_C, tm_pos, tm_st;
};

// ---------------------------------------------------------------------------
// Stage B, C (converted to fp32, time-major [t][n]) and head flags for the
// time window [j0, j0 + W) of row r into shared memory.
template <typename T, int N, int W, bool kVec, int S = N>  // S: row stride of sB/sC
PM_DEV void stage_bc(const T* __restrict__ B_r, const T* __restrict__ C_r,
                     const int32_t* __restrict__ pos_row, int L, int j0,
                     float (*sB)[S], float (*sC)[S], unsigned* sMask, bool t0_head) {
  static_assert(W % 8 == 0, "window must be a multiple of 8");
  for (int e = threadIdx.x; e < N * (W / 8); e += blockDim.x) {
    const int n = e % N, tb = (e / N) * 8;
    float vb[8], vc[8];
    load8<T, kVec>(B_r + (int64_t)n * L, j0 + tb, L, vb);
    load8<T, kVec>(C_r + (int64_t)n * L, j0 + tb, L, vc);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sB[tb + i][n] = vb[i];
      sC[tb + i][n] = vc[i];
    }
  }
  // head flags of the window as a bitmask (warp 0 ballots 32 steps at a time)
  if (threadIdx.x < 32) {
#pragma unroll
    for (int w0 = 0; w0 < W; w0 += 32) {
      const int t = j0 + w0 + (int)threadIdx.x;
      const bool f = (w0 + (int)threadIdx.x < W) &&
                     ((t >= L) || (t == 0 && t0_head) || __ldg(pos_row + t) == 0);
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (threadIdx.x == 0) sMask[w0 / 32] = m;
    }
  }
}


// The same staging split in two: tile_fetch() loads this thread's share of
// the window [j0, j0 + W) into registers (issued a whole tile ahead, so the
// global latency overlaps the previous tile's steps), tile_commit() converts
// it into shared memory and builds the head mask (between the caller's two
// barriers).  Shares: vector e = threadIdx.x (+ blockDim.x ...) of
// N * W / 8 8-step vectors; warp 0 holds pos of W steps (W / 32 per lane).
template <typename T, int N, int W, bool kVec>
struct TileRegs {
  static constexpr int kPer = (N * (W / 8) + 127) / 128;  // vectors per thread at 128 threads
  Raw8<T, kVec> b[kPer], c[kPer];
  int p[W / 32];
  PM_DEV void fetch(const T* __restrict__ B_r, const T* __restrict__ C_r,
                    const int32_t* __restrict__ pos_row, int L, int j0) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < N * (W / 8)) {
        const int n = e % N, tb = (e / N) * 8;
        b[k].load(B_r + (int64_t)n * L, j0 + tb, L);
        c[k].load(C_r + (int64_t)n * L, j0 + tb, L);
      }
    }
    if (threadIdx.x < 32) {
#pragma unroll
      for (int w = 0; w < W / 32; ++w) {
        const int t = j0 + w * 32 + (int)threadIdx.x;
        p[w] = t < L ? __ldg(pos_row + t) : 0;
      }
    }
  }
  template <int S>
  PM_DEV void commit(int L, int j0, float (*sB)[S], float (*sC)[S], unsigned* sMask,
                     bool t0_head) const {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < N * (W / 8)) {
        const int n = e % N, tb = (e / N) * 8;
        float vb[8], vc[8];
        b[k].unpack(vb);
        c[k].unpack(vc);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          sB[tb + i][n] = vb[i];
          sC[tb + i][n] = vc[i];
        }
      }
    }
    if (threadIdx.x < 32) {
#pragma unroll
      for (int w = 0; w < W / 32; ++w) {
        const int t = j0 + w * 32 + (int)threadIdx.x;
        const bool f = t >= L || (t == 0 && t0_head) || p[w] == 0;
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (threadIdx.x == 0) sMask[w] = m;
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Raw inputs of one backward chunk of kBwdCh channels (shared by the backward kernel and its staging helper)
template <typename T, int N, bool kGate>
struct BwdRaw {  // raw inputs of one chunk, filled by TMA or cp.async (vector path)
  alignas(128) T u[kBwdCh][kChunk];
  alignas(128) T dt[kBwdCh][kChunk];
  alignas(128) T dy[kBwdCh][kChunk];
  alignas(128) T B[N][kChunk];
  alignas(128) T C[N][kChunk];
  alignas(128) int32_t pos[kChunk];
  alignas(128) float st[N][kBwdCh];
  alignas(128) T z[kGate ? kBwdCh : 1][kChunk];
};

// Issue the cp.async copies of chunk c's raw inputs (vector path only:
// L*isz % 16 == 0, Dn % 4 == 0, 16-byte aligned pointers).
template <typename T, int N, bool kGate>
PM_DEV void bwd_issue_raw(BwdRaw<T, N, kGate>& rw, const ScanBwdArgs& a, int r, int dblk, int c,
                          int s0, bool cont0, uint64_t* bar) {
  constexpr int kEl = 16 / (int)sizeof(T);       // elements per 16-byte chunk
  constexpr int kRowQ = kChunk / kEl;            // chunks per (row, chunk)
  const int L = a.L, Dn = a.Dn, cb = c * kChunk;
  // the chunk's start state: inside the item, or at its start when the item
  // continues a sequence (h0 at slot 0; a time-split part inside a row)
  const bool with_st = cb > s0 || (cb == 0 && a.h0 != nullptr) || (cb == s0 && cont0);
  if (a.use_tma) {  // one thread issues the chunk's bulk tensor copies
    if (threadIdx.x == 0) {
      constexpr uint32_t kRows = kBwdCh * kChunk * sizeof(T);
      const uint32_t bytes = (kGate ? 4 : 3) * kRows + 2 * N * kChunk * sizeof(T) +
                             kChunk * sizeof(int32_t) + (with_st ? N * kBwdCh * sizeof(float) : 0);
      mbar_expect_tx(bar, bytes);
      const int d0 = dblk * kBwdCh;
      tma_load<3>(rw.u, &a.tm_u, bar, cb, d0, r);
      tma_load<3>(rw.dt, &a.tm_dt, bar, cb, d0, r);
      tma_load<3>(rw.dy, &a.tm_dy, bar, cb, d0, r);
      if constexpr (kGate) tma_load<3>(rw.z, &a.tm_z, bar, cb, d0, r);
      tma_load<3>(rw.B, &a.tm_B, bar, cb, 0, r);
      tma_load<3>(rw.C, &a.tm_C, bar, cb, 0, r);
      tma_load<2>(rw.pos, &a.tm_pos, bar, cb, r);
      if (with_st) tma_load<4>(rw.st, &a.tm_st, bar, d0, 0, c, r);
    }
    return;
  }
  constexpr int kTx = kBwdCh * kRowQ;
#pragma unroll
  for (int arr = 0; arr < (kGate ? 4 : 3); ++arr) {  // u, dt, dy (, z)
    const T* base = static_cast<const T*>(arr == 0 ? a.u : arr == 1 ? a.dt : arr == 2 ? a.dy : a.z);
    T(*dst)[kChunk] = arr == 0 ? rw.u : arr == 1 ? rw.dt : arr == 2 ? rw.dy : rw.z;
    for (int e = threadIdx.x; e < kTx; e += blockDim.x) {
      const int ch = e / kRowQ, q = e % kRowQ;
      const int d = dblk * kBwdCh + ch;
      const int t0 = cb + q * kEl;
      const bool ok = d < Dn && t0 < L;
      const T* src = ok ? base + ((int64_t)r * Dn + d) * L + t0 : base;
      cp_async16(&dst[ch][q * kEl], src, ok ? 16 : 0);
    }
  }
  const T* Bp = static_cast<const T*>(a.B) + (int64_t)r * N * L;
  const T* Cp = static_cast<const T*>(a.C) + (int64_t)r * N * L;
  for (int e = threadIdx.x; e < 2 * N * kRowQ; e += blockDim.x) {
    const int arr = e / (N * kRowQ), rem = e % (N * kRowQ), n = rem / kRowQ, q = rem % kRowQ;
    const int t0 = cb + q * kEl;
    const bool ok = t0 < L;
    const T* src = (arr == 0 ? Bp : Cp) + (int64_t)n * L + (ok ? t0 : 0);
    cp_async16(&(arr == 0 ? rw.B : rw.C)[n][q * kEl], src, ok ? 16 : 0);
  }
  for (int e = threadIdx.x; e < kChunk / 4; e += blockDim.x) {
    const int t0 = cb + 4 * e;
    const bool ok = t0 < L;
    cp_async16(&rw.pos[4 * e], a.pos + (int64_t)r * L + (ok ? t0 : 0), ok ? 16 : 0);
  }
  if (with_st) {
    for (int e = threadIdx.x; e < N * (kBwdCh / 4); e += blockDim.x) {
      const int n = e / (kBwdCh / 4), q = e % (kBwdCh / 4);
      const int d0 = dblk * kBwdCh + 4 * q;
      const bool ok = d0 < Dn;
      const float* src = a.states + (((int64_t)r * a.nchunk + c) * N + n) * Dn + (ok ? d0 : 0);
      cp_async16(&rw.st[n][4 * q], src, ok ? 16 : 0);
    }
  }
  cp_async_commit();
}

// ---------------------------------------------------------------------------
// host-side helpers shared by the three translation units
// ---------------------------------------------------------------------------
inline int n_chunks(int64_t L) { return (int)((L + kChunk - 1) / kChunk); }
inline int n_dblk(int64_t Dn) { return (int)((Dn + kScanThreads - 1) / kScanThreads); }
inline int n_dblk_bwd(int64_t Dn) { return (int)((Dn + kBwdCh - 1) / kBwdCh); }
// the wide backward (scan_bwd2.cu): 128 channels per CTA, two per thread
constexpr int kWideCh = 128;
inline int n_dblk_wide(int64_t Dn) { return (int)((Dn + kWideCh - 1) / kWideCh); }

// Forward launch shape.  Throughput-bound when the mean load per CTA slot
// (R*L*ceil(Dn/128) step-items over nsm*kFwdMinB slots) is >= 0.3 L: one
// thread per channel (S = 1) and the backward launched programmatically
// behind it.  Otherwise a few long segments are the critical path: S =
// kFwdSplit threads per channel (N/S states each) and a serialized backward.
// PM_FWD_SPLIT=1|S overrides the choice (A/B).
template <int N> constexpr int kFwdSplit = N >= 8 ? 4 : 2;
inline bool fwd_throughput_bound(int64_t R, int64_t L, int64_t Dn) {
  const int64_t load = R * L * ((Dn + kScanThreads - 1) / kScanThreads) / ((int64_t)sm_count() * kFwdMinB);
  return 10 * load >= 3 * L;
}
inline int fwd_split(int64_t R, int64_t L, int64_t Dn, int N) {
  const int sp = N >= 8 ? 4 : 2;
  if (const char* e = getenv("PM_FWD_SPLIT")) return atoi(e) > 1 ? sp : 1;
  return fwd_throughput_bound(R, L, Dn) ? 1 : sp;
}

// Segments per row: nominal cut every 256 steps (cuts snap to heads, so with
// the paper's length distribution a segment is ~one sequence), <= 64.
inline int n_seg(int64_t L) { return (int)std::max<int64_t>(1, std::min<int64_t>(64, L / 256)); }

// Backward time split (latency-bound launches): a segment longer than
// kPartLen steps is cut into up to kMaxParts parts at chunk boundaries, so the
// longest sequence no longer sets the backward's critical path.  Every part
// starts from the forward's checkpoint at its start; the carry entering its
// end comes from a reverse pre-pass over the following parts (tsplit.cu, the
// NEXT-2 context-parallel algebra applied inside a row).  PM_TSPLIT=0|1
// overrides.  (The forward stays unsplit: its prefix fix-up measured dearer
// than the critical path it saves -- DESIGN.md.)
#ifndef PM_MAX_PARTS
#define PM_MAX_PARTS 4
#endif
constexpr int kMaxParts = PM_MAX_PARTS;
#ifndef PM_PART_LEN
#define PM_PART_LEN 384
#endif
constexpr int kPartLen = PM_PART_LEN;
inline int n_parts(int64_t R, int64_t L, int64_t Dn) {
  if (const char* e = getenv("PM_TSPLIT")) return atoi(e) > 0 ? kMaxParts : 1;
  return fwd_throughput_bound(R, L, Dn) ? 1 : kMaxParts;
}
// backward work items per row (segments x parts)
inline int n_slots(int64_t R, int64_t L, int64_t Dn) { return n_seg(L) * n_parts(R, L, Dn); }

// states buffer = fp32 chunk states | 256 B counters | per-segment done
// counts | sorted segment list | unsorted segment list (the fwd writes the
// schedule; the bwd reuses it unless it splits segments in time).
// counters[0]: fwd work counter; [1]: bwd work counter; [2]: bwd CTAs exited
// (the last one resets [1] and [2], so the bwd needs no memset of its own and
// can launch programmatically right behind the fwd).  done[r*nseg+k]: fwd
// channels finished on segment (r,k) -- a bwd item starts once its segment's
// count reaches Dn.
inline size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
inline size_t states_f32_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return (size_t)R * n_chunks(L) * N * Dn * sizeof(float);
}
inline size_t done_bytes(int64_t R, int64_t L) { return up256((size_t)R * n_seg(L) * sizeof(int)); }
inline size_t list_bytes(int64_t n) { return up256((size_t)n * 16); }
inline size_t sched_bytes(int64_t R, int64_t L) {
  return 256 + done_bytes(R, L) + 2 * list_bytes(R * n_seg(L));
}
inline size_t state_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return up256(states_f32_bytes(R, Dn, L, N)) + sched_bytes(R, L);
}
struct Sched {
  int* counters;
  int* done;
  int4* sorted;
  int4* unsorted;
};
inline Sched sched_of(void* states, int64_t R, int64_t Dn, int64_t L, int32_t N) {
  char* b = static_cast<char*>(states) + up256(states_f32_bytes(R, Dn, L, N));
  Sched sc;
  sc.counters = reinterpret_cast<int*>(b);
  sc.done = reinterpret_cast<int*>(b + 256);
  b += 256 + done_bytes(R, L);
  sc.sorted = reinterpret_cast<int4*>(b);
  sc.unsorted = reinterpret_cast<int4*>(b + list_bytes(R * n_seg(L)));
  return sc;
}
// part summaries of the backward time split: (R*nslot, 2, N, Dn) fp32,
// {the part's local dLoss/dh0, decay = prod abar over the part}
inline size_t psum_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return n_parts(R, L, Dn) > 1 ? up256((size_t)R * n_slots(R, L, Dn) * 2 * N * Dn * sizeof(float))
                               : 0;
}

inline bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline pm_status check_common(int64_t R, int64_t Dn, int64_t L, int32_t N, pm_dtype io) {
  if (R < 1 || Dn < 1 || L < 1) return PM_ERR_INVALID_ARG;
  if (io != PM_F32 && io != PM_BF16) return PM_ERR_DTYPE;
  if (N != 4 && N != 8 && N != 16) return PM_ERR_UNSUPPORTED;
  if (R * L >= (int64_t(1) << 31) || Dn >= (int64_t(1) << 31)) return PM_ERR_SHAPE;
  if (R > 65535 || R * n_seg(L) * kMaxParts * ((Dn + kBwdCh - 1) / kBwdCh) >= (int64_t(1) << 31))
    return PM_ERR_SHAPE;
  return PM_OK;
}

inline bool elem_aligned(const void* p, pm_dtype io) {
  const uintptr_t m = io == PM_F32 ? 3u : 1u;
  return p == nullptr || (reinterpret_cast<uintptr_t>(p) & m) == 0;
}


// launchers (scan_fwd.cu / scan_bwd.cu)
pm_status run_scan_fwd(const ScanFwdArgs& a, int N, bool vec, pm_dtype io, cudaStream_t s);
pm_status run_scan_bwd(const ScanBwdArgs& a, int N, bool vec, pm_dtype io, float* dA, float* dB,
                       float* dC, float* dD, float* ddtb, cudaStream_t s);
pm_status launch_scan_bwd_wide(const ScanBwdArgs& a, pm_dtype io, cudaStream_t s);
// backward time split (tsplit.cu): plan the parts (unsorted/sorted lists),
// zero the work counters, run the reverse pre-pass that writes every part's
// summary into a.psum
pm_status run_part_bwd_pre(const ScanBwdArgs& a, int4* unsorted, int4* sorted, int* counters,
                           int N, bool vec, pm_dtype io, cudaStream_t s);
// the schedule kernels (scan_fwd.cu)
void launch_schedule(const int32_t* pos, int R, int L, int nseg, int P, int4* unsorted,
                     int4* sorted, cudaStream_t s);

}  // namespace pm
