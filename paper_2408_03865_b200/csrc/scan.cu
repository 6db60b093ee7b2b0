// scan.cu -- ScanOp_pack forward/backward for sm_100a (Alg 2 P:172-185,
// Eq 1a/1b/2a P:202-205, sec 3.4 P:199-224 of arXiv 2408.03865).
//
// Design:
//  * one thread = one (row, channel) lane holding all N states in registers,
//    sequential in time; a CTA = 128 consecutive channels of one row, so the
//    head predicate is CTA-uniform (no divergence) and B/C/pos tiles are
//    staged once in shared memory (fp32) and broadcast to all channels;
//  * time parallelism comes from the packing itself: a row is split at
//    sequence heads into independent segments (sequences never span
//    rows, and the reset cuts every carry), so no carry fix-up and no
//    redundant exponentials are needed;
//  * the reset is a select on the CTA-uniform head flag (h = b), never a
//    multiply by 0, so NaN/Inf and -0 cannot cross a boundary;
//  * forward saves the state every kChunk steps ("reused Mamba's structure
//    for handling hidden_state"); backward walks chunks in reverse,
//    recomputes kSub-step sub-chunks into registers, runs the reverse
//    recurrence g_t = C_t dy_t + abar_{t+1} g_{t+1} (abar = 0 at heads,
//    P:224) and reduces dB/dC over channels with a warp transpose through
//    shared memory, then over warps, into per-channel-block partials that a
//    finalize kernel sums in a fixed order (deterministic).
#include <algorithm>

#include "common.cuh"

namespace pm {

constexpr int kScanThreads = 128;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kTile = 64;   // fwd staging tile (time steps)
constexpr int kChunk = 16;  // checkpoint interval (time steps)
constexpr int kSub = 4;     // bwd register sub-chunk (time steps)
constexpr int kNSub = kChunk / kSub;

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
  int R, Dn, L, nseg, nchunk, softplus;
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
  int R, Dn, L, nseg, nchunk, softplus;
};

// Stage B, C (converted to fp32, time-major [t][n]) and head flags for the
// time window [j0, j0 + W) of row r into shared memory.
template <typename T, int N, int W, bool kVec>
PM_DEV void stage_bc(const T* __restrict__ B_r, const T* __restrict__ C_r,
                     const int32_t* __restrict__ pos_row, int L, int j0,
                     float (*sB)[N], float (*sC)[N], int* sHead) {
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
  for (int e = threadIdx.x; e < W; e += blockDim.x) {
    const int t = j0 + e;
    sHead[e] = (t >= L) ? 1 : (t == 0 || __ldg(pos_row + t) == 0);
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <typename T, int N, bool kVec>
__global__ void __launch_bounds__(kScanThreads)
scan_fwd_kernel(const ScanFwdArgs a) {
  __shared__ __align__(16) float sB[kTile][N];
  __shared__ __align__(16) float sC[kTile][N];
  __shared__ int sHead[kTile];
  __shared__ int s_red[kScanWarps];

  const int r = blockIdx.y, k = blockIdx.z;
  const int L = a.L, Dn = a.Dn;
  const int d_raw = blockIdx.x * kScanThreads + threadIdx.x;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  const int32_t* pos_row = a.pos + (int64_t)r * L;

  int s0, s1;
  segment_bounds(pos_row, L, k, a.nseg, s_red, s0, s1);
  if (s0 >= s1) return;

  const T* B_r = static_cast<const T*>(a.B) + (int64_t)r * N * L;
  const T* C_r = static_cast<const T*>(a.C) + (int64_t)r * N * L;
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* u_row = static_cast<const T*>(a.u) + lane;
  const T* dt_row = static_cast<const T*>(a.dt) + lane;
  T* y_row = a.y ? static_cast<T*>(a.y) + lane : nullptr;

  float A2[N];
#pragma unroll
  for (int n = 0; n < N; ++n) A2[n] = __ldg(a.A + (int64_t)d * N + n) * kLog2e;
  const float Dd = a.Dskip ? __ldg(a.Dskip + d) : 0.f;
  const float bias = a.dt_bias ? __ldg(a.dt_bias + d) : 0.f;

  float h[N];
#pragma unroll
  for (int n = 0; n < N; ++n) h[n] = 0.f;

  for (int j0 = s0 & ~(kTile - 1); j0 < s1; j0 += kTile) {
    __syncthreads();
    stage_bc<T, N, kTile, kVec>(B_r, C_r, pos_row, L, j0, sB, sC, sHead);
    __syncthreads();
    const int t_lo = max(s0, j0), t_hi = min(s1, j0 + kTile);
    for (int sb = (t_lo - j0) & ~7; sb < t_hi - j0; sb += 8) {
      const int tb = j0 + sb;
      float uu[8], vv[8], yy[8];
      load8<T, kVec>(u_row, tb, L, uu);
      load8<T, kVec>(dt_row, tb, L, vv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = tb + i;
        yy[i] = 0.f;
        if (t < t_lo || t >= t_hi) continue;  // CTA-uniform
        if (a.states != nullptr && (t % kChunk) == 0 && active) {
          float* st = a.states + (((int64_t)r * a.nchunk + t / kChunk) * N) * Dn + d;
#pragma unroll
          for (int n = 0; n < N; ++n) st[(int64_t)n * Dn] = h[n];
        }
        const float v = vv[i] + bias;
        const float delta = a.softplus ? softplusf(v) : v;
        const float dux = delta * uu[i];
        float yv = Dd * uu[i];
        const float* Bt = sB[sb + i];
        const float* Ct = sC[sb + i];
        if (sHead[sb + i]) {
#pragma unroll
          for (int n = 0; n < N; ++n) h[n] = dux * Bt[n];
        } else {
#pragma unroll
          for (int n = 0; n < N; ++n) h[n] = fmaf(ex2(delta * A2[n]), h[n], dux * Bt[n]);
        }
#pragma unroll
        for (int n = 0; n < N; ++n) yv = fmaf(Ct[n], h[n], yv);
        yy[i] = yv;
      }
      if (active && y_row != nullptr) store8<T, kVec>(y_row, tb, t_lo, t_hi, yy);
    }
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
template <int N>
struct BwdSmem {
  static constexpr int kQ = (2 * N) / 4;          // float4 quads of (dB, dC) values
  static constexpr int kRows = kSub * kQ;         // transpose rows per warp
  float4 sub[kNSub][N / 4][kScanThreads];         // sub-chunk start states
  float4 red[kScanWarps][kRows][33];              // warp transpose (padded)
  float4 xw[2][kScanWarps][32];                   // cross-warp partials
  float B[kChunk][N];
  float C[kChunk][N];
  int head[kChunk];
  int s_red[kScanWarps];
};

template <typename T, int N, bool kVec>
__global__ void __launch_bounds__(kScanThreads, 2)
scan_bwd_kernel(const ScanBwdArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = BwdSmem<N>;
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  constexpr int kQ = SM::kQ;
  static_assert(kQ <= 8 && SM::kRows <= 32, "transpose rows must fit a warp");

  const int r = blockIdx.y, k = blockIdx.z, dblk = blockIdx.x;
  const int L = a.L, Dn = a.Dn;
  const int lid = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int d_raw = dblk * kScanThreads + threadIdx.x;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  const int32_t* pos_row = a.pos + (int64_t)r * L;
  float* wsp = a.ws_param + (int64_t)(r * a.nseg + k) * (N + 2) * Dn;

  int s0, s1;
  segment_bounds(pos_row, L, k, a.nseg, sm.s_red, s0, s1);
  if (s0 >= s1) {
    if (active) {
      for (int n = 0; n < N + 2; ++n) wsp[(int64_t)n * Dn + d] = 0.f;
    }
    return;
  }

  const T* B_r = static_cast<const T*>(a.B) + (int64_t)r * N * L;
  const T* C_r = static_cast<const T*>(a.C) + (int64_t)r * N * L;
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* u_row = static_cast<const T*>(a.u) + lane;
  const T* dt_row = static_cast<const T*>(a.dt) + lane;
  const T* dy_row = static_cast<const T*>(a.dy) + lane;
  T* du_row = static_cast<T*>(a.du) + lane;
  T* ddt_row = static_cast<T*>(a.ddt) + lane;
  float* ws_bc_r = a.ws_bc + ((int64_t)dblk * a.R + r) * (int64_t)L * (2 * N);

  float A2[N], g[N], dA[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    A2[n] = __ldg(a.A + (int64_t)d * N + n) * kLog2e;
    g[n] = 0.f;
    dA[n] = 0.f;
  }
  const float Dd = a.Dskip ? __ldg(a.Dskip + d) : 0.f;
  const float bias = a.dt_bias ? __ldg(a.dt_bias + d) : 0.f;
  float dD = 0.f, ddtb = 0.f;
  int xbuf = 0;

  const int cfirst = s0 / kChunk, clast = (s1 - 1) / kChunk;
  for (int c = clast; c >= cfirst; --c) {
    const int cb = c * kChunk, c0 = max(cb, s0), c1 = min(cb + kChunk, s1);
    __syncthreads();
    stage_bc<T, N, kChunk, kVec>(B_r, C_r, pos_row, L, cb, sm.B, sm.C, sm.head);
    // chunk start state (state before step cb); irrelevant when cb <= s0
    // because s0 is a head.
    float h[N];
    if (cb > s0) {
      const float* st = a.states + (((int64_t)r * a.nchunk + c) * N) * Dn + d;
#pragma unroll
      for (int n = 0; n < N; ++n) h[n] = st[(int64_t)n * Dn];
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n) h[n] = 0.f;
    }
    __syncthreads();

    // ---- pass A: forward over the chunk, record sub-chunk start states ----
#pragma unroll
    for (int sb = 0; sb < kChunk; sb += 8) {
      float uu[8], vv[8];
      load8<T, kVec>(u_row, cb + sb, L, uu);
      load8<T, kVec>(dt_row, cb + sb, L, vv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ii = sb + i, t = cb + ii;
        if (ii % kSub == 0) {
#pragma unroll
          for (int q = 0; q < N / 4; ++q)
            sm.sub[ii / kSub][q][threadIdx.x] =
                make_float4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
        }
        if (t < c0 || t >= c1) continue;
        const float v = vv[i] + bias;
        const float delta = a.softplus ? softplusf(v) : v;
        const float dux = delta * uu[i];
        const float* Bt = sm.B[ii];
        if (sm.head[ii]) {
#pragma unroll
          for (int n = 0; n < N; ++n) h[n] = dux * Bt[n];
        } else {
#pragma unroll
          for (int n = 0; n < N; ++n) h[n] = fmaf(ex2(delta * A2[n]), h[n], dux * Bt[n]);
        }
      }
    }

    // ---- pass B: sub-chunks in reverse ----
    for (int sc = kNSub - 1; sc >= 0; --sc) {
      const int a0 = cb + sc * kSub;
      if (a0 >= c1 || a0 + kSub <= c0) continue;  // CTA-uniform
      float uu[4], vv[4], yy[4];
      load4<T, kVec>(u_row, a0, L, uu);
      load4<T, kVec>(dt_row, a0, L, vv);
      load4<T, kVec>(dy_row, a0, L, yy);
      float dl[4], sg[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float v = vv[i] + bias;
        if (a.softplus) {
          dl[i] = softplusf(v);
          sg[i] = sigmoidf_fast(v);
        } else {
          dl[i] = v;
          sg[i] = 1.f;
        }
      }
      // recompute h_t and abar_t for the sub-chunk into registers
      float hb[kSub][N], ab[kSub][N];
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        const float4 s = sm.sub[sc][q][threadIdx.x];
        h[4 * q] = s.x; h[4 * q + 1] = s.y; h[4 * q + 2] = s.z; h[4 * q + 3] = s.w;
      }
#pragma unroll
      for (int i = 0; i < kSub; ++i) {
        const int t = a0 + i, ii = t - cb;
        const bool valid = t >= c0 && t < c1;
        const float dux = dl[i] * uu[i];
        const float* Bt = sm.B[ii];
        const bool head = sm.head[ii];
#pragma unroll
        for (int n = 0; n < N; ++n) {
          float ab_ = head ? 0.f : ex2(dl[i] * A2[n]);
          float hn = head ? dux * Bt[n] : fmaf(ab_, h[n], dux * Bt[n]);
          if (!valid) { ab_ = 0.f; hn = h[n]; }
          ab[i][n] = ab_;
          hb[i][n] = hn;
          h[n] = hn;
        }
      }
      // reverse recurrence over the sub-chunk
      float duo[4], ddo[4];
#pragma unroll
      for (int i = kSub - 1; i >= 0; --i) {
        const int t = a0 + i, ii = t - cb;
        const bool valid = t >= c0 && t < c1;  // CTA-uniform
        float4* rrow = &sm.red[wid][i * kQ][lid];
        if (!valid) {
#pragma unroll
          for (int q = 0; q < kQ; ++q) rrow[q * 33] = make_float4(0.f, 0.f, 0.f, 0.f);
          duo[i] = 0.f;
          ddo[i] = 0.f;
          continue;
        }
        const float dyv = yy[i], ux = uu[i], delta = dl[i];
        const float dux = delta * ux;
        const bool head = sm.head[ii];
        const float* Bt = sm.B[ii];
        const float* Ct = sm.C[ii];
        float Ssum = 0.f, dq = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < N / 4; ++q4) {
          float vb[4], vc[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = 4 * q4 + j;
            g[n] = fmaf(Ct[n], dyv, g[n]);  // g holds abar_{t+1} g_{t+1}
            Ssum = fmaf(g[n], Bt[n], Ssum);
            const float hm = head ? 0.f : fmaf(-dux, Bt[n], hb[i][n]);  // abar_t h_{t-1}
            const float q = g[n] * hm;
            dA[n] = fmaf(delta, q, dA[n]);
            dq = fmaf(A2[n], q, dq);
            vb[j] = g[n] * dux;
            vc[j] = dyv * hb[i][n];
            g[n] = ab[i][n] * g[n];  // carry to t-1 (0 at heads)
          }
          rrow[q4 * 33] = make_float4(vb[0], vb[1], vb[2], vb[3]);
          rrow[(N / 4 + q4) * 33] = make_float4(vc[0], vc[1], vc[2], vc[3]);
        }
        duo[i] = fmaf(Dd, dyv, delta * Ssum);
        const float dd = fmaf(ux, Ssum, dq * kLn2);
        ddo[i] = dd * sg[i];
        dD = fmaf(dyv, ux, dD);
        ddtb += ddo[i];
      }
      if (active) {
        store4<T, kVec>(du_row, a0, c0, c1, duo);
        store4<T, kVec>(ddt_row, a0, c0, c1, ddo);
      }
      // warp transpose-reduce: lane j owns row j = (step i, quad q)
      __syncwarp();
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lid < SM::kRows) {
        const float4* row = sm.red[wid][lid];
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
          const float4 v = row[l];
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      sm.xw[xbuf][wid][lid] = acc;
      __syncthreads();
      // cross-warp sum; thread -> (step i, value v) ; 2N values per step
      for (int e = threadIdx.x; e < kSub * 2 * N; e += kScanThreads) {
        const int i = e / (2 * N), v = e % (2 * N);
        const int t = a0 + i;
        if (t >= c0 && t < c1) {
          const int row = i * kQ + v / 4, comp = v % 4;
          float s = 0.f;
#pragma unroll
          for (int w = 0; w < kScanWarps; ++w) {
            const float4 p = sm.xw[xbuf][w][row];
            s += comp == 0 ? p.x : comp == 1 ? p.y : comp == 2 ? p.z : p.w;
          }
          ws_bc_r[(int64_t)t * (2 * N) + v] = s;
        }
      }
      xbuf ^= 1;
      __syncwarp();
    }
  }
  if (active) {
#pragma unroll
    for (int n = 0; n < N; ++n) wsp[(int64_t)n * Dn + d] = dA[n];
    wsp[(int64_t)N * Dn + d] = dD;
    wsp[(int64_t)(N + 1) * Dn + d] = ddtb;
  }
}

// dB[r,n,t] = sum_blk ws_bc[blk,r,t,n]; dC with n + N.  Fixed summation order.
template <int N>
__global__ void __launch_bounds__(256)
scan_bwd_finalize_bc(const float* __restrict__ ws_bc, float* __restrict__ dB,
                     float* __restrict__ dC, int nblk, int R, int L) {
  constexpr int TT = 32;
  __shared__ float tile[2 * N][TT + 1];
  const int r = blockIdx.y, t0 = blockIdx.x * TT;
  for (int e = threadIdx.x; e < TT * 2 * N; e += blockDim.x) {
    const int tt = e / (2 * N), v = e % (2 * N), t = t0 + tt;
    float s = 0.f;
    if (t < L)
      for (int b = 0; b < nblk; ++b)
        s += ws_bc[(((int64_t)b * R + r) * L + t) * (2 * N) + v];
    tile[v][tt] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TT * 2 * N; e += blockDim.x) {
    const int v = e / TT, tt = e % TT, t = t0 + tt;
    if (t < L) {
      float* dst = v < N ? dB + ((int64_t)r * N + v) * L : dC + ((int64_t)r * N + (v - N)) * L;
      dst[t] = tile[v][tt];
    }
  }
}

// dA[d,n], dD[d], ddt_bias[d] = sum over (row, segment) partials.
template <int N>
__global__ void __launch_bounds__(256)
scan_bwd_finalize_param(const float* __restrict__ ws, float* __restrict__ dA,
                        float* __restrict__ dD, float* __restrict__ ddtb, int nrs, int Dn) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)(N + 2) * Dn) return;
  const int n = (int)(e / Dn), d = (int)(e % Dn);
  float s = 0.f;
  for (int i = 0; i < nrs; ++i) s += ws[((int64_t)i * (N + 2) + n) * Dn + d];
  if (n < N) dA[(int64_t)d * N + n] = s;
  else if (n == N) { if (dD) dD[d] = s; }
  else { if (ddtb) ddtb[d] = s; }
}

}  // namespace pm

// ===========================================================================
// host side
// ===========================================================================
namespace {

using namespace pm;

int n_chunks(int64_t L) { return (int)((L + kChunk - 1) / kChunk); }
int n_dblk(int64_t Dn) { return (int)((Dn + kScanThreads - 1) / kScanThreads); }

// Segments per row: enough CTAs for ~4 resident waves on 148 SMs, but keep
// nominal segments >= 256 steps (actual cuts snap to heads anyway).
int n_segments(int64_t R, int64_t Dn, int64_t L) {
  const int64_t ctas = R * n_dblk(Dn);
  const int64_t target = 4 * 148 * 2;
  int64_t s = (target + ctas - 1) / ctas;
  s = std::min<int64_t>(s, std::max<int64_t>(1, L / 256));
  s = std::max<int64_t>(s, 1);
  return (int)std::min<int64_t>(s, 64);
}

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

pm_status check_common(int64_t R, int64_t Dn, int64_t L, int32_t N, pm_dtype io) {
  if (R < 1 || Dn < 1 || L < 1) return PM_ERR_INVALID_ARG;
  if (io != PM_F32 && io != PM_BF16) return PM_ERR_DTYPE;
  if (N != 4 && N != 8 && N != 16) return PM_ERR_UNSUPPORTED;
  if (R * L >= (int64_t(1) << 31) || Dn >= (int64_t(1) << 31)) return PM_ERR_SHAPE;
  if (R > 65535) return PM_ERR_SHAPE;
  return PM_OK;
}

bool elem_aligned(const void* p, pm_dtype io) {
  const uintptr_t m = io == PM_F32 ? 3u : 1u;
  return p == nullptr || (reinterpret_cast<uintptr_t>(p) & m) == 0;
}

template <typename T, int N, bool kVec>
pm_status launch_fwd(const ScanFwdArgs& a, cudaStream_t s) {
  dim3 grid(n_dblk(a.Dn), a.R, a.nseg);
  scan_fwd_kernel<T, N, kVec><<<grid, kScanThreads, 0, s>>>(a);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, int N>
pm_status dispatch_fwd_vec(const ScanFwdArgs& a, bool vec, cudaStream_t s) {
  return vec ? launch_fwd<T, N, true>(a, s) : launch_fwd<T, N, false>(a, s);
}

template <typename T>
pm_status dispatch_fwd(const ScanFwdArgs& a, int N, bool vec, cudaStream_t s) {
  switch (N) {
    case 4: return dispatch_fwd_vec<T, 4>(a, vec, s);
    case 8: return dispatch_fwd_vec<T, 8>(a, vec, s);
    default: return dispatch_fwd_vec<T, 16>(a, vec, s);
  }
}

template <typename T, int N, bool kVec>
pm_status launch_bwd(const ScanBwdArgs& a, float* dA, float* dB, float* dC, float* dD,
                     float* ddtb, cudaStream_t s) {
  const size_t smem = sizeof(BwdSmem<N>);
  auto kern = scan_bwd_kernel<T, N, kVec>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return PM_ERR_CUDA;
  dim3 grid(n_dblk(a.Dn), a.R, a.nseg);
  kern<<<grid, kScanThreads, smem, s>>>(a);
  PM_LAUNCH_CHECK();
  dim3 g2((a.L + 31) / 32, a.R);
  scan_bwd_finalize_bc<N><<<g2, 256, 0, s>>>(a.ws_bc, dB, dC, n_dblk(a.Dn), a.R, a.L);
  PM_LAUNCH_CHECK();
  const int64_t np = (int64_t)(N + 2) * a.Dn;
  scan_bwd_finalize_param<N><<<(unsigned)((np + 255) / 256), 256, 0, s>>>(
      a.ws_param, dA, dD, ddtb, a.R * a.nseg, a.Dn);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, int N>
pm_status dispatch_bwd_vec(const ScanBwdArgs& a, bool vec, float* dA, float* dB, float* dC,
                           float* dD, float* ddtb, cudaStream_t s) {
  return vec ? launch_bwd<T, N, true>(a, dA, dB, dC, dD, ddtb, s)
             : launch_bwd<T, N, false>(a, dA, dB, dC, dD, ddtb, s);
}

template <typename T>
pm_status dispatch_bwd(const ScanBwdArgs& a, int N, bool vec, float* dA, float* dB, float* dC,
                       float* dD, float* ddtb, cudaStream_t s) {
  switch (N) {
    case 4: return dispatch_bwd_vec<T, 4>(a, vec, dA, dB, dC, dD, ddtb, s);
    case 8: return dispatch_bwd_vec<T, 8>(a, vec, dA, dB, dC, dD, ddtb, s);
    default: return dispatch_bwd_vec<T, 16>(a, vec, dA, dB, dC, dD, ddtb, s);
  }
}

size_t state_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return (size_t)R * n_chunks(L) * N * Dn * sizeof(float);
}

size_t bwd_ws_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N, bool recompute) {
  size_t bc = (size_t)n_dblk(Dn) * R * L * 2 * N * sizeof(float);
  size_t par = (size_t)R * n_segments(R, Dn, L) * (N + 2) * Dn * sizeof(float);
  size_t st = recompute ? state_bytes(R, Dn, L, N) : 0;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  return up(bc) + up(par) + up(st);
}

}  // namespace

extern "C" {

size_t pm_selective_scan_state_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  if (R < 1 || Dn < 1 || L < 1 || N < 1) return 0;
  return state_bytes(R, Dn, L, N);
}

size_t pm_selective_scan_bwd_workspace(int64_t R, int64_t Dn, int64_t L, int32_t N,
                                       int32_t recompute_states) {
  if (R < 1 || Dn < 1 || L < 1 || N < 1) return 0;
  return bwd_ws_bytes(R, Dn, L, N, recompute_states != 0);
}

pm_status pm_selective_scan_fwd(const void* u, const void* dt, const float* A, const void* B,
                                const void* C, const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos, void* y, float* states,
                                int64_t R, int64_t Dn, int64_t L, int32_t N, pm_dtype io,
                                pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!u || !dt || !A || !B || !C || !pos || (!y && !states)) return PM_ERR_INVALID_ARG;
  for (const void* p : {u, dt, B, C, (const void*)y})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)A, (const void*)Dskip, (const void*)dt_bias, (const void*)pos,
                        (const void*)states})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && aligned16(u) && aligned16(dt) && aligned16(B) &&
                   aligned16(C) && aligned16(y);
  ScanFwdArgs a{u, dt, A, B, C, Dskip, dt_bias, pos, y, states,
                (int)R, (int)Dn, (int)L, n_segments(R, Dn, L), n_chunks(L), dt_softplus ? 1 : 0};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return io == PM_F32 ? dispatch_fwd<float>(a, N, vec, s) : dispatch_fwd<__nv_bfloat16>(a, N, vec, s);
}

pm_status pm_selective_scan_bwd(const void* u, const void* dt, const float* A, const void* B,
                                const void* C, const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos, const float* states,
                                const void* dy, void* du, void* ddt, float* dA, float* dB,
                                float* dC, float* dD, float* ddt_bias, void* workspace,
                                size_t ws_bytes, int64_t R, int64_t Dn, int64_t L, int32_t N,
                                pm_dtype io, pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!u || !dt || !A || !B || !C || !pos || !dy || !du || !ddt || !dA || !dB || !dC)
    return PM_ERR_INVALID_ARG;
  const bool recompute = states == nullptr;
  if (!workspace || ws_bytes < bwd_ws_bytes(R, Dn, L, N, recompute)) return PM_ERR_WORKSPACE;
  if (!aligned16(workspace)) return PM_ERR_ALIGN;
  for (const void* p : {u, dt, B, C, dy, (const void*)du, (const void*)ddt})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)A, (const void*)Dskip, (const void*)dt_bias, (const void*)pos,
                        (const void*)states, (const void*)dA, (const void*)dB, (const void*)dC,
                        (const void*)dD, (const void*)ddt_bias})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && aligned16(u) && aligned16(dt) && aligned16(B) &&
                   aligned16(C) && aligned16(dy) && aligned16(du) && aligned16(ddt);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* w = static_cast<char*>(workspace);
  float* ws_bc = reinterpret_cast<float*>(w);
  w += up((size_t)n_dblk(Dn) * R * L * 2 * N * sizeof(float));
  float* ws_par = reinterpret_cast<float*>(w);
  w += up((size_t)R * n_segments(R, Dn, L) * (N + 2) * Dn * sizeof(float));
  const float* stp = states;
  if (recompute) {
    float* st_ws = reinterpret_cast<float*>(w);
    ScanFwdArgs fa{u, dt, A, B, C, Dskip, dt_bias, pos, nullptr, st_ws,
                   (int)R, (int)Dn, (int)L, n_segments(R, Dn, L), n_chunks(L), dt_softplus ? 1 : 0};
    pm_status fs = io == PM_F32 ? dispatch_fwd<float>(fa, N, vec, s)
                                : dispatch_fwd<__nv_bfloat16>(fa, N, vec, s);
    if (fs != PM_OK) return fs;
    stp = st_ws;
  }
  ScanBwdArgs a{u, dt, A, B, C, Dskip, dt_bias, pos, stp, dy, du, ddt, ws_bc, ws_par,
                (int)R, (int)Dn, (int)L, n_segments(R, Dn, L), n_chunks(L), dt_softplus ? 1 : 0};
  return io == PM_F32 ? dispatch_bwd<float>(a, N, vec, dA, dB, dC, dD, ddt_bias, s)
                      : dispatch_bwd<__nv_bfloat16>(a, N, vec, dA, dB, dC, dD, ddt_bias, s);
}

}  // extern "C"
