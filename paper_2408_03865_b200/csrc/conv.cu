// conv.cu -- conv1d_pack forward/backward for sm_100a (Alg 1 P:152-170,
// sec 3.3, sec 3.5 P:234-239 of arXiv 2408.03865).
//
// HBM-bound kernels.  A thread owns E consecutive time steps of one channel
// row (128-bit loads/stores along L, the contiguous dim), so a warp moves a
// contiguous 32*E-element stretch.  position_indices are read once per
// thread into registers ("continuous threads read the consecutive
// position_indices ... transferred to the corresponding thread's registers",
// P:237) and reused for CH channels.  The K-1 halo comes from the
// neighbouring lane through warp shuffles (the paper's SRAM "stagger" of
// reverse indices, becomes a register shuffle): conv fwd needs x from
// lane-1, conv bwd needs dpre and pos from lane+1.
// Boundary taps are SKIPPED by a predicate (o <= pos[t] && t-o >= 0), never
// multiplied by zero.
#include <algorithm>

#include "common.cuh"

namespace pm {

// One warp per channel row: a warp covers kSpan = 32 lanes x 8 steps of one
// channel per iteration (coalesced 128-bit loads/stores along L) and marches
// through its time range; the K-1 halo comes from the neighbouring lane by
// shuffle and is carried across iterations in registers (the paper's SRAM
// "stagger" of reverse indices, becomes a register shuffle).  A warp
// whose taps are all inside their sequences (every pos >= K-1: the common
// case) runs a branch-free path; otherwise each tap is selected by the
// predicate o <= pos[t] && t-o >= 0 (skipped, never multiplied by 0).
#ifndef PM_CONV_WARPS  // channels (warps) per conv fwd CTA
#define PM_CONV_WARPS 4
#endif
#ifndef PM_CONV_BWD_WARPS  // channels (warps) per conv bwd CTA
#define PM_CONV_BWD_WARPS 1
#endif
#ifndef PM_CONV_WANT  // target CTAs per SM when splitting rows in time
#define PM_CONV_WANT 2
#endif
constexpr int kConvWarps = PM_CONV_WARPS;      // channels per CTA
constexpr int kConvThreads = 32 * kConvWarps;
// the backward runs one warp per CTA: its 80-register warps then pack up to
// 25 per SM in any mix of rows (measured: 0.282 -> 0.251 ms at the 1.4B shape)
constexpr int kConvBwdWarps = PM_CONV_BWD_WARPS;
#ifndef PM_CONV_BWD_CH  // channels per conv bwd warp (they share pos, halo and the tap decision)
#define PM_CONV_BWD_CH 2
#endif
constexpr int kConvBwdCh = PM_CONV_BWD_CH;
// fp32 I/O keeps one channel per warp: its SiLU' is two MUFU ops per channel
// anyway (no packed form), and one channel measured faster at the 130m shape
// (0.065 vs 0.070 ms)
#ifndef PM_CONV_BWD_CH_F32
#define PM_CONV_BWD_CH_F32 1
#endif
template <typename T>
constexpr int conv_bwd_ch() { return sizeof(T) == 2 ? kConvBwdCh : PM_CONV_BWD_CH_F32; }
constexpr int kConvBwdThreads = 32 * kConvBwdWarps;
constexpr int kCE = 8;                         // steps per lane per iteration
constexpr int kSpan = 32 * kCE;                // steps per warp iteration

template <bool kVec>
PM_DEV void load_pos8(const int32_t* __restrict__ prow, int t0, int L, int (&p)[8]) {
  if (kVec && t0 + 8 <= L) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(prow + t0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(prow + t0 + 4));
    p[0] = a.x; p[1] = a.y; p[2] = a.z; p[3] = a.w;
    p[4] = b.x; p[5] = b.y; p[6] = b.z; p[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = (t0 + i < L) ? __ldg(prow + t0 + i) : 0;
  }
}

// 8 consecutive position indices held in registers (prefetch)
template <bool kVec>
struct Pos8 {
  int p[8];
  PM_DEV void load(const int32_t* __restrict__ prow, int t0, int L) { load_pos8<kVec>(prow, t0, L, p); }
};

PM_DEV float silu_grad(float pre) {  // d/dpre [pre * sigmoid(pre)] (fp32 path)
  const float s = sigmoidf_fast(pre);
  return s * fmaf(pre, 1.f - s, 1.f);
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
#ifndef PM_CONV_CH  // channels per warp in the forward (they share pos and the tap decision)
#define PM_CONV_CH 2
#endif
#ifndef PM_CONV_TANH  // SiLU (and its derivative) through one MUFU.TANH for bf16 I/O
#define PM_CONV_TANH 1
#endif
constexpr int kConvCh = PM_CONV_CH;

// x * sigmoid(x).  fp32 I/O: ex2 + rcp (max error a few ulp, the fp32
// tolerance is 1e-4).  bf16 I/O: 0.5 x (1 + tanh(x / 2)) with tanh.approx
// (one MUFU op; relative error ~5e-4, below half a bf16 ulp of the output).
template <typename T>
PM_DEV float silu_io(float v) {
  if constexpr (sizeof(T) == 2 && PM_CONV_TANH) {
    float t;
    const float hv = 0.5f * v;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(hv));
    return fmaf(hv, t, hv);
  } else {
    return v * sigmoidf_fast(v);
  }
}

// silu for a channel pair (packed; bf16 I/O: the same arithmetic as silu_io)
template <typename T>
PM_DEV float2 silu2_io(float2 v) {
  if constexpr (sizeof(T) == 2 && PM_CONV_TANH) {
    const float2 hv = fmul2(f2(0.5f), v);
    float2 t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(hv.x));
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(hv.y));
    return ffma2(hv, t, hv);
  } else {
    return make_float2(silu_io<T>(v.x), silu_io<T>(v.y));
  }
}
#ifndef PM_CONV_FWD_PACK  // full-window path of the forward as packed channel pairs
#define PM_CONV_FWD_PACK 1
#endif

// A warp serves kConvCh consecutive channels of one row over the same time
// range: per 256-step iteration the position indices are loaded and the tap
// decision taken once for all of them.
template <typename T, int K, bool kVec, bool kSilu>
__global__ void __launch_bounds__(kConvThreads)
conv_fwd_kernel(const T* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                const int32_t* __restrict__ pos, T* __restrict__ out, int Dn, int L, int tspan) {
  constexpr int CH = kConvCh;
  const int lid = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int d0 = (blockIdx.x * kConvWarps + wid) * CH;
  if (d0 >= Dn) return;  // warp-uniform
  const int r = blockIdx.y;
  const int tb = blockIdx.z * tspan, te = min(L, tb + tspan);
  const int32_t* prow = pos + (int64_t)r * L;
  // channel c of the warp: d0 + c (clamped; a missing channel computes the
  // last one again and does not store)
  const T* xr[CH];
  T* orow[CH];
  bool own[CH];
  float wk[CH][K], b[CH];
  float carry[CH][K > 1 ? K - 1 : 1];  // x[t-o] for the first step of the next iteration (lane 0)
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    own[c] = d0 + c < Dn;
    const int d = own[c] ? d0 + c : Dn - 1;
    const int64_t lane = ((int64_t)r * Dn + d) * L;
    xr[c] = x + lane;
    orow[c] = out + lane;
#pragma unroll
    for (int j = 0; j < K; ++j) wk[c][j] = __ldg(w + (int64_t)d * K + j);
    b[c] = bias ? __ldg(bias + d) : 0.f;
#pragma unroll
    for (int o = 1; o < K; ++o) carry[c][o - 1] = (tb - o >= 0) ? IO<T>::ld(xr[c] + tb - o) : 0.f;
  }

  // software pipeline: the next iteration's x/pos are in flight while this
  // one computes
  Raw8<T, kVec> nx[CH];
  Pos8<kVec> np;
#pragma unroll
  for (int c = 0; c < CH; ++c) nx[c].load(xr[c], tb + lid * kCE, te);
  np.load(prow, tb + lid * kCE, te);
  for (int t0b = tb; t0b < te; t0b += kSpan) {
    const int t0 = t0b + lid * kCE;
    float xv[CH][8];
    int p[8];
#pragma unroll
    for (int c = 0; c < CH; ++c) nx[c].unpack(xv[c]);
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = np.p[i];
    if (t0b + kSpan < te) {
#pragma unroll
      for (int c = 0; c < CH; ++c) nx[c].load(xr[c], t0 + kSpan, te);
      np.load(prow, t0 + kSpan, te);
    }
    float X[CH][K - 1 + 8];  // X[c][k] = x[t0 - (K-1) + k]
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#pragma unroll
      for (int o = 1; o < K; ++o) {
        const float v = __shfl_up_sync(0xffffffffu, xv[c][8 - o], 1);
        X[c][K - 1 - o] = lid == 0 ? carry[c][o - 1] : v;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) X[c][K - 1 + i] = xv[c][i];
#pragma unroll
      for (int o = 1; o < K; ++o) carry[c][o - 1] = __shfl_sync(0xffffffffu, xv[c][8 - o], 31);
    }
    // one decision per iteration for the warp's CH channels: all 8 steps
    // inside [tb, te) with every tap in range (the common case), all 8 steps
    // sequence heads (e.g. padding), else per-step tap masks
    int pmin = p[0], pmax = p[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      pmin = min(pmin, p[i]);
      pmax = max(pmax, p[i]);
    }
    const bool inr = t0 + 8 <= te;
    const bool full = inr && t0 >= K - 1 && pmin >= K - 1;
    const bool heads = inr && pmax == 0 && pmin == 0;
    float yv[CH][8];
    if (__all_sync(0xffffffffu, full)) {
      if constexpr (CH == 2 && PM_CONV_FWD_PACK) {  // the two channels as packed fp32x2 pairs
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float2 pre = make_float2(b[0], b[1]);
#pragma unroll
          for (int j = 0; j < K; ++j)
            pre = ffma2(make_float2(wk[0][j], wk[1][j]), make_float2(X[0][i + j], X[1][i + j]), pre);
          const float2 y2 = kSilu ? silu2_io<T>(pre) : pre;
          yv[0][i] = y2.x;
          yv[1][i] = y2.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float pre = b[c];
#pragma unroll
            for (int j = 0; j < K; ++j) pre = fmaf(wk[c][j], X[c][i + j], pre);
            yv[c][i] = kSilu ? silu_io<T>(pre) : pre;
          }
        }
      }
    } else if (__all_sync(0xffffffffu, heads)) {  // only the o = 0 tap survives
#pragma unroll
      for (int c = 0; c < CH; ++c) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float pre = fmaf(wk[c][K - 1], xv[c][i], b[c]);
          yv[c][i] = kSilu ? silu_io<T>(pre) : pre;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ci = min(p[i], t0 + i);  // tap o kept iff o <= pos[t] and t - o >= 0
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          float pre = b[c];
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (K - 1 - j <= ci) pre = fmaf(wk[c][j], X[c][i + j], pre);
          yv[c][i] = kSilu ? silu_io<T>(pre) : pre;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (own[c]) store8<T, kVec>(orow[c], t0, tb, te, yv[c]);
  }
}

// d/dpre [pre * sigmoid(pre)] = s (1 + pre (1 - s)); bf16 I/O through one
// MUFU.TANH: s = (1 + t) / 2, s (1 - s) = (1 - t^2) / 4, t = tanh(pre / 2)
template <typename T>
PM_DEV float silu_grad_io(float pre) {
  if constexpr (sizeof(T) == 2 && PM_CONV_TANH) {
    float t;
    const float h = 0.5f * pre;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    const float sg = fmaf(0.5f, t, 0.5f);
    return fmaf(0.5f * h, fmaf(-t, t, 1.f), sg);
  } else {
    return silu_grad(pre);
  }
}

// ---------------------------------------------------------------------------
// backward: march through the time range in REVERSE so the right halo (dpre
// and pos of the next K-1 steps -- the "reverse indices") is always carried
// from the previous iteration; dw/db accumulate in registers and are reduced
// once per warp into per-(row, time-range) partials (fixed-order finalize).
// ---------------------------------------------------------------------------
template <typename T, int K>
PM_DEV float dpre_at(const T* xr, const T* gr, const int32_t* prow, const float (&wk)[K], float b,
                     int t, int L, int silu) {
  if (t >= L) return 0.f;
  const int pt = __ldg(prow + t);
  float pre = b;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int o = K - 1 - j;
    if (o <= pt && t - o >= 0) pre = fmaf(wk[j], IO<T>::ld(xr + t - o), pre);
  }
  return IO<T>::ld(gr + t) * (silu ? silu_grad_io<T>(pre) : 1.f);
}

// silu'(pre) for a channel pair (packed fp32x2; bf16 I/O: one MUFU.TANH per
// channel, the same arithmetic as silu_grad_io)
template <typename T>
PM_DEV float2 silu_grad2_io(float2 pre) {
  if constexpr (sizeof(T) == 2 && PM_CONV_TANH) {
    const float2 h = fmul2(f2(0.5f), pre);
    float2 t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(h.x));
    asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(h.y));
    const float2 sg = ffma2(f2(0.5f), t, f2(0.5f));
    return ffma2(fmul2(f2(0.5f), h), ffma2(make_float2(-t.x, -t.y), t, f2(1.f)), sg);
  } else {
    return make_float2(silu_grad(pre.x), silu_grad(pre.y));
  }
}

// (an explicit register target, PM_CONV_BWD_MINB=n: 20/24 warps per SM spill
// and measured slower; n = 1 lets the allocator take 168 registers)
#ifdef PM_CONV_BWD_MINB
#define PM_CONV_BWD_BOUNDS __launch_bounds__(kConvBwdThreads, PM_CONV_BWD_MINB)
#else
#define PM_CONV_BWD_BOUNDS __launch_bounds__(kConvBwdThreads)
#endif
template <typename T, int K, bool kVec, bool kSilu, int CH>
__global__ void PM_CONV_BWD_BOUNDS
conv_bwd_kernel(const T* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                const int32_t* __restrict__ pos, const T* __restrict__ dout, T* __restrict__ dx,
                float* __restrict__ ws, int Dn, int L, int tspan, int ntc) {
  // one warp = CH consecutive channel rows of one row x (32 lanes x 8 steps)
  // per iteration, walked in reverse; the channels share the position
  // indices, their halo and the tap decision, and the full-window path runs
  // the two channels as packed fp32x2 pairs (FFMA2: half the instructions,
  // no shifted operands to build)
  constexpr int G = 32;
  const int g = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int d0 = (blockIdx.x * kConvBwdWarps + wid) * CH;
  if (d0 >= Dn) return;  // warp-uniform
  const int r = blockIdx.y, tc = blockIdx.z;
  const int tb = tc * tspan, te = min(L, tb + tspan);
  const int32_t* prow = pos + (int64_t)r * L;
  const T* xr[CH];
  const T* gr[CH];
  T* dxr[CH];
  bool own[CH];
  int dd[CH];
  float wk[CH][K], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    own[c] = d0 + c < Dn;
    dd[c] = own[c] ? d0 + c : Dn - 1;
    const int64_t lane = ((int64_t)r * Dn + dd[c]) * L;
    xr[c] = x + lane;
    gr[c] = dout + lane;
    dxr[c] = dx + lane;
#pragma unroll
    for (int j = 0; j < K; ++j) wk[c][j] = __ldg(w + (int64_t)dd[c] * K + j);
    b[c] = bias ? __ldg(bias + dd[c]) : 0.f;
  }
  constexpr int H = K > 1 ? K - 1 : 1;

  // right-halo carry: dpre (per channel) and pos of steps te .. te+K-2
  // (lane g = o-1 computes step te+o-1)
  float cdp[CH][H];
  int cp[H];
  {
    float myd[CH];
    int myp = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) myd[c] = 0.f;
    if (g < K - 1 && te + g < L) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        myd[c] = dpre_at<T, K>(xr[c], gr[c], prow, wk[c], b[c], te + g, L, kSilu ? 1 : 0);
      myp = __ldg(prow + te + g);
    }
#pragma unroll
    for (int o = 1; o < K; ++o) {
#pragma unroll
      for (int c = 0; c < CH; ++c) cdp[c][o - 1] = __shfl_sync(0xffffffffu, myd[c], o - 1, G);
      cp[o - 1] = __shfl_sync(0xffffffffu, myp, o - 1, G);
    }
  }
  float acc_w[CH][K], acc_b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    acc_b[c] = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) acc_w[c][j] = 0.f;
  }

  const int nblk = (te - tb + kSpan - 1) / kSpan;
  Raw8<T, kVec> nx[CH], ng[CH];
  Pos8<kVec> np;
  // left halo of x for lane g = 0 (x[t0-K+1 .. t0-1]), loaded one iteration
  // ahead so no dependent global load sits in the loop body
  float hx[CH][H];
  auto load_halo = [&](int t0l) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int o = 1; o < K; ++o)
        hx[c][o - 1] = (g == 0 && t0l - o >= 0) ? IO<T>::ld(xr[c] + t0l - o) : 0.f;
  };
  {
    const int t0 = tb + (nblk - 1) * kSpan + g * kCE;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      nx[c].load(xr[c], t0, te);
      ng[c].load(gr[c], t0, te);
    }
    np.load(prow, t0, te);
    load_halo(tb + (nblk - 1) * kSpan);
  }
  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int t0 = tb + blk * kSpan + g * kCE;
    float xv[CH][8], gv[CH][8];
    int p[8];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      nx[c].unpack(xv[c]);
      ng[c].unpack(gv[c]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = np.p[i];
    // left halo of x: lane g-1 (g = 0: the value prefetched last iteration)
    float X[CH][K - 1 + 8];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#pragma unroll
      for (int o = 1; o < K; ++o) {
        const float v = __shfl_up_sync(0xffffffffu, xv[c][8 - o], 1, G);
        X[c][K - 1 - o] = g == 0 ? hx[c][o - 1] : v;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) X[c][K - 1 + i] = xv[c][i];
    }
    if (blk > 0) {  // prefetch the earlier block and its halo
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        nx[c].load(xr[c], t0 - kSpan, te);
        ng[c].load(gr[c], t0 - kSpan, te);
      }
      np.load(prow, t0 - kSpan, te);
      load_halo(tb + (blk - 1) * kSpan);
    }
    // right halo of pos from lane g+1 (g = G-1: carry)
    int ph[H];
#pragma unroll
    for (int o = 1; o < K; ++o) {
      const int vp = __shfl_down_sync(0xffffffffu, p[o - 1], 1, G);
      ph[o - 1] = g == G - 1 ? cp[o - 1] : vp;
    }
    // one decision per warp iteration for all CH channels: every forward tap
    // and every dx tap valid, all 8 steps inside the range (the common
    // case), else per-tap predicates
    int pmin = p[0], pmax = p[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      pmin = min(pmin, p[i]);
      pmax = max(pmax, p[i]);
    }
#pragma unroll
    for (int o = 1; o < K; ++o) {
      pmin = min(pmin, ph[o - 1]);
      pmax = max(pmax, ph[o - 1]);
    }
    const bool inr = t0 + 8 <= te;
    const bool full = inr && t0 >= K - 1 && t0 + 8 + K - 2 < L && pmin >= K - 1;
    const bool wfull = __all_sync(0xffffffffu, full);
    // every slot of the window (and of its right halo) a head -- e.g. the
    // padding run at the end of a row: only the o = 0 tap survives
    const bool heads = inr && pmax == 0 && pmin == 0;
    const bool wheads = K > 1 && !wfull && __all_sync(0xffffffffu, heads);
    float dp[CH][8 + H];
    float dxv[CH][8];
    if (wfull && CH == 2) {
      // packed: lane .x = channel d0, .y = channel d0 + 1
      float2 X2[K - 1 + 8], w2[K], dp2[8 + H];
#pragma unroll
      for (int k = 0; k < K - 1 + 8; ++k) X2[k] = make_float2(X[0][k], X[CH - 1][k]);
#pragma unroll
      for (int j = 0; j < K; ++j) w2[j] = make_float2(wk[0][j], wk[CH - 1][j]);
      float2 ab2 = make_float2(acc_b[0], acc_b[CH - 1]);
      float2 aw2[K];
#pragma unroll
      for (int j = 0; j < K; ++j) aw2[j] = make_float2(acc_w[0][j], acc_w[CH - 1][j]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 pre = make_float2(b[0], b[CH - 1]);
#pragma unroll
        for (int j = 0; j < K; ++j) pre = ffma2(w2[j], X2[i + j], pre);
        const float2 g2 = make_float2(gv[0][i], gv[CH - 1][i]);
        const float2 dpv = kSilu ? fmul2(g2, silu_grad2_io<T>(pre)) : g2;
        dp2[i] = dpv;
        ab2 = fadd2(ab2, dpv);
#pragma unroll
        for (int j = 0; j < K; ++j) aw2[j] = ffma2(dpv, X2[i + j], aw2[j]);
      }
#pragma unroll
      for (int o = 1; o < K; ++o) {
        const float vx = __shfl_down_sync(0xffffffffu, dp2[o - 1].x, 1, G);
        const float vy = __shfl_down_sync(0xffffffffu, dp2[o - 1].y, 1, G);
        dp2[8 + o - 1] = g == G - 1 ? make_float2(cdp[0][o - 1], cdp[CH - 1][o - 1]) : make_float2(vx, vy);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int o = 0; o < K; ++o) a2 = ffma2(w2[K - 1 - o], dp2[i + o], a2);
        dxv[0][i] = a2.x;
        dxv[CH - 1][i] = a2.y;
      }
#pragma unroll
      for (int k = 0; k < 8 + H; ++k) {
        dp[0][k] = dp2[k].x;
        dp[CH - 1][k] = dp2[k].y;
      }
      acc_b[0] = ab2.x;
      acc_b[CH - 1] = ab2.y;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        acc_w[0][j] = aw2[j].x;
        acc_w[CH - 1][j] = aw2[j].y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (wheads) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float pre = fmaf(wk[c][K - 1], xv[c][i], b[c]);
            const float dpv = gv[c][i] * (kSilu ? silu_grad_io<T>(pre) : 1.f);
            dp[c][i] = dpv;
            acc_b[c] += dpv;
            acc_w[c][K - 1] = fmaf(dpv, xv[c][i], acc_w[c][K - 1]);
            dxv[c][i] = wk[c][K - 1] * dpv;
          }
        } else if (wfull) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float pre = b[c];
#pragma unroll
            for (int j = 0; j < K; ++j) pre = fmaf(wk[c][j], X[c][i + j], pre);
            const float dpv = gv[c][i] * (kSilu ? silu_grad_io<T>(pre) : 1.f);
            dp[c][i] = dpv;
            acc_b[c] += dpv;
#pragma unroll
            for (int j = 0; j < K; ++j) acc_w[c][j] = fmaf(dpv, X[c][i + j], acc_w[c][j]);
          }
#pragma unroll
          for (int o = 1; o < K; ++o) {
            const float vd = __shfl_down_sync(0xffffffffu, dp[c][o - 1], 1, G);
            dp[c][8 + o - 1] = g == G - 1 ? cdp[c][o - 1] : vd;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float a = 0.f;
#pragma unroll
            for (int o = 0; o < K; ++o) a = fmaf(wk[c][K - 1 - o], dp[c][i + o], a);
            dxv[c][i] = a;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int t = t0 + i;
            const int ci = min(p[i], t);  // tap o is kept iff o <= pos[t] and t - o >= 0
            float pre = b[c];
#pragma unroll
            for (int j = 0; j < K; ++j)
              if (K - 1 - j <= ci) pre = fmaf(wk[c][j], X[c][i + j], pre);
            const float dpv = (t < te) ? gv[c][i] * (kSilu ? silu_grad_io<T>(pre) : 1.f) : 0.f;
            dp[c][i] = dpv;
            acc_b[c] += dpv;
#pragma unroll
            for (int j = 0; j < K; ++j)
              if (K - 1 - j <= ci) acc_w[c][j] = fmaf(dpv, X[c][i + j], acc_w[c][j]);
          }
#pragma unroll
          for (int o = 1; o < K; ++o) {
            const float vd = __shfl_down_sync(0xffffffffu, dp[c][o - 1], 1, G);
            dp[c][8 + o - 1] = g == G - 1 ? cdp[c][o - 1] : vd;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float a = 0.f;
#pragma unroll
            for (int o = 0; o < K; ++o) {
              // dp is 0 at and beyond L (own block: t >= te; carry: 0 past L)
              const int pt = (i + o < 8) ? p[i + o] : ph[i + o - 8];
              if (o <= pt) a = fmaf(wk[c][K - 1 - o], dp[c][i + o], a);
            }
            dxv[c][i] = a;
          }
        }
      }
    }
    // next (earlier) iteration's carry = this block's first K-1 steps (lane g = 0)
#pragma unroll
    for (int o = 1; o < K; ++o) {
#pragma unroll
      for (int c = 0; c < CH; ++c) cdp[c][o - 1] = __shfl_sync(0xffffffffu, dp[c][o - 1], 0, G);
      cp[o - 1] = __shfl_sync(0xffffffffu, p[o - 1], 0, G);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (own[c]) store8<T, kVec>(dxr[c], t0, tb, te, dxv[c]);
  }
  // one warp reduction of (dw, db) per channel for this (row, time range)
#pragma unroll
  for (int c = 0; c < CH; ++c) {
#pragma unroll
    for (int j = 0; j <= K; ++j) {
      float v = j < K ? acc_w[c][j] : acc_b[c];
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
      if (g == 0 && own[c]) ws[(((int64_t)r * ntc + tc) * Dn + dd[c]) * (K + 1) + j] = v;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(256)
conv_bwd_finalize(const float* __restrict__ ws, float* __restrict__ dw, float* __restrict__ db,
                  int nparts, int Dn) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)Dn * (K + 1)) return;
  const int d = (int)(e / (K + 1)), j = (int)(e % (K + 1));
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += ws[((int64_t)i * Dn + d) * (K + 1) + j];
  if (j < K) dw[(int64_t)d * K + j] = s;
  else if (db) db[d] = s;
}

}  // namespace pm

// ===========================================================================
// host side
// ===========================================================================
namespace {
using namespace pm;

// time range per CTA: whole rows when R x Dn gives enough CTAs, else split
// (multiples of kSpan) so that ~8 waves of CTAs exist.
// (chans = channels per CTA, span = steps per warp iteration)
int conv_tspan(int64_t R, int64_t Dn, int64_t L, int chans, int span) {
  const int64_t ctas = R * ((Dn + chans - 1) / chans);
  const int64_t want = (int64_t)PM_CONV_WANT * sm_count() * 8;
  int64_t nt = (want + ctas - 1) / ctas;
  const int64_t nblk = (L + span - 1) / span;
  nt = std::max<int64_t>(1, std::min<int64_t>(nt, nblk));
  const int64_t blk_per = (nblk + nt - 1) / nt;
  return (int)(blk_per * span);
}
int conv_ntc(int64_t L, int tspan) { return (int)((L + tspan - 1) / tspan); }
int bwd_tspan(int64_t R, int64_t Dn, int64_t L, int ch) {
  return conv_tspan(R, Dn, L, kConvBwdWarps * ch, kSpan);
}

bool a16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

pm_status check_conv(int64_t R, int64_t Dn, int64_t L, int32_t K, pm_dtype io) {
  if (R < 1 || Dn < 1 || L < 1) return PM_ERR_INVALID_ARG;
  if (io != PM_F32 && io != PM_BF16) return PM_ERR_DTYPE;
  if (K < 1 || K > 4) return PM_ERR_UNSUPPORTED;
  if (R > 65535 || R * L >= (int64_t(1) << 31) || (Dn + kConvBwdWarps - 1) / kConvBwdWarps >= (1 << 30))
    return PM_ERR_SHAPE;
  return PM_OK;
}

bool ealigned(const void* p, pm_dtype io) {
  const uintptr_t m = io == PM_F32 ? 3u : 1u;
  return p == nullptr || (reinterpret_cast<uintptr_t>(p) & m) == 0;
}

template <typename T, int K, bool V>
pm_status fwd_launch(const void* x, const float* w, const float* b, const int32_t* pos, void* out,
                     int64_t R, int64_t Dn, int64_t L, int silu, cudaStream_t s) {
  const int tspan = conv_tspan(R, Dn, L, kConvWarps * kConvCh, kSpan);
  const int64_t per_cta = (int64_t)kConvWarps * kConvCh;
  dim3 grid((unsigned)((Dn + per_cta - 1) / per_cta), (unsigned)R, (unsigned)conv_ntc(L, tspan));
  if (silu)
    conv_fwd_kernel<T, K, V, true><<<grid, kConvThreads, 0, s>>>(
        static_cast<const T*>(x), w, b, pos, static_cast<T*>(out), (int)Dn, (int)L, tspan);
  else
    conv_fwd_kernel<T, K, V, false><<<grid, kConvThreads, 0, s>>>(
        static_cast<const T*>(x), w, b, pos, static_cast<T*>(out), (int)Dn, (int)L, tspan);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, int K, bool V>
pm_status bwd_launch(const void* x, const float* w, const float* b, const int32_t* pos,
                     const void* dout, void* dx, float* dw, float* db, float* ws, int64_t R,
                     int64_t Dn, int64_t L, int silu, cudaStream_t s) {
  constexpr int CH = conv_bwd_ch<T>();
  const int tspan = bwd_tspan(R, Dn, L, CH), ntc = conv_ntc(L, tspan);
  const int64_t per_cta = (int64_t)kConvBwdWarps * CH;
  dim3 grid((unsigned)((Dn + per_cta - 1) / per_cta), (unsigned)R, (unsigned)ntc);
  if (silu)
    conv_bwd_kernel<T, K, V, true, CH><<<grid, kConvBwdThreads, 0, s>>>(
        static_cast<const T*>(x), w, b, pos, static_cast<const T*>(dout), static_cast<T*>(dx), ws,
        (int)Dn, (int)L, tspan, ntc);
  else
    conv_bwd_kernel<T, K, V, false, CH><<<grid, kConvBwdThreads, 0, s>>>(
        static_cast<const T*>(x), w, b, pos, static_cast<const T*>(dout), static_cast<T*>(dx), ws,
        (int)Dn, (int)L, tspan, ntc);
  PM_LAUNCH_CHECK();
  const int64_t n = Dn * (K + 1);
  conv_bwd_finalize<K><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ws, dw, db, (int)(R * ntc), (int)Dn);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, bool V>
pm_status fwd_k(int K, const void* x, const float* w, const float* b, const int32_t* pos, void* out,
                int64_t R, int64_t Dn, int64_t L, int silu, cudaStream_t s) {
  switch (K) {
    case 1: return fwd_launch<T, 1, V>(x, w, b, pos, out, R, Dn, L, silu, s);
    case 2: return fwd_launch<T, 2, V>(x, w, b, pos, out, R, Dn, L, silu, s);
    case 3: return fwd_launch<T, 3, V>(x, w, b, pos, out, R, Dn, L, silu, s);
    default: return fwd_launch<T, 4, V>(x, w, b, pos, out, R, Dn, L, silu, s);
  }
}

template <typename T, bool V>
pm_status bwd_k(int K, const void* x, const float* w, const float* b, const int32_t* pos,
                const void* dout, void* dx, float* dw, float* db, float* ws, int64_t R, int64_t Dn,
                int64_t L, int silu, cudaStream_t s) {
  switch (K) {
    case 1: return bwd_launch<T, 1, V>(x, w, b, pos, dout, dx, dw, db, ws, R, Dn, L, silu, s);
    case 2: return bwd_launch<T, 2, V>(x, w, b, pos, dout, dx, dw, db, ws, R, Dn, L, silu, s);
    case 3: return bwd_launch<T, 3, V>(x, w, b, pos, dout, dx, dw, db, ws, R, Dn, L, silu, s);
    default: return bwd_launch<T, 4, V>(x, w, b, pos, dout, dx, dw, db, ws, R, Dn, L, silu, s);
  }
}

}  // namespace

extern "C" {

pm_status pm_causal_conv1d_fwd(const void* x, const float* w, const float* bias, const int32_t* pos,
                               void* out, int64_t R, int64_t Dn, int64_t L, int32_t K, pm_dtype io,
                               int32_t silu, pm_stream_t stream) {
  pm_status st = check_conv(R, Dn, L, K, io);
  if (st != PM_OK) return st;
  if (!x || !w || !pos || !out) return PM_ERR_INVALID_ARG;
  if (!ealigned(x, io) || !ealigned(out, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)w, (const void*)bias, (const void*)pos})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && L % 4 == 0 && a16(x) && a16(out) && a16(pos);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int sl = silu ? 1 : 0;
  if (io == PM_F32)
    return vec ? fwd_k<float, true>(K, x, w, bias, pos, out, R, Dn, L, sl, s)
               : fwd_k<float, false>(K, x, w, bias, pos, out, R, Dn, L, sl, s);
  return vec ? fwd_k<__nv_bfloat16, true>(K, x, w, bias, pos, out, R, Dn, L, sl, s)
             : fwd_k<__nv_bfloat16, false>(K, x, w, bias, pos, out, R, Dn, L, sl, s);
}

size_t pm_causal_conv1d_bwd_workspace(int64_t R, int64_t Dn, int64_t L, int32_t K) {
  if (R < 1 || Dn < 1 || L < 1 || K < 1 || K > 4) return 0;
  // (the larger of the two launch shapes: fp32 and bf16 I/O may use
  // different channels per warp, hence different time splits)
  const int ntc = std::max(conv_ntc(L, bwd_tspan(R, Dn, L, conv_bwd_ch<float>())),
                           conv_ntc(L, bwd_tspan(R, Dn, L, conv_bwd_ch<__nv_bfloat16>())));
  return (size_t)R * ntc * Dn * (K + 1) * sizeof(float);
}

pm_status pm_causal_conv1d_bwd(const void* x, const float* w, const float* bias, const int32_t* pos,
                               const void* dout, void* dx, float* dw, float* dbias, int64_t R,
                               int64_t Dn, int64_t L, int32_t K, pm_dtype io, int32_t silu,
                               void* workspace, size_t ws_bytes, pm_stream_t stream) {
  pm_status st = check_conv(R, Dn, L, K, io);
  if (st != PM_OK) return st;
  if (!x || !w || !pos || !dout || !dx || !dw) return PM_ERR_INVALID_ARG;
  if (!workspace || ws_bytes < pm_causal_conv1d_bwd_workspace(R, Dn, L, K)) return PM_ERR_WORKSPACE;
  if (!ealigned(x, io) || !ealigned(dout, io) || !ealigned(dx, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)w, (const void*)bias, (const void*)pos, (const void*)dw,
                        (const void*)dbias, (const void*)workspace})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && L % 4 == 0 && a16(x) && a16(dout) && a16(dx) && a16(pos);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* ws = static_cast<float*>(workspace);
  const int sl = silu ? 1 : 0;
  if (io == PM_F32)
    return vec ? bwd_k<float, true>(K, x, w, bias, pos, dout, dx, dw, dbias, ws, R, Dn, L, sl, s)
               : bwd_k<float, false>(K, x, w, bias, pos, dout, dx, dw, dbias, ws, R, Dn, L, sl, s);
  return vec ? bwd_k<__nv_bfloat16, true>(K, x, w, bias, pos, dout, dx, dw, dbias, ws, R, Dn, L, sl, s)
             : bwd_k<__nv_bfloat16, false>(K, x, w, bias, pos, dout, dx, dw, dbias, ws, R, Dn, L, sl, s);
}

}  // extern "C"
