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
#include "common.cuh"

namespace pm {

constexpr int kConvThreads = 128;
constexpr int kConvCh = 16;  // channels per CTA (pos reuse)

template <int K>
struct Taps {
  // valid[i][o] for o in [1, K-1] (o = 0 is always valid)
};

// ---------------------------------------------------------------------------
// forward: thread = 8 time steps x kConvCh channels
// ---------------------------------------------------------------------------
template <typename T, int K, bool kVec>
__global__ void __launch_bounds__(kConvThreads)
conv_fwd_kernel(const T* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                const int32_t* __restrict__ pos, T* __restrict__ out, int Dn, int L, int silu) {
  constexpr int E = 8;
  const int r = blockIdx.z;
  const int lid = threadIdx.x & 31;
  const int t0 = (blockIdx.x * kConvThreads + threadIdx.x) * E;
  const bool live = t0 < L;
  const int32_t* pos_row = pos + (int64_t)r * L;

  // tap masks: ok[i][o] <=> o <= pos[t0+i] && t0+i-o >= 0
  bool ok[E][K];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int t = t0 + i;
    const int p = (t < L) ? __ldg(pos_row + t) : 0;
#pragma unroll
    for (int o = 0; o < K; ++o) ok[i][o] = (o <= p) && (t - o >= 0);
  }

  const int dbase = blockIdx.y * kConvCh;
  for (int c = 0; c < kConvCh; ++c) {
    const int d = dbase + c;
    if (d >= Dn) break;  // CTA-uniform
    const int64_t lane = ((int64_t)r * Dn + d) * L;
    float xv[E];
    load8<T, kVec>(x + lane, t0, L, xv);
    // halo x[t0-1 .. t0-(K-1)] from lane-1 (its last K-1 values)
    float halo[K > 1 ? K - 1 : 1];
#pragma unroll
    for (int o = 1; o < K; ++o) {
      float v = __shfl_up_sync(0xffffffffu, xv[E - o], 1);
      if (lid == 0) v = (t0 - o >= 0 && t0 - o < L) ? IO<T>::ld(x + lane + t0 - o) : 0.f;
      halo[o - 1] = v;
    }
    float wk[K];
#pragma unroll
    for (int j = 0; j < K; ++j) wk[j] = __ldg(w + (int64_t)d * K + j);
    const float b = bias ? __ldg(bias + d) : 0.f;
    float yv[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      float pre = b;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int o = K - 1 - j;
        const float xs = (i - o >= 0) ? xv[i - o] : halo[o - i - 1];
        if (ok[i][o]) pre = fmaf(wk[j], xs, pre);
      }
      yv[i] = silu ? pre * sigmoidf_fast(pre) : pre;
    }
    if (live) store8<T, kVec>(out + lane, t0, 0, L, yv);
  }
}

// ---------------------------------------------------------------------------
// backward: thread = 8 time steps x kConvCh channels
//   dpre[t] = dout[t] * silu'(pre[t]);
//   dx[s]   = sum_o [s+o < L && o <= pos[s+o]] w[K-1-o] dpre[s+o]
//   dw[j]  += dpre[t] x[t-o] (o = K-1-j, valid tap);  db += dpre[t]
// Per-warp partials of (dw, db) go to ws (R * nwb, Dn, K+1); a finalize
// kernel sums them in a fixed order.
// ---------------------------------------------------------------------------
template <typename T, int K, bool kVec>
__global__ void __launch_bounds__(kConvThreads)
conv_bwd_kernel(const T* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                const int32_t* __restrict__ pos, const T* __restrict__ dout, T* __restrict__ dx,
                float* __restrict__ ws, int Dn, int L, int silu, int nwb) {
  constexpr int E = 8;
  const int r = blockIdx.z;
  const int lid = threadIdx.x & 31;
  const int gw = (blockIdx.x * kConvThreads + threadIdx.x) >> 5;  // global warp-block in row
  const int t0 = (blockIdx.x * kConvThreads + threadIdx.x) * E;
  const bool live = t0 < L;
  const int32_t* pos_row = pos + (int64_t)r * L;

  // own pos and the right halo pos[t0+E .. t0+E+K-2]
  int p[E + K - 1];
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = (t0 + i < L) ? __ldg(pos_row + t0 + i) : 0;
#pragma unroll
  for (int o = 1; o < K; ++o) {
    int v = __shfl_down_sync(0xffffffffu, p[o - 1], 1);
    const int t = t0 + E + o - 1;
    if (lid == 31) v = (t < L) ? __ldg(pos_row + t) : 0;
    p[E + o - 1] = v;
  }

  const int dbase = blockIdx.y * kConvCh;
  for (int c = 0; c < kConvCh; ++c) {
    const int d = dbase + c;
    if (d >= Dn) break;  // CTA-uniform
    const int64_t lane = ((int64_t)r * Dn + d) * L;
    float wk[K];
#pragma unroll
    for (int j = 0; j < K; ++j) wk[j] = __ldg(w + (int64_t)d * K + j);
    const float b = bias ? __ldg(bias + d) : 0.f;

    float xv[E], gv[E];
    load8<T, kVec>(x + lane, t0, L, xv);
    load8<T, kVec>(dout + lane, t0, L, gv);
    float halo[K > 1 ? K - 1 : 1];  // x[t0-1 .. t0-(K-1)]
#pragma unroll
    for (int o = 1; o < K; ++o) {
      float v = __shfl_up_sync(0xffffffffu, xv[E - o], 1);
      if (lid == 0) v = (t0 - o >= 0 && t0 - o < L) ? IO<T>::ld(x + lane + t0 - o) : 0.f;
      halo[o - 1] = v;
    }
    // dpre for own steps
    float dp[E + K - 1];
    float acc_w[K], acc_b = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) acc_w[j] = 0.f;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int t = t0 + i;
      float pre = b;
      float xs_[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int o = K - 1 - j;
        xs_[j] = (i - o >= 0) ? xv[i - o] : halo[o - i - 1];
        const bool okt = (o <= p[i]) && (t - o >= 0);
        if (okt) pre = fmaf(wk[j], xs_[j], pre);
        else xs_[j] = 0.f;  // excluded tap contributes nothing to dw
      }
      float gd = 1.f;
      if (silu) {
        const float s = sigmoidf_fast(pre);
        gd = s * fmaf(pre, 1.f - s, 1.f);
      }
      const float dpv = (t < L) ? gv[i] * gd : 0.f;
      dp[i] = dpv;
      acc_b += dpv;
#pragma unroll
      for (int j = 0; j < K; ++j) acc_w[j] = fmaf(dpv, xs_[j], acc_w[j]);
    }
    // right halo of dpre from lane+1; lane 31 recomputes it
#pragma unroll
    for (int o = 1; o < K; ++o) {
      float v = __shfl_down_sync(0xffffffffu, dp[o - 1], 1);
      if (lid == 31) {
        const int t = t0 + E + o - 1;
        v = 0.f;
        if (t < L) {
          float pre = b;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int oo = K - 1 - j;
            if (oo <= p[E + o - 1] && t - oo >= 0) pre = fmaf(wk[j], IO<T>::ld(x + lane + t - oo), pre);
          }
          float gd = 1.f;
          if (silu) {
            const float s = sigmoidf_fast(pre);
            gd = s * fmaf(pre, 1.f - s, 1.f);
          }
          v = IO<T>::ld(dout + lane + t) * gd;
        }
      }
      dp[E + o - 1] = v;
    }
    float dxv[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      float acc = 0.f;
#pragma unroll
      for (int o = 0; o < K; ++o) {
        const int t = t0 + i + o;
        if (t < L && o <= p[i + o]) acc = fmaf(wk[K - 1 - o], dp[i + o], acc);
      }
      dxv[i] = acc;
    }
    if (live) store8<T, kVec>(dx + lane, t0, 0, L, dxv);
    // warp reduce (dw, db) and write the per-warp partial
#pragma unroll
    for (int j = 0; j <= K; ++j) {
      float v = j < K ? acc_w[j] : acc_b;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lid == 0 && gw < nwb) ws[(((int64_t)r * nwb + gw) * Dn + d) * (K + 1) + j] = v;
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

constexpr int kE = 8;

int n_tblk(int64_t L) { return (int)((L + kConvThreads * kE - 1) / (kConvThreads * kE)); }
int n_wblk(int64_t L) { return n_tblk(L) * (kConvThreads / 32); }

bool a16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

pm_status check_conv(int64_t R, int64_t Dn, int64_t L, int32_t K, pm_dtype io) {
  if (R < 1 || Dn < 1 || L < 1) return PM_ERR_INVALID_ARG;
  if (io != PM_F32 && io != PM_BF16) return PM_ERR_DTYPE;
  if (K < 1 || K > 4) return PM_ERR_UNSUPPORTED;
  if (R > 65535 || (Dn + kConvCh - 1) / kConvCh > 65535 || R * L >= (int64_t(1) << 31))
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
  dim3 grid(n_tblk(L), (unsigned)((Dn + kConvCh - 1) / kConvCh), (unsigned)R);
  conv_fwd_kernel<T, K, V><<<grid, kConvThreads, 0, s>>>(
      static_cast<const T*>(x), w, b, pos, static_cast<T*>(out), (int)Dn, (int)L, silu);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, int K, bool V>
pm_status bwd_launch(const void* x, const float* w, const float* b, const int32_t* pos,
                     const void* dout, void* dx, float* dw, float* db, float* ws, int64_t R,
                     int64_t Dn, int64_t L, int silu, cudaStream_t s) {
  dim3 grid(n_tblk(L), (unsigned)((Dn + kConvCh - 1) / kConvCh), (unsigned)R);
  const int nwb = n_wblk(L);
  conv_bwd_kernel<T, K, V><<<grid, kConvThreads, 0, s>>>(
      static_cast<const T*>(x), w, b, pos, static_cast<const T*>(dout), static_cast<T*>(dx), ws,
      (int)Dn, (int)L, silu, nwb);
  PM_LAUNCH_CHECK();
  const int64_t n = Dn * (K + 1);
  conv_bwd_finalize<K><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ws, dw, db, (int)(R * nwb), (int)Dn);
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
  const bool vec = (L * isz) % 16 == 0 && a16(x) && a16(out);
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
  return (size_t)R * n_wblk(L) * Dn * (K + 1) * sizeof(float);
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
  const bool vec = (L * isz) % 16 == 0 && a16(x) && a16(dout) && a16(dx);
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
