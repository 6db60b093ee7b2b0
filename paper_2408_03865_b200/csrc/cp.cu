// cp.cu -- context-parallel scan over cut sequences (the
// paper's future work: "cut long sequences into multiple parts and pass the
// hidden state between these parts").
//
// A sequence longer than a pack continues from row r-1 into row r when
// pos[r, 0] != 0 (its position indices keep counting; reading Q9 with h0).
// The recurrence is linear in the state entering a row, so a row's true
// results are its local results (state entering = 0) plus a correction that
// only touches the row's continuing PREFIX (the slots before its first head):
//   h_t = h_t^local + P_t h_in,   P_t = prod_{i<=t} abar_i,   t < first head
// (after a head the reset removes every trace of h_in).  The pieces:
//   chain_fwd : h_in[r] = decay[r-1] h_in[r-1] + h_last_local[r-1] along the
//               chain (decay = d h_last / d h0, the row summary the forward
//               writes), h_last[r] = decay[r] h_in[r] + h_last_local[r];
//   fwd_fixup : out_t += C_t . (P_t h_in) (x silu(z_t) with the gate) for the
//               prefix slots, and the prefix's chunk checkpoints += P h_in,
//               so the backward recomputes the true states;
//   dh0       : the gradient of a row's own outputs w.r.t. its h0,
//               dh0_local = sum_{t<first head} P_t C_t dy_t (reverse walk);
//   chain_bwd : G[r] = dh_last_ext[r] + dh0_local[r+1] + decay[r+1] G[r+1]
//               when row r+1 continues row r -- the cotangent of h_last[r]
//               that the backward takes as dh_last.
// Across GPUs the same composition runs on per-rank summaries (the rank's
// chain_decay, its last h_last / first dh0), exchanged with one all_gather.
#include "scan_impl.cuh"

namespace pm {
namespace {

constexpr int kCpThreads = 128;
constexpr int kCpTile = 64;

PM_DEV bool row_continues(const int32_t* pos, const int32_t* cont, int64_t L, int r) {
  return cont != nullptr ? cont[r] != 0 : __ldg(pos + (int64_t)r * L) != 0;
}

__global__ void __launch_bounds__(256)
chain_fwd_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ cont, int64_t L,
                 const float* __restrict__ decay, const float* __restrict__ hll,
                 const float* __restrict__ h_init, float* __restrict__ h_in,
                 float* __restrict__ h_last, float* __restrict__ chain_decay, int R, int64_t DnN) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= DnN) return;
  bool c = row_continues(pos, cont, L, 0);
  float H = (c && h_init != nullptr) ? h_init[e] : 0.f;
  float D = c ? 1.f : 0.f;  // d h_last[R-1] / d h_init
  for (int r = 0; r < R; ++r) {
    if (r > 0) {
      c = row_continues(pos, cont, L, r);
      const int64_t p = (int64_t)(r - 1) * DnN + e;
      H = c ? fmaf(decay[p], H, hll[p]) : 0.f;
      D = c ? D : 0.f;
    }
    const int64_t i = (int64_t)r * DnN + e;
    h_in[i] = H;
    if (h_last != nullptr) h_last[i] = fmaf(decay[i], H, hll[i]);
    D *= decay[i];
  }
  if (chain_decay != nullptr) chain_decay[e] = D;
}

__global__ void __launch_bounds__(256)
chain_bwd_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ cont, int64_t L,
                 const float* __restrict__ decay, const float* __restrict__ dh0l,
                 const float* __restrict__ ext, const float* __restrict__ g_end,
                 float* __restrict__ G_out, float* __restrict__ dh_init, int R, int64_t DnN) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= DnN) return;
  int64_t i = (int64_t)(R - 1) * DnN + e;
  float G = (ext != nullptr ? ext[i] : 0.f) + (g_end != nullptr ? g_end[e] : 0.f);
  G_out[i] = G;
  for (int r = R - 2; r >= 0; --r) {
    const int64_t n = (int64_t)(r + 1) * DnN + e;
    i = (int64_t)r * DnN + e;
    const float carry = row_continues(pos, cont, L, r + 1) ? fmaf(decay[n], G, dh0l[n]) : 0.f;
    G = (ext != nullptr ? ext[i] : 0.f) + carry;
    G_out[i] = G;
  }
  if (dh_init != nullptr)
    dh_init[e] = row_continues(pos, cont, L, 0) ? fmaf(decay[e], G, dh0l[e]) : 0.f;
}

// C of a kCpTile window of row r to fp32 [t][n] in shared memory.
template <typename T, int N, bool kVec>
PM_DEV void stage_c(const T* __restrict__ C_r, int L, int j0, float (*sC)[N]) {
  for (int e = threadIdx.x; e < N * (kCpTile / 8); e += blockDim.x) {
    const int n = e % N, tb = (e / N) * 8;
    float v[8];
    load8<T, kVec>(C_r + (int64_t)n * L, j0 + tb, L, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) sC[tb + i][n] = v[i];
  }
}

PM_DEV float delta_of(float v, int softplus) { return softplus ? softplusf(v) : v; }

// Forward fix-up of the continuing prefix of each row: thread = channel,
// all N states (Ph = P_t h_in) in registers, sequential over the prefix.
template <typename T, int N, bool kVec, bool kGate>
__global__ void __launch_bounds__(kCpThreads)
fwd_fixup_kernel(const T* __restrict__ dt, const float* __restrict__ A, const T* __restrict__ C,
                 const float* __restrict__ dt_bias, int softplus, const int32_t* __restrict__ pos,
                 const T* __restrict__ z, const float* __restrict__ h_in, T* __restrict__ out,
                 float* __restrict__ states, int Dn, int L, int nchunk) {
  __shared__ __align__(16) float sC[kCpTile][N];
  __shared__ int s_red[kCpThreads / 32];
  const int r = blockIdx.y;
  const int32_t* pos_row = pos + (int64_t)r * L;
  if (__ldg(pos_row) == 0) return;  // the row starts a sequence: nothing to fix (CTA-uniform)
  const int fh = first_head_from(pos_row, L, 1, s_red);  // end of the continuing prefix
  const int d_raw = blockIdx.x * kCpThreads + threadIdx.x;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  const float bias = dt_bias ? __ldg(dt_bias + d) : 0.f;
  float A2[N], Ph[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    A2[n] = __ldg(A + (int64_t)d * N + n) * kLog2e;
    Ph[n] = __ldg(h_in + ((int64_t)r * Dn + d) * N + n);
  }
  auto fix_state = [&](int c) {  // checkpoint c = state entering step 16 c
    if (states != nullptr && active) {
      float* st = states + ((int64_t)r * nchunk + c) * N * Dn + d;
#pragma unroll
      for (int n = 0; n < N; ++n) st[(int64_t)n * Dn] += Ph[n];
    }
  };
  fix_state(0);
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* C_r = C + (int64_t)r * N * L;
  for (int tb = 0; tb < fh; tb += 8) {
    if ((tb & (kCpTile - 1)) == 0) {
      __syncthreads();
      stage_c<T, N, kVec>(C_r, L, tb, sC);
      __syncthreads();
    }
    float vv[8], yy[8], zz[8];
    load8<T, kVec>(dt + lane, tb, L, vv);
    load8<T, kVec>(out + lane, tb, L, yy);
    if constexpr (kGate) load8<T, kVec>(z + lane, tb, L, zz);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = tb + i;
      if (t >= fh) break;  // CTA-uniform
      const float delta = delta_of(vv[i] + bias, softplus);
      const float* Ct = sC[t & (kCpTile - 1)];
      float dy0 = 0.f, dy1 = 0.f;
#pragma unroll
      for (int n = 0; n < N; n += 2) {
        Ph[n] *= ex2(delta * A2[n]);
        Ph[n + 1] *= ex2(delta * A2[n + 1]);
        dy0 = fmaf(Ct[n], Ph[n], dy0);
        dy1 = fmaf(Ct[n + 1], Ph[n + 1], dy1);
      }
      float dyv = dy0 + dy1;
      if constexpr (kGate) dyv *= zz[i] * sigmoidf_fast(zz[i]);  // out = y silu(z)
      yy[i] += dyv;
      if (((t + 1) % kChunk) == 0 && t + 1 < L) fix_state((t + 1) / kChunk);
    }
    if (active) store8<T, kVec>(out + lane, tb, 0, fh, yy);
  }
}

// dh0_local[r,d,:] = sum_{t < first head} (prod_{i<=t} abar_i) C_t dy_t,
// dy = dout (x silu(z) with the gate): the reverse walk g_t = C_t dy_t +
// abar_{t+1} g_{t+1} over the continuing prefix, dh0 = abar_0 g_0.
template <typename T, int N, bool kVec, bool kGate>
__global__ void __launch_bounds__(kCpThreads)
dh0_kernel(const T* __restrict__ dt, const float* __restrict__ A, const T* __restrict__ C,
           const float* __restrict__ dt_bias, int softplus, const int32_t* __restrict__ pos,
           const T* __restrict__ z, const T* __restrict__ dout, float* __restrict__ dh0l, int Dn,
           int L) {
  __shared__ __align__(16) float sC[kCpTile][N];
  __shared__ int s_red[kCpThreads / 32];
  const int r = blockIdx.y;
  const int32_t* pos_row = pos + (int64_t)r * L;
  const int d_raw = blockIdx.x * kCpThreads + threadIdx.x;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  float* dst = dh0l + ((int64_t)r * Dn + d) * N;
  if (__ldg(pos_row) == 0) {  // the row starts a sequence: h0 is never read
    if (active) {
#pragma unroll
      for (int n = 0; n < N; ++n) dst[n] = 0.f;
    }
    return;
  }
  const int fh = first_head_from(pos_row, L, 1, s_red);
  const float bias = dt_bias ? __ldg(dt_bias + d) : 0.f;
  float A2[N], g[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    A2[n] = __ldg(A + (int64_t)d * N + n) * kLog2e;
    g[n] = 0.f;
  }
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* C_r = C + (int64_t)r * N * L;
  int j0 = -1;
  for (int tb = (fh - 1) & ~7; tb >= 0; tb -= 8) {
    if (j0 < 0 || tb < j0) {  // (CTA-uniform) stage the window holding tb
      j0 = tb & ~(kCpTile - 1);
      __syncthreads();
      stage_c<T, N, kVec>(C_r, L, j0, sC);
      __syncthreads();
    }
    float vv[8], yy[8], zz[8];
    load8<T, kVec>(dt + lane, tb, L, vv);
    load8<T, kVec>(dout + lane, tb, L, yy);
    if constexpr (kGate) load8<T, kVec>(z + lane, tb, L, zz);
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      const int t = tb + i;
      if (t >= fh) continue;  // CTA-uniform
      const float delta = delta_of(vv[i] + bias, softplus);
      float dyv = yy[i];
      if constexpr (kGate) dyv *= zz[i] * sigmoidf_fast(zz[i]);
      const float* Ct = sC[t - j0];
#pragma unroll
      for (int n = 0; n < N; ++n) g[n] = fmaf(Ct[n], dyv, g[n]) * ex2(delta * A2[n]);
    }
  }
  if (active) {
#pragma unroll
    for (int n = 0; n < N; ++n) dst[n] = g[n];
  }
}

template <typename T, int N, bool kVec>
void launch_fixup(const void* dt, const float* A, const void* C, const float* dt_bias, int sp,
                  const int32_t* pos, const void* z, const float* h_in, void* out, float* states,
                  int R, int Dn, int L, cudaStream_t s) {
  const dim3 grid((Dn + kCpThreads - 1) / kCpThreads, R);
  auto args = [&](auto kern) {
    kern<<<grid, kCpThreads, 0, s>>>(static_cast<const T*>(dt), A, static_cast<const T*>(C),
                                     dt_bias, sp, pos, static_cast<const T*>(z), h_in,
                                     static_cast<T*>(out), states, Dn, L, n_chunks(L));
  };
  if (z != nullptr) args(fwd_fixup_kernel<T, N, kVec, true>);
  else args(fwd_fixup_kernel<T, N, kVec, false>);
}

template <typename T, int N, bool kVec>
void launch_dh0(const void* dt, const float* A, const void* C, const float* dt_bias, int sp,
                const int32_t* pos, const void* z, const void* dout, float* dh0l, int R, int Dn,
                int L, cudaStream_t s) {
  const dim3 grid((Dn + kCpThreads - 1) / kCpThreads, R);
  auto args = [&](auto kern) {
    kern<<<grid, kCpThreads, 0, s>>>(static_cast<const T*>(dt), A, static_cast<const T*>(C),
                                     dt_bias, sp, pos, static_cast<const T*>(z),
                                     static_cast<const T*>(dout), dh0l, Dn, L);
  };
  if (z != nullptr) args(dh0_kernel<T, N, kVec, true>);
  else args(dh0_kernel<T, N, kVec, false>);
}

template <typename T>
struct TypeTag {
  using type = T;
};

// dispatch on (io, N, vec) for the two per-lane kernels
template <template <typename, int, bool> class F, typename... Args>
void dispatch(pm_dtype io, int N, bool vec, Args... args) {
  auto go = [&](auto t_tag, auto n_tag) {
    using T = typename decltype(t_tag)::type;
    constexpr int NN = decltype(n_tag)::value;
    if (vec) F<T, NN, true>()(args...);
    else F<T, NN, false>()(args...);
  };
  auto by_n = [&](auto t_tag) {
    if (N == 4) go(t_tag, std::integral_constant<int, 4>{});
    else if (N == 8) go(t_tag, std::integral_constant<int, 8>{});
    else go(t_tag, std::integral_constant<int, 16>{});
  };
  if (io == PM_F32) by_n(TypeTag<float>{});
  else by_n(TypeTag<__nv_bfloat16>{});
}
template <typename T, int N, bool kVec>
struct FixupF {
  template <typename... A>
  void operator()(A... a) const { launch_fixup<T, N, kVec>(a...); }
};
template <typename T, int N, bool kVec>
struct Dh0F {
  template <typename... A>
  void operator()(A... a) const { launch_dh0<T, N, kVec>(a...); }
};

pm_status check_chain(const int32_t* pos, const int32_t* cont, int64_t R, int64_t Dn, int64_t L,
                      int32_t N) {
  if (R < 1 || Dn < 1 || N < 1 || (pos == nullptr && cont == nullptr)) return PM_ERR_INVALID_ARG;
  if (pos != nullptr && cont == nullptr && L < 1) return PM_ERR_INVALID_ARG;
  if (Dn * N >= (int64_t(1) << 31)) return PM_ERR_SHAPE;
  return PM_OK;
}

}  // namespace
}  // namespace pm

using namespace pm;

extern "C" {

pm_status pm_scan_chain_fwd(const int32_t* pos, const int32_t* cont, const float* decay,
                            const float* h_last_local, const float* h_init, float* h_in,
                            float* h_last, float* chain_decay, int64_t R, int64_t Dn, int64_t L,
                            int32_t N, pm_stream_t stream) {
  pm_status st = check_chain(pos, cont, R, Dn, L, N);
  if (st != PM_OK) return st;
  if (!decay || !h_last_local || !h_in) return PM_ERR_INVALID_ARG;
  const int64_t DnN = Dn * N;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  chain_fwd_kernel<<<(unsigned)((DnN + 255) / 256), 256, 0, s>>>(
      pos, cont, L, decay, h_last_local, h_init, h_in, h_last, chain_decay, (int)R, DnN);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

pm_status pm_scan_chain_bwd(const int32_t* pos, const int32_t* cont, const float* decay,
                            const float* dh0_local, const float* dh_last_ext, const float* g_end,
                            float* dh_last, float* dh_init, int64_t R, int64_t Dn, int64_t L,
                            int32_t N, pm_stream_t stream) {
  pm_status st = check_chain(pos, cont, R, Dn, L, N);
  if (st != PM_OK) return st;
  if (!decay || !dh0_local || !dh_last) return PM_ERR_INVALID_ARG;
  const int64_t DnN = Dn * N;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  chain_bwd_kernel<<<(unsigned)((DnN + 255) / 256), 256, 0, s>>>(
      pos, cont, L, decay, dh0_local, dh_last_ext, g_end, dh_last, dh_init, (int)R, DnN);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

pm_status pm_selective_scan_fwd_fixup(const void* dt, const float* A, const void* C,
                                      const float* dt_bias, int32_t dt_softplus,
                                      const int32_t* pos, const void* z, const float* h_in,
                                      void* out, float* states, int64_t R, int64_t Dn, int64_t L,
                                      int32_t N, pm_dtype io, pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!dt || !A || !C || !pos || !h_in || !out) return PM_ERR_INVALID_ARG;
  for (const void* p : {dt, C, z, (const void*)out})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  if (!aligned16(states)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && aligned16(dt) && aligned16(C) && aligned16(z) &&
                   aligned16(out);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dispatch<FixupF>(io, N, vec, dt, A, C, dt_bias, dt_softplus ? 1 : 0, pos, z, h_in, out, states,
                   (int)R, (int)Dn, (int)L, s);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

pm_status pm_selective_scan_dh0(const void* dt, const float* A, const void* C, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos, const void* z,
                                const void* dout, float* dh0_local, int64_t R, int64_t Dn,
                                int64_t L, int32_t N, pm_dtype io, pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!dt || !A || !C || !pos || !dout || !dh0_local) return PM_ERR_INVALID_ARG;
  for (const void* p : {dt, C, z, dout})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && aligned16(dt) && aligned16(C) && aligned16(z) &&
                   aligned16(dout);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dispatch<Dh0F>(io, N, vec, dt, A, C, dt_bias, dt_softplus ? 1 : 0, pos, z, dout, dh0_local,
                 (int)R, (int)Dn, (int)L, s);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

}  // extern "C"
