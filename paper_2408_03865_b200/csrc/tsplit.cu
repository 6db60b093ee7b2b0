// tsplit.cu -- backward time split of long segments inside a row
// (latency-bound launches): the NEXT-2 context-parallel algebra of cp.cu
// applied to the parts of one segment.
//
// A segment (head-aligned) longer than kPartLen is cut at chunk boundaries
// into up to kMaxParts parts (seg_plan_kernel); every part is an independent
// work item of the persistent backward kernel, which starts pass A from the
// forward's checkpoint at the part's start (its TRUE state -- the forward is
// not split).  The only coupling is the reverse carry entering each part's
// end, linear in the following parts:
//   G[p] = dh0[p+1] + decay[p+1] G[p+1],
//   dh0[p] = sum_{t<first head} (prod_{s0<=i<=t} abar_i) C_t dy_t  (the part's
//            own dLoss/dh0; dh_last folded in for the part that ends the row),
//   decay[p] = prod abar over the part (0 if it holds a head, or if the part
//            starts a sequence).
// part_dh0 writes (dh0, decay) of every part (a reverse walk over the part's
// continuing prefix); the backward kernel composes G at each item's start.
#include "scan_impl.cuh"

namespace pm {
namespace {

constexpr int kTsThreads = 128;
constexpr int kTsTile = 128;

template <typename T, int N, bool kVec>
PM_DEV void stage_c_tile(const T* __restrict__ C_r, int L, int j0, float (*sC)[N]) {
  for (int e = threadIdx.x; e < N * (kTsTile / 8); e += blockDim.x) {
    const int n = e % N, tb = (e / N) * 8;
    float v[8];
    load8<T, kVec>(C_r + (int64_t)n * L, j0 + tb, L, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) sC[tb + i][n] = v[i];
  }
}

PM_DEV float delta_v(float v, int softplus) { return softplus ? softplusf(v) : v; }

// psum layout: ((slot * 2 + j) * N + n) * Dn + d
PM_DEV int64_t ps_idx(int64_t slot, int j, int n, int N, int Dn, int d) {
  return ((slot * 2 + j) * N + n) * Dn + d;
}

constexpr int kTsS = 4;  // lanes per channel in the pre-pass (N/kTsS states each)

// Each part's (dh0', decay): reverse walk of g_t = C_t dy_t + abar_{t+1}
// g_{t+1} over the part's continuing prefix, dh0 = abar_{s0} g_{s0}; decay =
// prod abar over the part when it holds no head; S lanes per channel, N/S
// independent states each.  Parts that start a sequence (or are the first
// of their segment) and empty slots get (0, 0).
template <typename T, int N, bool kVec, bool kGate>
__global__ void __launch_bounds__(kTsThreads)
part_dh0(const int4* __restrict__ items, int P, const T* __restrict__ dt,
         const float* __restrict__ A, const T* __restrict__ C, const float* __restrict__ dt_bias,
         int softplus, const int32_t* __restrict__ pos, const T* __restrict__ z,
         const T* __restrict__ dout, const float* __restrict__ dh_last,
         float* __restrict__ psum, int Dn, int L) {
  constexpr int S = kTsS, NS = N / S, kCh = kTsThreads / S;
  __shared__ __align__(16) float sC[kTsTile][N];
  __shared__ int s_red[kTsThreads / 32];
  const int64_t slot = blockIdx.y;
  const int4 it = items[slot];
  const int r = it.x, s0 = it.z, s1 = it.w;
  const int32_t* pos_row = pos + (int64_t)r * L;
  const int part = threadIdx.x % S, n0 = part * NS;
  const int d_raw = blockIdx.x * kCh + threadIdx.x / S;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  if (s0 >= s1 || it.y % P == 0 || __ldg(pos_row + s0) == 0) {  // (CTA-uniform)
    if (active) {
#pragma unroll
      for (int n = 0; n < NS; ++n) {
        psum[ps_idx(slot, 0, n0 + n, N, Dn, d)] = 0.f;
        psum[ps_idx(slot, 1, n0 + n, N, Dn, d)] = 0.f;
      }
    }
    return;
  }
  const int fh = min(s1, first_head_from(pos_row, L, s0 + 1, s_red));
  const float bias = dt_bias ? __ldg(dt_bias + d) : 0.f;
  float A2[NS], g[NS], pr[NS];
#pragma unroll
  for (int n = 0; n < NS; ++n) {
    A2[n] = __ldg(A + (int64_t)d * N + n0 + n) * kLog2e;
    g[n] = 0.f;
    pr[n] = 1.f;
  }
  const bool full = fh == s1;  // no head inside: the decay and dh_last pass through
  if (full && s1 == L && dh_last != nullptr) {
#pragma unroll
    for (int n = 0; n < NS; ++n) g[n] = __ldg(dh_last + ((int64_t)r * Dn + d) * N + n0 + n);
  }
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* C_r = C + (int64_t)r * N * L;
  int j0 = -1;
  // dt / dout (/ z) of the next (earlier) 8 steps are in flight while these
  // are computed (software pipeline: the walk is otherwise bound by one
  // dependent global load per 8 steps)
  const int tb_first = s0 + ((fh - 1 - s0) & ~7);
  Raw8<T, kVec> pv, py, pz;
  pv.load(dt + lane, tb_first, L);
  py.load(dout + lane, tb_first, L);
  if constexpr (kGate) pz.load(z + lane, tb_first, L);
  for (int tb = tb_first; tb >= s0; tb -= 8) {
    if (j0 < 0 || tb < j0) {  // (CTA-uniform) the window holding tb
      j0 = tb & ~(kTsTile - 1);
      __syncthreads();
      stage_c_tile<T, N, kVec>(C_r, L, j0, sC);
      __syncthreads();
    }
    float vv[8], yy[8], zz[8];
    pv.unpack(vv);
    py.unpack(yy);
    if constexpr (kGate) pz.unpack(zz);
    // delta of the 8 steps: the S lanes of a channel compute 8/S of them
    // each and share them by shuffle (instead of all S lanes all 8)
    float dls[8];
    {
      float mine[8 / S];
#pragma unroll
      for (int k = 0; k < 8 / S; ++k) mine[k] = delta_v(vv[part + S * k] + bias, softplus);
      const int base = (int)(threadIdx.x & 31) & ~(S - 1);
#pragma unroll
      for (int i = 0; i < 8; ++i) dls[i] = __shfl_sync(0xffffffffu, mine[i / S], base | (i % S));
    }
    if (tb - 8 >= s0) {
      pv.load(dt + lane, tb - 8, L);
      py.load(dout + lane, tb - 8, L);
      if constexpr (kGate) pz.load(z + lane, tb - 8, L);
    }
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      const int t = tb + i;
      if (t >= fh) continue;  // CTA-uniform
      const float delta = dls[i];
      float dyv = yy[i];
      if constexpr (kGate) dyv *= zz[i] * sigmoidf_fast(zz[i]);
      const float* Ct = sC[t - j0] + n0;
#pragma unroll
      for (int n = 0; n < NS; ++n) {
        const float ab = ex2(delta * A2[n]);
        g[n] = fmaf(Ct[n], dyv, g[n]) * ab;
        pr[n] *= ab;
      }
    }
  }
  if (active) {
#pragma unroll
    for (int n = 0; n < NS; ++n) {
      psum[ps_idx(slot, 0, n0 + n, N, Dn, d)] = g[n];
      psum[ps_idx(slot, 1, n0 + n, N, Dn, d)] = full ? pr[n] : 0.f;
    }
  }
}

template <typename T, int N, bool kVec>
pm_status part_bwd(const ScanBwdArgs& a, const int4* items, cudaStream_t s) {
  const dim3 grid((a.Dn + kTsThreads / kTsS - 1) / (kTsThreads / kTsS), a.R * a.nseg);
  auto go = [&](auto kern) {
    kern<<<grid, kTsThreads, 0, s>>>(items, a.nparts, static_cast<const T*>(a.dt), a.A,
                                     static_cast<const T*>(a.C), a.dt_bias, a.softplus, a.pos,
                                     static_cast<const T*>(a.z), static_cast<const T*>(a.dy),
                                     a.dh_last, const_cast<float*>(a.psum), a.Dn, a.L);
  };
  if (a.z != nullptr) go(part_dh0<T, N, kVec, true>);
  else go(part_dh0<T, N, kVec, false>);
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T>
pm_status bwd_t(const ScanBwdArgs& a, const int4* items, int N, bool vec, cudaStream_t s) {
  switch (N) {
    case 4: return vec ? part_bwd<T, 4, true>(a, items, s) : part_bwd<T, 4, false>(a, items, s);
    case 8: return vec ? part_bwd<T, 8, true>(a, items, s) : part_bwd<T, 8, false>(a, items, s);
    default: return vec ? part_bwd<T, 16, true>(a, items, s) : part_bwd<T, 16, false>(a, items, s);
  }
}

}  // namespace

pm_status run_part_bwd_pre(const ScanBwdArgs& a, int4* unsorted, int4* sorted, int* counters,
                           int N, bool vec, pm_dtype io, cudaStream_t s) {
  if (cudaMemsetAsync(counters, 0, 256, s) != cudaSuccess) return PM_ERR_CUDA;
  launch_schedule(a.pos, a.R, a.L, a.nseg / a.nparts, a.nparts, unsorted, sorted, s);
  PM_LAUNCH_CHECK();
  return io == PM_F32 ? bwd_t<float>(a, unsorted, N, vec, s)
                      : bwd_t<__nv_bfloat16>(a, unsorted, N, vec, s);
}

}  // namespace pm
