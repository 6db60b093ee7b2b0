// scan_bwd2.cu -- the "wide" ScanOp_pack backward (the backward's two
// scan operators with A-bar_{position_indices=0} -> 0), used for N = 16 on
// the TMA vector path without the gate or ZOH (the bench workloads); every
// other case runs scan_bwd.cu's kernel.
//
// Why a second layout: the ncu capture of scan_bwd_kernel (profiles/
// r02d_ncu_summary.md) shows its shared-memory pipe ~74 % busy (61.6
// wavefronts per warp-step of 256 elements), 57 % of it the warp transpose
// that sums dB_t = sum_d g du and dC_t = sum_d dy h over channels.  Here each
// thread of a lane pair serves TWO channels x N/2 states: the two channels'
// dB/dC terms are summed in registers (the FMUL that formed a term becomes
// an FFMA), so the transpose carries half the bytes per element, and B_t/C_t
// loads and per-step overhead are shared by two channels.
//
//   thread (j, hf) of a CTA: channel pair {2j, 2j+1} of the CTA's 128
//   channels, states [hf*N/2, hf*N/2 + N/2).  Its local channel 0 is channel
//   2j + hf (the one this lane FINISHES: du, ddt, dD, ddt_bias), local
//   channel 1 is 2j + (hf ^ 1) (finished by the partner lane), so the pair's
//   sum_n exchange is one shuffle per value with no select.
//   CTA = 128 threads (4 warps, one per TMEM lane quarter), 2 CTAs per SM:
//   each thread parks 16 states x 16 steps = 256 TMEM columns per chunk.
#include "scan_impl.cuh"

namespace pm {

constexpr int kW2Ch = kWideCh;             // channels per CTA (128)
constexpr int kW2Threads = kW2Ch;          // 64 channel pairs x 2 state halves
constexpr int kW2Warps = kW2Threads / 32;  // = 4: one warp per TMEM lane quarter
constexpr int kW2MinB = 2;                 // resident CTAs per SM (TMEM: 2 x 256 columns)
#ifndef PM_W2_AUNROLL  // steps unrolled per iteration of the full-chunk forward recompute
#define PM_W2_AUNROLL 4
#endif
#ifndef PM_W2_UNROLL  // 2-step rounds unrolled per iteration of the full-chunk reverse pass
#define PM_W2_UNROLL 2
#endif
constexpr int kW2AUnroll = PM_W2_AUNROLL;
constexpr int kW2Unroll = PM_W2_UNROLL;

template <typename T, int N>
struct W2Raw {  // raw inputs of one chunk, filled by TMA
  alignas(128) T u[kW2Ch][kChunk];
  alignas(128) T dt[kW2Ch][kChunk];
  alignas(128) T dy[kW2Ch][kChunk];
  alignas(128) T B[N][kChunk];
  alignas(128) T C[N][kChunk];
  alignas(128) int32_t pos[kChunk];
  alignas(128) float st[N][kW2Ch];
};

template <typename T, int N>
struct W2Smem {
  static constexpr int NH = N / 2;     // states per thread and channel
  static constexpr int kQ = N / 4;     // float4 quads of (dB | dC) per thread-step
  static constexpr int kRows = 2 * kQ; // transpose rows per 2-step round
  W2Raw<T, N> raw;
  // per-(t,d) scalars {delta, u, dy, softplus'(v)}, split by channel parity:
  // sc[d & 1][t][d >> 1] (a warp's load of one parity is 256 contiguous
  // bytes); after a round consumed them, {du, ddt} of the finishing lane
  float4 sc[2][kChunk][kW2Ch / 2];
  float4 red[kW2Warps][kRows][32];
  float4 xw[kChunk / 2][kW2Warps][kRows][2];
  static constexpr int kBS = N + 4;  // fp32 B/C rows [t][n], padded (conflicts)
  float B[kChunk][kBS];
  float C[kChunk][kBS];
  uint64_t bar;
  unsigned hmask[1];
  int s_red[kW2Warps];
  uint32_t tmem_base;
};

template <typename T, int N>
PM_DEV void w2_issue(W2Raw<T, N>& rw, const ScanBwdArgs& a, int r, int dblk, int c, int s0,
                     bool cont0, uint64_t* bar) {
  if (threadIdx.x != 0) return;
  const int cb = c * kChunk;
  const bool with_st = cb > s0 || (cb == 0 && a.h0 != nullptr) || (cb == s0 && cont0);
  const uint32_t bytes = 3 * kW2Ch * kChunk * sizeof(T) + 2 * N * kChunk * sizeof(T) +
                         kChunk * sizeof(int32_t) + (with_st ? N * kW2Ch * sizeof(float) : 0);
  mbar_expect_tx(bar, bytes);
  const int d0 = dblk * kW2Ch;
  tma_load<3>(rw.u, &a.tm_u, bar, cb, d0, r);
  tma_load<3>(rw.dt, &a.tm_dt, bar, cb, d0, r);
  tma_load<3>(rw.dy, &a.tm_dy, bar, cb, d0, r);
  tma_load<3>(rw.B, &a.tm_B, bar, cb, 0, r);
  tma_load<3>(rw.C, &a.tm_C, bar, cb, 0, r);
  tma_load<2>(rw.pos, &a.tm_pos, bar, cb, r);
  if (with_st) tma_load<4>(rw.st, &a.tm_st, bar, d0, 0, c, r);
}

// Split TMEM load: issue 16 columns of my lane into r (no wait) ...
PM_DEV void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// ... and wait for it: the registers are operands of the wait, so no use of
// them is scheduled before it (the load is asynchronous until the wait)
PM_DEV void tmem_ld16_wait(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
                 "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}

// 8-byte shared store kept as such (the compiler would merge two into a
// 16-byte store and copy the pairs into a register quad first)
PM_DEV void sts64(uint32_t addr, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

template <typename T, int N>
__global__ void __launch_bounds__(kW2Threads, kW2MinB)
scan_bwd_wide_kernel(const __grid_constant__ ScanBwdArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using SM = W2Smem<T, N>;
  constexpr int NH = SM::NH, kQ = SM::kQ, kRows = SM::kRows;
  constexpr int NP = NH / 2;  // packed fp32x2 state pairs per channel
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int L = a.L, Dn = a.Dn;
  const int tid = threadIdx.x, lid = tid & 31, wid = tid >> 5;
  const int j = tid >> 1, hf = tid & 1;
  const int n0 = hf * NH;
  const int ndblk = (Dn + kW2Ch - 1) / kW2Ch;
  constexpr uint32_t kCols = kChunk * 2 * NH;  // 256
  static_assert(kCols * kW2MinB <= 512, "TMEM columns per SM");
  if (wid == 0) tmem_alloc(&sm.tmem_base, kCols);
  if (tid == 32) mbar_init(&sm.bar, 1);
  uint32_t bar_phase = 0;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = sm.tmem_base + ((uint32_t)(wid * 32) << 16);
  // scalars of my local channel 0 (2j + hf) and 1 (2j + (hf ^ 1)); the
  // column of channel pair j in parity array h is j ^ 4h, so the two arrays
  // (16 KB apart: same banks) fall in opposite bank halves per quarter-warp
  float4(*P0)[kW2Ch / 2] = sm.sc[hf];
  float4(*P1)[kW2Ch / 2] = sm.sc[hf ^ 1];
  const int jc0 = j ^ (hf << 2), jc1 = j ^ ((hf ^ 1) << 2);
  const int jme = (tid >> 1) ^ ((tid & 1) << 2);  // column of block channel tid (phase 1, rows out)

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const int w = atomicAdd(a.counter, 1);
      sm.s_red[0] = w;
      if (w < a.n_items * ndblk && a.done != nullptr) {
        // programmatic launch behind the forward: wait until every forward
        // channel of this segment has released its states (bounded: trap)
        const int4 it = a.items[w / ndblk];
        const int* dp = a.done + it.x * a.nseg + it.y;
        int spin = 0;
        while (ld_acquire(dp) < a.Dn) {
          if (++spin > (1 << 24)) __trap();
          __nanosleep(256);
        }
        fence_proxy_async_global();  // the states are read by TMA (async proxy)
      }
    }
    __syncthreads();
    const int w = sm.s_red[0];
    __syncthreads();
    if (w >= a.n_items * ndblk) break;
    const int4 it = a.items[w / ndblk];
    const int r = it.x, k = it.y, dblk = w % ndblk, s0 = it.z, s1 = it.w;

    int dch[2];
    bool act[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int d = dblk * kW2Ch + 2 * j + (c ^ hf);
      act[c] = d < Dn;
      dch[c] = act[c] ? d : Dn - 1;
    }
    float* wsp = a.ws_param + (int64_t)(r * a.nseg + k) * (N + 2) * Dn;
    if (s0 >= s1) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (act[c]) {
#pragma unroll
          for (int q = 0; q < NH; ++q) wsp[(int64_t)(n0 + q) * Dn + dch[c]] = 0.f;
        }
      if (act[0]) {
        wsp[(int64_t)N * Dn + dch[0]] = 0.f;
        wsp[(int64_t)(N + 1) * Dn + dch[0]] = 0.f;
      }
      continue;
    }
    float* ws_bc_r = a.ws_bc + ((int64_t)dblk * a.R + r) * (int64_t)L * (2 * N);

    float2 A2[2][NP], g[2][NP], dA[2][NP];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float* Ap = a.A + (int64_t)dch[c] * N + n0 + 2 * p;
        A2[c][p] = make_float2(__ldg(Ap) * kLog2e, __ldg(Ap + 1) * kLog2e);
        g[c][p] = make_float2(0.f, 0.f);
        dA[c][p] = make_float2(0.f, 0.f);
      }
    const float Dd = a.Dskip ? __ldg(a.Dskip + dch[0]) : 0.f;  // local channel 0 only
    const float bias = a.dt_bias ? __ldg(a.dt_bias + dblk * kW2Ch + min(tid, Dn - 1 - dblk * kW2Ch)) : 0.f;
    float dD = 0.f, ddtb = 0.f;

    const int cfirst = s0 / kChunk, clast = (s1 - 1) / kChunk;
    const bool cont0 = s0 > 0 && __ldg(a.pos + (int64_t)r * L + s0) != 0;
    w2_issue<T, N>(sm.raw, a, r, dblk, clast, s0, cont0, &sm.bar);
    if (a.psum != nullptr && !(s1 == L && a.dh_last != nullptr)) {
      // time split: carry entering this part's end, composed from the
      // following parts' summaries (see scan_bwd.cu)
      const int P = a.nparts, pp0 = k % P;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float* base = a.psum + ((int64_t)r * a.nseg + (k - pp0)) * 2 * N * Dn + dch[c];
        for (int pp = P - 1; pp > pp0; --pp) {
          const float* ps = base + (int64_t)pp * 2 * N * Dn;
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const float2 h0v = make_float2(ps[(int64_t)(n0 + 2 * p) * Dn], ps[(int64_t)(n0 + 2 * p + 1) * Dn]);
            const float2 dec = make_float2(ps[(int64_t)(N + n0 + 2 * p) * Dn],
                                           ps[(int64_t)(N + n0 + 2 * p + 1) * Dn]);
            g[c][p] = ffma2(dec, g[c][p], h0v);
          }
        }
      }
    } else if (s1 == L && a.dh_last != nullptr) {  // NEXT-2: cotangent of the carried-out state
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float* gp = a.dh_last + ((int64_t)r * Dn + dch[c]) * N + n0;
#pragma unroll
        for (int p = 0; p < NP; ++p) g[c][p] = make_float2(__ldg(gp + 2 * p), __ldg(gp + 2 * p + 1));
      }
    }

    for (int ck = clast; ck >= cfirst; --ck) {
      const int cb = ck * kChunk, c0 = max(cb, s0), c1 = min(cb + kChunk, s1);
      mbar_wait(&sm.bar, bar_phase);
      bar_phase ^= 1u;
      __syncthreads();  // raw chunk visible; previous chunk's smem readers done
      // ---- phase 1: thread tid computes block channel tid's 16 scalars ----
      float2 h[2][NP];
      {
        const bool ach = dblk * kW2Ch + tid < Dn;
        float4(*dst)[kW2Ch / 2] = sm.sc[tid & 1];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float uu[8], vv[8], yy[8];
          smem_load8<T>(&sm.raw.u[tid][8 * half], uu);
          smem_load8<T>(&sm.raw.dt[tid][8 * half], vv);
          smem_load8<T>(&sm.raw.dy[tid][8 * half], yy);
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float2 v2 = make_float2(vv[i] + bias, vv[i + 1] + bias);
            float dl[2], sg[2];
            if (a.softplus) {
              float2 x2;
              const float2 d2 = softplus2_x(v2, x2);
              dl[0] = d2.x;
              dl[1] = d2.y;
              sg[0] = v2.x > 20.f ? 1.f : __fdividef(x2.x, 1.f + x2.x);
              sg[1] = v2.y > 20.f ? 1.f : __fdividef(x2.y, 1.f + x2.y);
            } else {
              dl[0] = v2.x;
              dl[1] = v2.y;
              sg[0] = sg[1] = 1.f;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e)
              dst[8 * half + i + e][jme] =
                  make_float4(dl[e], ach ? uu[i + e] : 0.f, ach ? yy[i + e] : 0.f, sg[e]);
          }
        }
        // B/C -> fp32 [t][n], two steps per thread (contiguous reads)
        for (int e = tid; e < N * kChunk / 2; e += kW2Threads) {
          const int n = e / (kChunk / 2), t = 2 * (e % (kChunk / 2));
          sm.B[t][n] = IO<T>::cvt(sm.raw.B[n][t]);
          sm.B[t + 1][n] = IO<T>::cvt(sm.raw.B[n][t + 1]);
          sm.C[t][n] = IO<T>::cvt(sm.raw.C[n][t]);
          sm.C[t + 1][n] = IO<T>::cvt(sm.raw.C[n][t + 1]);
        }
        if (tid < 32) {
          const int t = cb + tid;
          const bool f = tid < kChunk && (t >= L || (t == 0 && a.h0 == nullptr) ||
                                          sm.raw.pos[tid & (kChunk - 1)] == 0);
          const unsigned m = __ballot_sync(0xffffffffu, f);
          if (tid == 0) sm.hmask[0] = m;
        }
        if (cb > s0 || (cb == 0 && a.h0 != nullptr) || (cb == s0 && cont0)) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int dl = 2 * j + (c ^ hf);
#pragma unroll
            for (int p = 0; p < NP; ++p)
              h[c][p] = make_float2(sm.raw.st[n0 + 2 * p][dl], sm.raw.st[n0 + 2 * p + 1][dl]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int p = 0; p < NP; ++p) h[c][p] = make_float2(0.f, 0.f);
        }
      }
      __syncthreads();  // scalars visible; raw buffer free
      const uint32_t hmask = sm.hmask[0];
      if (ck > cfirst) w2_issue<T, N>(sm.raw, a, r, dblk, ck - 1, s0, cont0, &sm.bar);

      // warp transpose-reduce of a round's dB/dC terms over the warp's 16
      // channel pairs (lane -> row, state half, column half), then park my
      // channel's (du, ddt) of the round's steps in their consumed slots
      auto reduce_round = [&](const int rs, const float (&fdu)[2], const float (&fddt)[2]) {
        __syncwarp();
        {
          const int row = lid >> 2, rh = lid & 1, ch = (lid >> 1) & 1;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < kRows) {
            const float4* rp = &sm.red[wid][row][2 * ch + rh];
            const int o = (row & 1) << 2;
            float4 p0 = rp[0 ^ o], p1 = rp[4 ^ o], p2 = rp[8 ^ o], p3 = rp[12 ^ o];
            float4 p4 = rp[16 ^ o], p5 = rp[20 ^ o], p6 = rp[24 ^ o], p7 = rp[28 ^ o];
            auto lo = [](float4 v) { return make_float2(v.x, v.y); };
            auto hi = [](float4 v) { return make_float2(v.z, v.w); };
            const float2 sl = fadd2(fadd2(fadd2(lo(p0), lo(p1)), fadd2(lo(p2), lo(p3))),
                                    fadd2(fadd2(lo(p4), lo(p5)), fadd2(lo(p6), lo(p7))));
            const float2 sh = fadd2(fadd2(fadd2(hi(p0), hi(p1)), fadd2(hi(p2), hi(p3))),
                                    fadd2(fadd2(hi(p4), hi(p5)), fadd2(hi(p6), hi(p7))));
            acc = make_float4(sl.x, sl.y, sh.x, sh.y);
          }
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
          acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 2);
          acc.w += __shfl_xor_sync(0xffffffffu, acc.w, 2);
          if (row < kRows && ch == 0) sm.xw[rs][wid][row][rh] = acc;
        }
        __syncwarp();
        // (both lanes of a pair read the round's scalars before the sync)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          *reinterpret_cast<float2*>(&P0[2 * rs + i][jc0]) = make_float2(fdu[i], fddt[i]);
      };
      // one reverse step t = cb + ii given the state after it (hc), the state
      // entering it (hpv) and its abar (ab; unused at a head):
      //   g += C dy;  S += g B;  dB <- sum_c g du;  dC <- sum_c dy h_t;
      //   g <- abar g (0 at heads);  q = g h_{t-1};  dA += delta q;  dq += A q
      // The step's dB/dC terms go to transpose row i of the round.
      auto bstep = [&](const int ii, const int i, const bool head, const float2 (&hc)[2][NP],
                       const float2 (&hpv)[2][NP], const float2 (&ab)[2][NP], float& fdu,
                       float& fddt) {
        const float4 sv0 = P0[ii][jc0], sv1 = P1[ii][jc1];
        const float4 sv[2] = {sv0, sv1};
        const float2* Bt = reinterpret_cast<const float2*>(&sm.B[ii][n0]);
        const float2* Ct = reinterpret_cast<const float2*>(&sm.C[ii][n0]);
        float2 vB[NP], vC[NP], Sp[2], dqp[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float2 dux2 = f2(sv[c].x * sv[c].y), dy2 = f2(sv[c].z);
          Sp[c] = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            g[c][p] = ffma2(Ct[p], dy2, g[c][p]);
            Sp[c] = ffma2(g[c][p], Bt[p], Sp[c]);
            vB[p] = c == 0 ? fmul2(g[c][p], dux2) : ffma2(g[c][p], dux2, vB[p]);
            vC[p] = c == 0 ? fmul2(dy2, hc[c][p]) : ffma2(dy2, hc[c][p], vC[p]);
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float2 dl2 = f2(sv[c].x);
          dqp[c] = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if (head) {  // abar = 0: no carry, no dA / dq term
              g[c][p] = make_float2(0.f, 0.f);
            } else {
              g[c][p] = fmul2(ab[c][p], g[c][p]);  // carry to t-1
              const float2 q = fmul2(g[c][p], hpv[c][p]);
              dA[c][p] = ffma2(dl2, q, dA[c][p]);
              dqp[c] = ffma2(A2[c][p], q, dqp[c]);
            }
          }
        }
        // (two 8-byte stores per slot: the fp32x2 pairs are register pairs
        // already, a 16-byte store would first copy them into a quad)
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const uint32_t slot = smem_u32(&sm.red[wid][i * kQ + q][lid]);
          sts64(slot, q < NP / 2 ? vB[2 * q] : vC[2 * q - NP]);
          sts64(slot + 8, q < NP / 2 ? vB[2 * q + 1] : vC[2 * q + 1 - NP]);
        }
        // sum_n over the pair: keep local channel 0, send local channel 1
        const float S = (Sp[0].x + Sp[0].y) + __shfl_xor_sync(0xffffffffu, Sp[1].x + Sp[1].y, 1);
        const float dq = (dqp[0].x + dqp[0].y) + __shfl_xor_sync(0xffffffffu, dqp[1].x + dqp[1].y, 1);
        fdu = fmaf(Dd, sv0.z, sv0.x * S);
        fddt = fmaf(sv0.y, S, dq * kLn2) * sv0.w;
        dD = fmaf(sv0.z, sv0.y, dD);
        ddtb += fddt;
      };
      auto abar = [&](const int ii, float2 (&ab)[2][NP]) {
        const float d0 = P0[ii][jc0].x, d1 = P1[ii][jc1].x;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          ab[0][p] = ex2x2(fmul2(f2(d0), A2[0][p]));
          ab[1][p] = ex2x2(fmul2(f2(d1), A2[1][p]));
        }
      };

      if (c0 == cb && c1 == cb + kChunk && hmask == 0u) {
        // ---- hot path: a full chunk without sequence heads: no per-step
        // head branch, so the scheduler interleaves the MUFU exponentials
        // with the FMA work around them.  Pass A parks the state entering
        // every step in TMEM columns [16 ii, 16 ii + 16); pass B loads a
        // round's second-step state during the previous round's transpose
        // and its first-step state during the second step's arithmetic.
#pragma unroll kW2AUnroll
        for (int ii = 0; ii < kChunk; ++ii) {
          tmem_st<2 * NH>(tbase + (uint32_t)(ii * 2 * NH), reinterpret_cast<const float*>(h));
          const float4 sv0 = P0[ii][jc0], sv1 = P1[ii][jc1];
          const float2 dl2[2] = {f2(sv0.x), f2(sv1.x)};
          const float2 dux2[2] = {f2(sv0.x * sv0.y), f2(sv1.x * sv1.y)};
          const float2* Bt = reinterpret_cast<const float2*>(&sm.B[ii][n0]);
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int p = 0; p < NP; ++p)
              h[c][p] = ffma2(ex2x2(fmul2(dl2[c], A2[c][p])), h[c][p], fmul2(dux2[c], Bt[p]));
        }
        tmem_wait_st();
        auto unpack = [&](const uint32_t (&r)[16], float2 (&v)[2][NP]) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int p = 0; p < NP; ++p)
              v[c][p] = make_float2(__uint_as_float(r[c * NH + 2 * p]), __uint_as_float(r[c * NH + 2 * p + 1]));
        };
        uint32_t pre1[16];
        tmem_ld16_issue(tbase + (uint32_t)((kChunk - 1) * 2 * NH), pre1);
#pragma unroll kW2Unroll
        for (int rs = kChunk / 2 - 1; rs >= 0; --rs) {
          const int k0 = 2 * rs;
          float2 hp0[2][NP], hp1[2][NP], ab[2][NP];
          uint32_t r0[16];
          tmem_ld16_wait(pre1);
          unpack(pre1, hp1);
          tmem_ld16_issue(tbase + (uint32_t)(k0 * 2 * NH), r0);
          float fdu[2], fddt[2];
          abar(k0 + 1, ab);
          bstep(k0 + 1, 1, false, h, hp1, ab, fdu[1], fddt[1]);
          tmem_ld16_wait(r0);
          unpack(r0, hp0);
          abar(k0, ab);
          bstep(k0, 0, false, hp1, hp0, ab, fdu[0], fddt[0]);
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int p = 0; p < NP; ++p) h[c][p] = hp0[c][p];
          if (rs > 0) tmem_ld16_issue(tbase + (uint32_t)((k0 - 1) * 2 * NH), pre1);
          reduce_round(rs, fdu, fddt);
        }
      } else {
        // ---- generic path (a partial chunk, or sequence heads inside):
        // every step's entering state parked in TMEM, per-step checks ----
        const bool full = c0 == cb && c1 == cb + kChunk;
#pragma unroll 1
        for (int ii = 0; ii < kChunk; ++ii) {
          const int t = cb + ii;
          tmem_st<2 * NH>(tbase + (uint32_t)(ii * 2 * NH), reinterpret_cast<const float*>(h));
          if (!full && (t < c0 || t >= c1)) continue;  // CTA-uniform
          const float4 sv0 = P0[ii][jc0], sv1 = P1[ii][jc1];
          const float2 dux2[2] = {f2(sv0.x * sv0.y), f2(sv1.x * sv1.y)};
          const float2* Bt = reinterpret_cast<const float2*>(&sm.B[ii][n0]);
          if ((hmask >> ii) & 1u) {  // reset: h = delta u B (a select, never 0 * h)
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int p = 0; p < NP; ++p) h[c][p] = fmul2(dux2[c], Bt[p]);
          } else {
            float2 ab[2][NP];
            abar(ii, ab);
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int p = 0; p < NP; ++p) h[c][p] = ffma2(ab[c][p], h[c][p], fmul2(dux2[c], Bt[p]));
          }
        }
        tmem_wait_st();
#pragma unroll 1
        for (int rs = kChunk / 2 - 1; rs >= 0; --rs) {
          const int a0 = cb + 2 * rs;
          float2 hp[2][2][NP];  // [step][local channel][pair]: states entering a0, a0+1
          tmem_ld<4 * NH>(tbase + (uint32_t)(rs * 4 * NH), reinterpret_cast<float*>(hp));
          if (a0 >= c1 || a0 + 2 <= c0) {  // CTA-uniform: the round is outside the item
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int p = 0; p < NP; ++p) h[c][p] = hp[0][c][p];
            continue;
          }
          float fdu[2], fddt[2];
#pragma unroll
          for (int i = 1; i >= 0; --i) {
            const int t = a0 + i, ii = t - cb;
            if (t < c0 || t >= c1) {  // CTA-uniform
#pragma unroll
              for (int q = 0; q < kQ; ++q) sm.red[wid][i * kQ + q][lid] = make_float4(0.f, 0.f, 0.f, 0.f);
              fdu[i] = fddt[i] = 0.f;
              continue;
            }
            const bool head = (hmask >> ii) & 1u;
            float2 ab[2][NP];
            if (!head) abar(ii, ab);
            bstep(ii, i, head, i == 1 ? h : hp[1], hp[i], ab, fdu[i], fddt[i]);
          }
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int p = 0; p < NP; ++p) h[c][p] = hp[0][c][p];
          reduce_round(rs, fdu, fddt);
        }
      }
      // ---- cross-warp sum of the chunk's dB/dC partials: one barrier ----
      __syncthreads();
      {
        constexpr int kV4 = 2 * N / 4;  // float4 groups per step
        for (int e = tid; e < kChunk * kV4; e += kW2Threads) {
          const int s16 = e / kV4, v = 4 * (e % kV4);
          const int t = cb + s16;
          if (t >= c0 && t < c1) {
            const int n = v < N ? v : v - N;
            const int rh = n / NH;
            const int kk = (v < N ? 0 : NH) + n % NH;
            const int row = (s16 & 1) * kQ + kk / 4;
            float4 acc = sm.xw[s16 >> 1][0][row][rh];
#pragma unroll
            for (int w2 = 1; w2 < kW2Warps; ++w2) {
              const float4 q = sm.xw[s16 >> 1][w2][row][rh];
              const float2 lo = fadd2(make_float2(acc.x, acc.y), make_float2(q.x, q.y));
              const float2 hi = fadd2(make_float2(acc.z, acc.w), make_float2(q.z, q.w));
              acc = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
            *reinterpret_cast<float4*>(ws_bc_r + (int64_t)t * (2 * N) + v) = acc;
          }
        }
      }
      // ---- du / ddt rows of the chunk: thread tid writes block channel tid
      {
        const int dd = dblk * kW2Ch + tid;
        if (dd < Dn) {
          const float4(*src)[kW2Ch / 2] = sm.sc[tid & 1];
          float vu[2][8], vd[2][8];
#pragma unroll
          for (int ii = 0; ii < kChunk; ++ii) {
            const float2 q = *reinterpret_cast<const float2*>(&src[ii][jme]);
            vu[ii >> 3][ii & 7] = q.x;
            vd[ii >> 3][ii & 7] = q.y;
          }
          T* du_row = static_cast<T*>(a.du) + ((int64_t)r * Dn + dd) * L;
          T* ddt_row = static_cast<T*>(a.ddt) + ((int64_t)r * Dn + dd) * L;
          store8<T, true>(du_row, cb, c0, c1, vu[0]);
          store8<T, true>(du_row, cb + 8, c0, c1, vu[1]);
          store8<T, true>(ddt_row, cb, c0, c1, vd[0]);
          store8<T, true>(ddt_row, cb + 8, c0, c1, vd[1]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (!act[c]) continue;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        wsp[(int64_t)(n0 + 2 * p) * Dn + dch[c]] = dA[c][p].x;
        wsp[(int64_t)(n0 + 2 * p + 1) * Dn + dch[c]] = dA[c][p].y;
      }
      if (s0 == 0 && a.dh0 != nullptr) {  // NEXT-2: g now holds abar_0 g_0 = dL/dh0
        float* gp = a.dh0 + ((int64_t)r * Dn + dch[c]) * N + n0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          gp[2 * p] = g[c][p].x;
          gp[2 * p + 1] = g[c][p].y;
        }
      }
    }
    if (act[0]) {
      wsp[(int64_t)N * Dn + dch[0]] = dD;
      wsp[(int64_t)(N + 1) * Dn + dch[0]] = ddtb;
    }
  }  // work loop
  if (tid == 0) {
    // the last CTA out resets the schedule counters for the next launch
    if (atomicAdd(a.counter + 1, 1) == (int)gridDim.x - 1) {
      a.counter[0] = 0;
      a.counter[1] = 0;
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (wid == 0) {
    tmem_fence_after();
    tmem_dealloc(sm.tmem_base, kCols);
  }
}

namespace {
template <typename T>
pm_status launch_wide_t(const ScanBwdArgs& a, cudaStream_t s) {
  constexpr int N = 16;
  const size_t smem = sizeof(W2Smem<T, N>);
  auto kern = scan_bwd_wide_kernel<T, N>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return PM_ERR_CUDA;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return PM_ERR_CUDA;
  int dev = 0, smem_sm = 228 * 1024, resv = 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  const int nb = std::max(1, std::min<int>(kW2MinB, (int)(smem_sm / (smem + resv))));
  const int64_t items = (int64_t)a.n_items * n_dblk_wide(a.Dn);
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count() * nb, items));
  if (getenv("PM_DEBUG"))
    fprintf(stderr, "[pm] wide bwd persistent grid: %d x %d CTAs/SM (smem %zu) -> %d\n", sm_count(),
            nb, smem, g);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(kW2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // programmatic launch only behind the library's own forward (see scan_bwd.cu)
  const bool pdl = a.pdl && a.done != nullptr && getenv("PM_NO_PDL") == nullptr &&
                   (getenv("PM_PDL") != nullptr || fwd_throughput_bound(a.R, a.L, a.Dn));
  cfg.numAttrs = pdl ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return PM_ERR_CUDA;
  PM_LAUNCH_CHECK();
  return PM_OK;
}
}  // namespace

pm_status launch_scan_bwd_wide(const ScanBwdArgs& a, pm_dtype io, cudaStream_t s) {
  return io == PM_F32 ? launch_wide_t<float>(a, s) : launch_wide_t<__nv_bfloat16>(a, s);
}

}  // namespace pm
