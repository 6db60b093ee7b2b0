// scan_fwd.cu -- ScanOp_pack forward (Alg 2; Eq 1a/1b/2a
// P:202-205) and the segment schedule (plan + longest-first sort).
#include "scan_impl.cuh"

#ifndef PM_FWD_RING  // sub-blocks of u/dt in flight per thread (vector path); 1 = register prefetch
#define PM_FWD_RING 2
#endif

namespace pm {

// Work scheduling.  Segment lengths follow the sequence-length distribution
// (57..2048 steps), so a plain grid leaves a long tail.  A planning kernel
// lists every row's segments, one CTA sorts them longest-first, and the scan
// kernels are persistent: each CTA pulls (segment, channel-block) items from
// an atomic counter in that order (LPT), so the last items are the shortest.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) seg_plan_kernel(const int32_t* __restrict__ pos, int L,
                                                      int nseg, int P, int4* __restrict__ items) {
  // cut k (1 <= k < nseg) = first head at or after k * ceil(L / nseg), as in
  // segment_bounds(); one warp per cut, 32 positions per ballot
  __shared__ int cut[65];
  const int r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t* pos_row = pos + (int64_t)r * L;
  const int seg = (L + nseg - 1) / nseg;
  for (int k = 1 + warp; k < nseg; k += blockDim.x >> 5) {
    int b = L;
    // 128 positions per ballot round (4 per lane), one load round trip each
    for (int base = k * seg; base < L; base += 128) {
      int f = 4;  // first head among my 4 positions (4 = none)
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int t = base + 4 * lane + q;
        if (t < L && __ldg(pos_row + t) == 0) f = q;
      }
      const unsigned m = __ballot_sync(0xffffffffu, f < 4);
      if (m) {
        const int src = __ffs(m) - 1;
        b = base + 4 * src + __shfl_sync(0xffffffffu, f, src);
        break;
      }
    }
    if (lane == 0) cut[k] = min(b, L);
  }
  if (threadIdx.x == 0) {
    cut[0] = 0;
    cut[nseg] = L;
  }
  __syncthreads();
  // time split (P > 1): a segment longer than kPartLen is cut into up to P
  // parts at chunk boundaries (slot k*P + p; unused slots are empty)
  for (int k = threadIdx.x; k < nseg; k += blockDim.x) {
    const int c0 = cut[k], c1 = max(cut[k], cut[k + 1]), len = c1 - c0;
    const int np = P > 1 ? min(P, max(1, (len + kPartLen - 1) / kPartLen)) : 1;
    int b = c0;
    for (int p = 0; p < P; ++p) {
      const int e = p + 1 < np ? ((c0 + (int)((int64_t)(p + 1) * len / np)) & ~(kChunk - 1))
                               : c1;
      const int s1 = p < np ? max(b, e) : b;
      items[(r * nseg + k) * P + p] = make_int4(r, k * P + p, b, s1);
      b = s1;
    }
  }
}

// Longest-first order of the segment list (one CTA).  n <= 4096: exact rank
// sort (length descending, ties by index); larger n: bucket sort on 1024
// length bins (order within a bin is arbitrary -- results never depend on
// the processing order, only the load balance does).
__global__ void __launch_bounds__(1024) seg_sort_kernel(const int4* __restrict__ in, int n, int L,
                                                       int4* __restrict__ out) {
  if (n <= 4096) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int4 a = in[i];
      const int la = a.w - a.z;
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const int4 b = in[j];
        const int lb = b.w - b.z;
        rank += (lb > la) || (lb == la && j < i);
      }
      out[rank] = a;
    }
    return;
  }
  constexpr int kBins = 1024;
  __shared__ int cnt[kBins];
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  auto bin_of = [&](const int4 v) {  // longest first: bin 0 = longest
    const int len = v.w - v.z;
    return kBins - 1 - (int)(((int64_t)len * (kBins - 1)) / max(L, 1));
  };
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[bin_of(in[i])], 1);
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan -> bin cursors
    int acc = 0;
    for (int b = 0; b < kBins; ++b) {
      const int c = cnt[b];
      cnt[b] = acc;
      acc += c;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int4 v = in[i];
    out[atomicAdd(&cnt[bin_of(v)], 1)] = v;
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
// S threads per channel (S = 1: all N states in one thread; S > 1, for
// latency-bound launches: N/S states each, y summed over the S lanes by
// shuffle -- a few long segments then run S times as many warps).
#ifndef PM_FWD_TILE_PREFETCH
#define PM_FWD_TILE_PREFETCH 1
#endif
#ifndef PM_FWD_TILE_ASYNC
#define PM_FWD_TILE_ASYNC 1
#endif
template <typename T, int N, bool kVec, int MinB, bool kGate, bool kZoh, int S = 1>
__global__ void __launch_bounds__(kScanThreads, MinB)
scan_fwd_kernel(const ScanFwdArgs a) {
  constexpr int kCh = kScanThreads / S;  // channels per CTA
  constexpr int NS = N / S;              // states per thread
  static_assert(NS % 2 == 0, "states are processed in pairs");
  __shared__ __align__(16) float sB[kTile][N];
  __shared__ __align__(16) float sC[kTile][N];
  __shared__ unsigned sMask[kTile / 32];
  __shared__ int s_red[kScanWarps];
  __shared__ int s_work;
  constexpr bool kRing = kVec && PM_FWD_RING > 1;
  constexpr int kRingDepth = kRing ? PM_FWD_RING : 1;
  constexpr int kQv = (int)sizeof(T) / 2;  // 16-byte pieces per 8-element block
  static_assert((kRingDepth & (kRingDepth - 1)) == 0, "ring depth: power of 2");
  __shared__ __align__(16) uint4 ring[kRingDepth][2][kQv][kRing ? kScanThreads : 1];
  // one-lane-per-channel vector path: the next tile's raw B/C/pos arrive by
  // per-thread cp.async (issued right after a block's ring wait, so the next
  // block's wait completes them), converted at the tile boundary
  constexpr bool kTileAsync = kRing && S == 1 && PM_FWD_TILE_ASYNC != 0;
  __shared__ __align__(16) T tB[kTileAsync ? N : 1][kTileAsync ? kTile : 8];
  __shared__ __align__(16) T tC[kTileAsync ? N : 1][kTileAsync ? kTile : 8];
  __shared__ __align__(16) int32_t tP[kTileAsync ? kTile : 4];

  const int L = a.L, Dn = a.Dn;
  const int ndblk = (Dn + kCh - 1) / kCh;
  const int part = S > 1 ? (int)threadIdx.x % S : 0;
  const int n0 = part * NS;  // first state of this thread
  // the backward (launched programmatically behind this kernel) takes the SM
  // slots this kernel's CTAs leave; it waits per segment on a.done
  pdl_launch_dependents();
  for (int iter = 0;; ++iter) {
  int r, dblk, s0, s1;
  if (a.items != nullptr) {  // persistent: longest segments first
    __syncthreads();  // the previous item's states / y are written by every thread
    if (threadIdx.x == 0) {
      // release the finished item's segment (thread 0 re-reads its item
      // rather than keeping it in a register across the item)
      if (iter > 0) {
        // (counted in channels, so the backward's completion test, == Dn,
        // does not depend on this launch's channel-block width)
        const int4 pv = a.items[s_work / ndblk];
        const int pb = s_work % ndblk;
        red_release_add(a.done + pv.x * a.nseg + pv.y, min(kCh, Dn - pb * kCh));
      }
      s_work = atomicAdd(a.counter, 1);
    }
    __syncthreads();
    const int w = s_work;
    if (w >= a.n_items * ndblk) break;
    const int4 it = a.items[w / ndblk];
    r = it.x;
    dblk = w % ndblk;
    s0 = it.z;
    s1 = it.w;
  } else {
    if (iter > 0) break;
    r = blockIdx.y;
    dblk = blockIdx.x;
    segment_bounds(a.pos + (int64_t)r * L, L, blockIdx.z, a.nseg, s_red, s0, s1);
  }
  if (s0 >= s1) continue;
  const int d_raw = dblk * kCh + (int)threadIdx.x / S;
  const bool active = d_raw < Dn;
  const int d = active ? d_raw : Dn - 1;
  const int32_t* pos_row = a.pos + (int64_t)r * L;

  const T* B_r = static_cast<const T*>(a.B) + (int64_t)r * N * L;
  const T* C_r = static_cast<const T*>(a.C) + (int64_t)r * N * L;
  const int64_t lane = ((int64_t)r * Dn + d) * L;
  const T* u_row = static_cast<const T*>(a.u) + lane;
  const T* dt_row = static_cast<const T*>(a.dt) + lane;
  T* y_row = a.y ? static_cast<T*>(a.y) + lane : nullptr;
  const T* z_row = kGate ? static_cast<const T*>(a.z) + lane : nullptr;

  // states are processed in pairs with packed fp32x2 arithmetic (FFMA2)
  constexpr int NP = NS / 2;
  float2 A2[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p)
    A2[p] = make_float2(__ldg(a.A + (int64_t)d * N + n0 + 2 * p) * kLog2e,
                        __ldg(a.A + (int64_t)d * N + n0 + 2 * p + 1) * kLog2e);
  float2 invA[kZoh ? NP : 1];  // 1/A for the ZOH factor (inf at A = 0: series branch)
  if constexpr (kZoh) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
      invA[p] = make_float2(1.f / __ldg(a.A + (int64_t)d * N + n0 + 2 * p),
                            1.f / __ldg(a.A + (int64_t)d * N + n0 + 2 * p + 1));
  }
  const float Dd = (a.Dskip && part == 0) ? __ldg(a.Dskip + d) : 0.f;  // skip term once per channel
  const float bias = a.dt_bias ? __ldg(a.dt_bias + d) : 0.f;

  float2 h[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) h[p] = make_float2(0.f, 0.f);
  if (s0 == 0 && a.h0 != nullptr) {  // NEXT-2: state carried into the row
    const float* hp = a.h0 + ((int64_t)r * Dn + d) * N + n0;
#pragma unroll
    for (int p = 0; p < NP; ++p) h[p] = make_float2(__ldg(hp + 2 * p), __ldg(hp + 2 * p + 1));
  }

  // Flat loop over 8-step sub-blocks; u/dt of the next sub-block are loaded
  // into registers before the current one is computed (software pipeline),
  // B/C/head tiles are restaged at every kTile boundary.  Sub-blocks fully
  // inside the segment (all but at most two) run without per-step checks.
  int tb = s0 & ~7;
  float sdl = 0.f;    // sum of delta over the segment (decay summary)
  bool anyh = false;  // a head inside the segment
  Raw8<T, kVec> pu, pt, pz;
  // vector path: u/dt of the next kRingDepth-1 sub-blocks are in flight as
  // per-thread cp.async copies into a shared ring (each thread reads back
  // only its own slots: no barrier), deeper than one register block
  auto ring_issue = [&](int t) {
    if constexpr (kRing) {
      if (t < s1) {
        const int sl = (t >> 3) & (kRingDepth - 1);
#pragma unroll
        for (int q = 0; q < kQv; ++q) {  // fp32: the upper half may pass L (L % 8 == 4): zero-fill
          const int tq = t + q * 4;
          const int nb = tq < L ? 16 : 0;
          cp_async16(&ring[sl][0][q][threadIdx.x], nb ? u_row + tq : u_row, nb);
          cp_async16(&ring[sl][1][q][threadIdx.x], nb ? dt_row + tq : dt_row, nb);
        }
      }
      cp_async_commit();  // (empty past the segment: keeps the group count)
    }
  };
  if constexpr (kRing) {
#pragma unroll
    for (int q = 0; q < kRingDepth - 1; ++q) ring_issue(tb + 8 * q);
  } else {
    pu.load(u_row, tb, L);
    pt.load(dt_row, tb, L);
  }
  if (kGate) pz.load(z_row, tb, L);
  int j0 = -1;
  unsigned long long hmask = 0ull;
  // Latency-bound launches (S > 1 lanes per channel): B/C/pos of the NEXT
  // 64-step tile are loaded into registers a whole tile ahead, so the
  // staging's global latency (ncu: ~14 % of the stall samples at the bf16
  // conversions) overlaps the previous tile's steps -- 130m forward 0.443 ->
  // 0.421 ms.  The one-lane-per-channel launch (1.4B) keeps the synchronous
  // staging: at its 128-register cap the prefetch spills (0.808 -> 0.813 ms).
  TileRegs<T, N, kTile, kVec> tr;
  constexpr bool kTilePf = PM_FWD_TILE_PREFETCH != 0 && S > 1;
  if constexpr (kTilePf) tr.fetch(B_r, C_r, pos_row, L, tb & ~(kTile - 1));
  bool tile_pending = false;  // kTileAsync: the next tile's raw copies are to be issued
  auto tile_issue = [&](int jn) {  // raw B/C/pos of the tile at jn (cp.async, own slots)
    if constexpr (kTileAsync) {
      constexpr int kE = 16 / (int)sizeof(T);  // elements per 16-byte piece
      for (int e = threadIdx.x; e < 2 * N * (kTile / kE); e += blockDim.x) {
        const int arr = e / (N * (kTile / kE)), rem = e % (N * (kTile / kE));
        const int n = rem % N, q = rem / N;
        const int t0 = jn + q * kE;
        const int nb = t0 < L ? 16 : 0;  // (L % 4 == 0 on the vector path: whole pieces)
        const T* src = (arr == 0 ? B_r : C_r) + (int64_t)n * L;
        cp_async16(&(arr == 0 ? tB : tC)[n][q * kE], nb ? src + t0 : src, nb);
      }
      for (int e = threadIdx.x; e < kTile / 4; e += blockDim.x) {
        const int t0 = jn + 4 * e;
        const int nb = t0 < L ? 16 : 0;
        cp_async16(&tP[4 * e], nb ? pos_row + t0 : pos_row, nb);
      }
      cp_async_commit();
    }
  };
  for (; tb < s1; tb += 8) {
    if (j0 < 0 || (tb & (kTile - 1)) == 0) {  // CTA-uniform
      const bool first = j0 < 0;
      j0 = tb & ~(kTile - 1);
      __syncthreads();
      if constexpr (kTilePf) {
        tr.commit(L, j0, sB, sC, sMask, a.h0 == nullptr);
      } else if constexpr (kTileAsync) {
        if (first) {
          stage_bc<T, N, kTile, kVec>(B_r, C_r, pos_row, L, j0, sB, sC, sMask, a.h0 == nullptr);
        } else {  // the raw tile was fetched during the previous tile
          // (normally long complete; a segment that started late in the
          // previous tile may have issued it one block ago -- the wait also
          // covers this block's ring group, which the block needs anyway)
          cp_async_wait<0>();
          constexpr int kE = 16 / (int)sizeof(T);
          for (int e = threadIdx.x; e < 2 * N * (kTile / kE); e += blockDim.x) {
            const int arr = e / (N * (kTile / kE)), rem = e % (N * (kTile / kE));
            const int n = rem % N, q = rem / N;
#pragma unroll
            for (int i = 0; i < kE; ++i)
              (arr == 0 ? sB : sC)[q * kE + i][n] = IO<T>::cvt((arr == 0 ? tB : tC)[n][q * kE + i]);
          }
          __syncthreads();  // tP was written by other threads' copies (each waited on its own)
          if (threadIdx.x < 32) {
#pragma unroll
            for (int w0 = 0; w0 < kTile; w0 += 32) {
              const int t = j0 + w0 + (int)threadIdx.x;
              const bool f = t >= L || (t == 0 && a.h0 == nullptr) || tP[w0 + threadIdx.x] == 0;
              const unsigned m = __ballot_sync(0xffffffffu, f);
              if (threadIdx.x == 0) sMask[w0 / 32] = m;
            }
          }
        }
      } else {
        stage_bc<T, N, kTile, kVec>(B_r, C_r, pos_row, L, j0, sB, sC, sMask, a.h0 == nullptr);
      }
      __syncthreads();
      if constexpr (kTilePf) {
        if (j0 + kTile < s1) tr.fetch(B_r, C_r, pos_row, L, j0 + kTile);
      }
      if constexpr (kTileAsync) tile_pending = j0 + kTile < s1;
      // head flags of the tile as a register bitmask (CTA-uniform): no
      // shared-memory load on the per-step critical path
      hmask = (unsigned long long)sMask[0] | ((unsigned long long)sMask[1] << 32);
    }
    float uu[8], vv[8], yy[8], zz[8];
    if constexpr (kRing) {
      ring_issue(tb + 8 * (kRingDepth - 1));
      cp_async_wait<kRingDepth - 1>();  // this sub-block's group has landed
      if constexpr (kTileAsync) {
        // committed after this block's ring group: the next block's wait
        // completes it (one 8-step block of latency cover, no stall here)
        if (tile_pending) {
          tile_issue(j0 + kTile);
          tile_pending = false;
        }
      }
      const int sl = (tb >> 3) & (kRingDepth - 1);
      if constexpr (sizeof(T) == 2) {
        Raw8<T, kVec> ru, rt;
        ru.q = ring[sl][0][0][threadIdx.x];
        rt.q = ring[sl][1][0][threadIdx.x];
        ru.unpack(uu);
        rt.unpack(vv);
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float4 a4 = *reinterpret_cast<const float4*>(&ring[sl][0][q][threadIdx.x]);
          const float4 b4 = *reinterpret_cast<const float4*>(&ring[sl][1][q][threadIdx.x]);
          uu[4 * q] = a4.x; uu[4 * q + 1] = a4.y; uu[4 * q + 2] = a4.z; uu[4 * q + 3] = a4.w;
          vv[4 * q] = b4.x; vv[4 * q + 1] = b4.y; vv[4 * q + 2] = b4.z; vv[4 * q + 3] = b4.w;
        }
      }
    } else {
      pu.unpack(uu);
      pt.unpack(vv);
    }
    if (kGate) pz.unpack(zz);
    if (tb + 8 < s1) {
      if constexpr (!kRing) {
        pu.load(u_row, tb + 8, L);
        pt.load(dt_row, tb + 8, L);
      }
      if (kGate) pz.load(z_row, tb + 8, L);
    }
    const int sb = tb - j0;
    // checkpoint = state before step tb (only step i == 0 can be a multiple of kChunk)
    if (a.states != nullptr && (tb % kChunk) == 0 && tb >= s0 && active) {
      float* st = a.states + (((int64_t)r * a.nchunk + tb / kChunk) * N + n0) * Dn + d;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        st[(int64_t)(2 * p) * Dn] = h[p].x;
        st[(int64_t)(2 * p + 1) * Dn] = h[p].y;
      }
    }
    // kFull: all 8 steps inside the segment; kNoHead: and none is a head
    // (most blocks) -- no per-step check at all
    // delta of the 8 steps, two at a time (packed fp32x2)
    float dls[8];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const float2 v2 = make_float2(vv[i] + bias, vv[i + 1] + bias);
      const float2 d2 = a.softplus ? softplus2(v2) : v2;
      dls[i] = d2.x;
      dls[i + 1] = d2.y;
    }
    auto block = [&](auto full_tag, auto nohead_tag) {
      constexpr bool kFull = decltype(full_tag)::value;
      constexpr bool kNoHead = decltype(nohead_tag)::value;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = tb + i;
        yy[i] = 0.f;
        if (!kFull && (t < s0 || t >= s1)) continue;  // CTA-uniform
        const float delta = dls[i];
        const float2 dux2 = f2(delta * uu[i]), dl2 = f2(delta);
        const float2* Bt = reinterpret_cast<const float2*>(sB[sb + i] + n0);
        const float2* Ct = reinterpret_cast<const float2*>(sC[sb + i] + n0);
        if constexpr (kZoh) {  // B-bar u = f(z) delta B u (Eq 2b); abar needed at heads too
          const bool head = !kNoHead && ((hmask >> (sb + i)) & 1ull);
          const float2 u2 = f2(uu[i]);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const float2 m = fmul2(dl2, A2[p]);
            const float2 ab = ex2x2(m);
            const float2 zz2 = fmul2(m, f2(kLn2));
            const float2 bf = make_float2(zoh_bfac(ab.x, zz2.x, invA[p].x, delta),
                                          zoh_bfac(ab.y, zz2.y, invA[p].y, delta));
            const float2 bx = fmul2(bf, fmul2(u2, Bt[p]));
            h[p] = head ? bx : ffma2(ab, h[p], bx);
          }
        } else if (!kNoHead && ((hmask >> (sb + i)) & 1ull)) {
#pragma unroll
          for (int p = 0; p < NP; ++p) h[p] = fmul2(dux2, Bt[p]);
        } else {
#pragma unroll
          for (int p = 0; p < NP; ++p) h[p] = ffma2(ex2x2(fmul2(dl2, A2[p])), h[p], fmul2(dux2, Bt[p]));
        }
        float2 yp[2] = {make_float2(Dd * uu[i], 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int p = 0; p < NP; ++p) yp[p & 1] = ffma2(Ct[p], h[p], yp[p & 1]);
        const float2 ys = fadd2(yp[0], yp[1]);
        float yv = ys.x + ys.y;
#pragma unroll
        for (int o = 1; o < S; o <<= 1) yv += __shfl_xor_sync(0xffffffffu, yv, o);  // CTA-uniform path
        yy[i] = yv;
        if (kGate) yy[i] *= zz[i] * sigmoidf_fast(zz[i]);  // out = y * silu(z)
      }
    };
    if (tb >= s0 && tb + 8 <= s1) {
      if (((hmask >> sb) & 0xffull) == 0ull) block(std::true_type{}, std::true_type{});
      else block(std::true_type{}, std::false_type{});
    } else {
      block(std::false_type{}, std::false_type{});
    }
    if (active && part == 0 && y_row != nullptr) store8<T, kVec>(y_row, tb, s0, s1, yy);
    if (a.decay != nullptr) {  // NEXT-2 row summary: sum of delta, any head
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (tb + i >= s0 && tb + i < s1) {
          sdl += dls[i];
          anyh = anyh || ((hmask >> (sb + i)) & 1ull);
        }
      }
    }
  }
  if (s1 == L && a.decay != nullptr && active) {
    // d h_last / d h0 = prod_t abar_t = exp(A sum_t delta_t) when no slot of
    // the row is a head (the whole row is then one segment), else 0
    float* dp = a.decay + ((int64_t)r * Dn + d) * N + n0;
    const bool live = s0 == 0 && !anyh;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      dp[2 * p] = live ? ex2(A2[p].x * sdl) : 0.f;
      dp[2 * p + 1] = live ? ex2(A2[p].y * sdl) : 0.f;
    }
  }
  if (s1 == L && a.h_last != nullptr && active) {  // state after the row's last step
    float* hp = a.h_last + ((int64_t)r * Dn + d) * N + n0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      hp[2 * p] = h[p].x;
      hp[2 * p + 1] = h[p].y;
    }
  }
  }  // work loop
}

// ===========================================================================
// host side
// ===========================================================================
namespace {

// persistent grid: resident CTAs on all SMs, capped by the number of items
template <typename K>
int persistent_grid(K kern, int threads, size_t smem, int64_t items) {
  int nb = 1;
  const int nsm = sm_count();
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
  const int64_t g = (int64_t)nsm * std::max(nb, 1);
  if (getenv("PM_DEBUG"))
    fprintf(stderr, "[pm] persistent grid: nsm=%d blocks/SM=%d (err=%d) smem=%zu items=%lld -> %lld\n",
            nsm, nb, (int)e, smem, (long long)items, (long long)std::min<int64_t>(g, items));
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, items));
}

template <typename T, int N, bool kVec, int MinB, bool kGate, bool kZoh, int S = 1>
void fwd_go(const ScanFwdArgs& a, cudaStream_t s) {
  auto kern = scan_fwd_kernel<T, N, kVec, MinB, kGate, kZoh, S>;
  if (a.items != nullptr) {
    const int64_t nd = (a.Dn + kScanThreads / S - 1) / (kScanThreads / S);
    const int g = persistent_grid(kern, kScanThreads, 0, (int64_t)a.n_items * nd);
    kern<<<g, kScanThreads, 0, s>>>(a);
  } else {
    kern<<<dim3(n_dblk(a.Dn), a.R, a.nseg), kScanThreads, 0, s>>>(a);
  }
}

template <typename T, int N, bool kVec>
pm_status launch_fwd(const ScanFwdArgs& a, cudaStream_t s) {
  if (a.items != nullptr) {  // schedule: plan + sort (reads pos only), reset counter
    Sched sc = sched_of(a.states, a.R, a.Dn, a.L, N);
    if (cudaMemsetAsync(sc.counters, 0, 256 + done_bytes(a.R, a.L), s) != cudaSuccess)
      return PM_ERR_CUDA;
    launch_schedule(a.pos, a.R, a.L, a.nseg, 1, sc.unsorted, sc.sorted, s);
    PM_LAUNCH_CHECK();
  }
  if (a.zoh) {
    // ZOH carries 1/A and the series: 3 CTAs/SM (168 registers) avoid spills
    if (a.z != nullptr) fwd_go<T, N, kVec, 3, true, true>(a, s);
    else fwd_go<T, N, kVec, 3, false, true>(a, s);
  } else {
    if (a.z != nullptr) fwd_go<T, N, kVec, kFwdMinB, true, false>(a, s);
    else if (a.items != nullptr && fwd_split(a.R, a.L, a.Dn, N) > 1)
      fwd_go<T, N, kVec, kFwdMinB, false, false, kFwdSplit<N>>(a, s);
    else fwd_go<T, N, kVec, kFwdMinB, false, false>(a, s);
  }
  PM_LAUNCH_CHECK();
  return PM_OK;
}

template <typename T, int N>
pm_status dispatch_fwd_vec(const ScanFwdArgs& a, bool vec, cudaStream_t s) {
  return vec ? launch_fwd<T, N, true>(a, s) : launch_fwd<T, N, false>(a, s);
}

template <typename T>
pm_status dispatch_fwd_t(const ScanFwdArgs& a, int N, bool vec, cudaStream_t s) {
  switch (N) {
    case 4: return dispatch_fwd_vec<T, 4>(a, vec, s);
    case 8: return dispatch_fwd_vec<T, 8>(a, vec, s);
    default: return dispatch_fwd_vec<T, 16>(a, vec, s);
  }
}

}  // namespace

// segment (and, P > 1, part) list of every row, sorted longest-first
void launch_schedule(const int32_t* pos, int R, int L, int nseg, int P, int4* unsorted,
                     int4* sorted, cudaStream_t s) {
  seg_plan_kernel<<<R, 256, 0, s>>>(pos, L, nseg, P, unsorted);
  seg_sort_kernel<<<1, 1024, 0, s>>>(unsorted, R * nseg * P, L, sorted);
}

pm_status run_scan_fwd(const ScanFwdArgs& a, int N, bool vec, pm_dtype io, cudaStream_t s) {
  return io == PM_F32 ? dispatch_fwd_t<float>(a, N, vec, s) : dispatch_fwd_t<__nv_bfloat16>(a, N, vec, s);
}

}  // namespace pm
