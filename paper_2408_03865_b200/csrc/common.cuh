// common.cuh -- device helpers shared by libpm's sm_100a kernels.
// (Product path.  Shares nothing with oracle/.)
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors; no driver library link needed)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pm.h"

#define PM_DEV __device__ __forceinline__

namespace pm {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ---------------------------------------------------------------- math ----
PM_DEV float ex2(float x) {  // MUFU.EX2 (flush-to-zero)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
PM_DEV float rcp(float x) {  // MUFU.RCP
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
PM_DEV float sigmoidf_fast(float v) { return rcp(1.f + ex2(-v * kLog2e)); }

// Eq 2b (ZOH): B-bar = f(z) delta B, f(z) = (e^z - 1)/z, z = delta A.
// bfac = f(z) delta: for |z| >= 0.1 as (abar - 1) / A from the abar = e^z the
// scan computes anyway; below, delta (1 + z/2 + z^2/6 + z^3/24 + z^4/120)
// (truncation < 2e-8 relative; no cancellation).  A select, so A = 0 (1/A =
// inf) takes the series.  dfp = delta f'(z) = (e^z - f)/A, series
// delta (1/2 + z/3 + z^2/8 + z^3/30 + z^4/144).
PM_DEV float zoh_series_f(float z) {
  return fmaf(z, fmaf(z, fmaf(z, fmaf(z, 1.f / 120.f, 1.f / 24.f), 1.f / 6.f), 0.5f), 1.f);
}
PM_DEV float zoh_series_df(float z) {
  return fmaf(z, fmaf(z, fmaf(z, fmaf(z, 1.f / 144.f, 1.f / 30.f), 1.f / 8.f), 1.f / 3.f), 0.5f);
}
PM_DEV float zoh_bfac(float ab, float z, float invA, float dl) {
  return fabsf(z) < 0.1f ? dl * zoh_series_f(z) : fmaf(ab, invA, -invA);
}
// (bfac, delta f'(z)); rdl = 1/delta
PM_DEV void zoh_coef(float ab, float z, float invA, float dl, float rdl, float& bfac, float& dfp) {
  if (fabsf(z) < 0.1f) {
    bfac = dl * zoh_series_f(z);
    dfp = dl * zoh_series_df(z);
  } else {
    bfac = fmaf(ab, invA, -invA);
    dfp = fmaf(-bfac, rdl, ab) * invA;
  }
}

// Packed fp32x2 arithmetic (sm_100a FFMA2/FMUL2/FADD2): two IEEE fp32
// operations per instruction, bit-identical to the scalar ones.
PM_DEV float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
PM_DEV float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
PM_DEV float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
PM_DEV float2 f2(float v) { return make_float2(v, v); }
PM_DEV float2 ex2x2(float2 a) { return make_float2(ex2(a.x), ex2(a.y)); }

PM_DEV float lg2(float x) {  // MUFU.LG2
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// softplus(v) = log(1 + x), x = e^v (reading Q4).  Branch-free and short:
//  * x < 1/32: 5-term Taylor series of log1p (relative error < x^5/6 < 2e-9)
//    -- keeps full accuracy where delta is tiny (dt ~ 1e-4);
//  * x >= 1/32: lg2.approx(1 + x) * ln2 (absolute error ~1.7e-7, i.e.
//    < 6e-6 relative since log1p(x) >= 0.03 there);
//  * v > 20: v (error < 2e-9 relative).
// Also returns x (callers derive sigmoid(v) = x / (1 + x) from it).
PM_DEV float softplus_x(float v, float& x) {
  x = ex2(v * kLog2e);
  const float p = x * fmaf(x, fmaf(x, fmaf(x, fmaf(x, 0.2f, -0.25f), 0.33333334f), -0.5f), 1.f);
  const float l = lg2(1.f + x) * kLn2;
  const float d = x < 0.03125f ? p : l;
  return v > 20.f ? v : d;
}
PM_DEV float softplusf(float v) {
  float x;
  return softplus_x(v, x);
}
// Two at once with packed fp32x2 arithmetic (same operations and rounding
// as softplus_x per lane; FFMA2/FMUL2 are bit-identical to the scalar ops).
PM_DEV float2 softplus2_x(float2 v, float2& x) {
  x = ex2x2(fmul2(v, f2(kLog2e)));
  float2 q = ffma2(x, f2(0.2f), f2(-0.25f));
  q = ffma2(x, q, f2(0.33333334f));
  q = ffma2(x, q, f2(-0.5f));
  q = ffma2(x, q, f2(1.f));
  const float2 pp = fmul2(x, q);
  const float2 onex = fadd2(f2(1.f), x);
  const float2 l = fmul2(make_float2(lg2(onex.x), lg2(onex.y)), f2(kLn2));
  return make_float2(v.x > 20.f ? v.x : (x.x < 0.03125f ? pp.x : l.x),
                     v.y > 20.f ? v.y : (x.y < 0.03125f ? pp.y : l.y));
}
PM_DEV float2 softplus2(float2 v) {
  float2 x;
  return softplus2_x(v, x);
}

// ----------------------------------------------------------------- I/O ----
template <typename T> struct IO;
template <> struct IO<float> {
  static PM_DEV float ld(const float* p) { return __ldg(p); }
  static PM_DEV void st(float* p, float v) { *p = v; }
  static PM_DEV float cvt(float v) { return v; }
  static PM_DEV float from(float v) { return v; }
  static constexpr int kIsz = 4;
};
template <> struct IO<__nv_bfloat16> {
  static PM_DEV float ld(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
  static PM_DEV void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
  static PM_DEV float cvt(__nv_bfloat16 v) { return __bfloat162float(v); }
  static PM_DEV __nv_bfloat16 from(float v) { return __float2bfloat16_rn(v); }
  static constexpr int kIsz = 2;
};

// Load 8 consecutive elements p[i..i+7] of a row of length n (elements
// outside [0, n) read as 0).  kVec: caller guarantees 16-byte alignment of
// p + i whenever i % 8 == 0 and the whole vector is inside the row.
template <typename T, bool kVec>
PM_DEV void load8(const T* __restrict__ p, int64_t i, int64_t n, float (&v)[8]) {
  if (kVec && i >= 0 && i + 8 <= n) {
    if constexpr (sizeof(T) == 2) {
      uint4 q = __ldg(reinterpret_cast<const uint4*>(p + i));
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 f = __bfloat1622float2(b[k]);
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
      }
    } else {
      float4 a = __ldg(reinterpret_cast<const float4*>(p + i));
      float4 b = __ldg(reinterpret_cast<const float4*>(p + i + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      v[k] = (i + k >= 0 && i + k < n) ? IO<T>::ld(p + i + k) : 0.f;
  }
}

// Store v[k] to p[i+k] for the k with lo <= i+k < hi.
template <typename T, bool kVec>
PM_DEV void store8(T* __restrict__ p, int64_t i, int64_t lo, int64_t hi, const float (&v)[8]) {
  if (kVec && i >= lo && i + 8 <= hi) {
    if constexpr (sizeof(T) == 2) {
      uint4 q;
      __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) b[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      *reinterpret_cast<uint4*>(p + i) = q;
    } else {
      *reinterpret_cast<float4*>(p + i) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(p + i + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i + k >= lo && i + k < hi) IO<T>::st(p + i + k, v[k]);
  }
}

// Load 4 consecutive elements (same contract as load8 with 4).
template <typename T, bool kVec>
PM_DEV void load4(const T* __restrict__ p, int64_t i, int64_t n, float (&v)[4]) {
  if (kVec && i >= 0 && i + 4 <= n) {
    if constexpr (sizeof(T) == 2) {
      uint2 q = __ldg(reinterpret_cast<const uint2*>(p + i));
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
      float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
      v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
    } else {
      float4 a = __ldg(reinterpret_cast<const float4*>(p + i));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      v[k] = (i + k >= 0 && i + k < n) ? IO<T>::ld(p + i + k) : 0.f;
  }
}

template <typename T, bool kVec>
PM_DEV void store4(T* __restrict__ p, int64_t i, int64_t lo, int64_t hi, const float (&v)[4]) {
  if (kVec && i >= lo && i + 4 <= hi) {
    if constexpr (sizeof(T) == 2) {
      uint2 q;
      __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&q);
      b[0] = __floats2bfloat162_rn(v[0], v[1]);
      b[1] = __floats2bfloat162_rn(v[2], v[3]);
      *reinterpret_cast<uint2*>(p + i) = q;
    } else {
      *reinterpret_cast<float4*>(p + i) = make_float4(v[0], v[1], v[2], v[3]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k >= lo && i + k < hi) IO<T>::st(p + i + k, v[k]);
  }
}

template <typename T, bool kVec>
PM_DEV void store2(T* __restrict__ p, int64_t i, int64_t lo, int64_t hi, const float (&v)[2]) {
  if (kVec && i >= lo && i + 2 <= hi) {
    if constexpr (sizeof(T) == 2) {
      *reinterpret_cast<__nv_bfloat162*>(p + i) = __floats2bfloat162_rn(v[0], v[1]);
    } else {
      *reinterpret_cast<float2*>(p + i) = make_float2(v[0], v[1]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (i + k >= lo && i + k < hi) IO<T>::st(p + i + k, v[k]);
  }
}

// 8 consecutive elements from 16-byte aligned shared memory, as fp32
template <typename T>
PM_DEV void smem_load8(const T* p, float (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(b[k]);
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <typename T, bool kVec>
struct Raw8 {  // 8 consecutive I/O elements held raw in registers (prefetch)
  float v[8];
  PM_DEV void load(const T* p, int64_t i, int64_t n) { load8<T, kVec>(p, i, n, v); }
  PM_DEV void unpack(float (&o)[8]) const {
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = v[k];
  }
};
template <>
struct Raw8<__nv_bfloat16, true> {
  // kVec guarantees L % 8 == 0, so an 8-aligned vector is either fully inside
  // the row or fully outside it (then it reads as zeros).
  uint4 q;
  PM_DEV void load(const __nv_bfloat16* p, int64_t i, int64_t n) {
    q = (i >= 0 && i + 8 <= n) ? __ldg(reinterpret_cast<const uint4*>(p + i)) : make_uint4(0, 0, 0, 0);
  }
  PM_DEV void unpack(float (&o)[8]) const {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 x = __bfloat1622float2(b[k]);
      o[2 * k] = x.x;
      o[2 * k + 1] = x.y;
    }
  }
};

// ----------------------------------------------------- TMA + mbarrier ----
// Bulk tensor copies (cp.async.bulk.tensor, SASS UTMALDG) complete on a
// shared-memory mbarrier that counts the transferred bytes.
PM_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
PM_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
PM_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
PM_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
template <int D>
PM_DEV void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2 = 0,
                     int c3 = 0) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if constexpr (D == 2) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
  } else if constexpr (D == 3) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0),
        "r"(c1), "r"(c2)
        : "memory");
  } else {
    static_assert(D == 4, "2, 3 or 4 dimensions");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
  }
}

// ------------------------------------------------------------ cp.async ----
// 16-byte global->shared async copy (LDGSTS); src_bytes < 16 zero-fills.
PM_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
PM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
PM_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
template <int N>
PM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- TMEM ----
// Tensor memory used as per-thread scratch: a warp's 32 threads own the 32
// TMEM lanes of quarter (warp % 4); a thread's values sit in consecutive
// 32-bit columns of its lane.  (sm_100a tcgen05; allocation in powers of 2
// >= 32 columns by one warp, which also deallocates.)
PM_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {  // whole warp
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(s), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
PM_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp (the allocating one)
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols)
               : "memory");
}
PM_DEV void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
PM_DEV void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
PM_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
PM_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

template <int M>  // store M (2, 4, 8 or 16) fp32 values to columns [c, c+M) of my lane
PM_DEV void tmem_st(uint32_t taddr, const float* v) {
  if constexpr (M == 16) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
  } else if constexpr (M == 8) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
        : "memory");
  } else if constexpr (M == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3]))
                 : "memory");
  } else {
    static_assert(M == 2, "M in {2, 4, 8}");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1]))
                 : "memory");
  }
}

template <int M>  // load M (2..32, power of 2) values from columns [c, c+M) of my lane, then wait
PM_DEV void tmem_ld(uint32_t taddr, float* v) {
  static_assert(M == 2 || M == 4 || M == 8 || M == 16 || M == 32, "M in {2, 4, 8, 16, 32}");
  uint32_t r[M];
  if constexpr (M == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
  } else if constexpr (M == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
  } else if constexpr (M == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
  } else if constexpr (M == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr)
                 : "memory");
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(taddr)
                 : "memory");
  }
  tmem_wait_ld();
#pragma unroll
  for (int k = 0; k < M; ++k) {
    asm volatile("" : "+r"(r[k]));  // keep every use of the value after the wait
    v[k] = __uint_as_float(r[k]);
  }
}

// --------------------------------------------------- segment splitting ----
// A packed row is a concatenation of independent sequences (no
// sequence spans rows; the reset at heads cuts every carry).  So a row can
// be split at heads into independent time segments without any carry
// fix-up.  Segment k of nseg covers [b_k, b_{k+1}) where b_0 = 0,
// b_nseg = L and b_k = first head at or after k*ceil(L/nseg).  Boundaries
// are monotone; a segment may be empty.  All threads of the block call this.
PM_DEV int first_head_from(const int32_t* __restrict__ pos_row, int L, int t0, int* s_red) {
  // block-cooperative search for min{t >= t0 : pos[t] == 0} (or L)
  if (t0 >= L) return L;
  if (t0 <= 0) return 0;
  int found = L;
  for (int base = t0; base < L; base += blockDim.x) {
    int t = base + threadIdx.x;
    int hit = (t < L && __ldg(pos_row + t) == 0) ? t : L;
    // block min
    for (int o = 16; o > 0; o >>= 1) hit = min(hit, __shfl_xor_sync(0xffffffffu, hit, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = hit;
    __syncthreads();
    int m = L;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = min(m, s_red[w]);
    if (m < L) { found = m; break; }
  }
  __syncthreads();
  return found;
}

PM_DEV void segment_bounds(const int32_t* __restrict__ pos_row, int L, int k, int nseg,
                           int* s_red, int& s0, int& s1) {
  const int seg = (L + nseg - 1) / nseg;
  s0 = (k == 0) ? 0 : first_head_from(pos_row, L, k * seg, s_red);
  s1 = (k == nseg - 1) ? L : first_head_from(pos_row, L, (k + 1) * seg, s_red);
}

}  // namespace pm

// ------------------------------------- cross-kernel / cross-CTA sync ----
// Programmatic dependent launch: the next kernel in the stream (launched with
// cudaLaunchAttributeProgrammaticStreamSerialization) may start once every
// CTA of this one has executed this (its CTAs then take SM slots as this
// kernel's CTAs exit).
PM_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
PM_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PM_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// generic-proxy writes (another CTA's st.global) before async-proxy reads (TMA)
PM_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// SM count of the current device (host; 148 if the query fails)
inline int sm_count() {
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();  // clear: no device is not a launch error
    nsm = 148;
  }
  return nsm;
}

// host-side error helper
#define PM_LAUNCH_CHECK()                                     \
  do {                                                        \
    if (cudaGetLastError() != cudaSuccess) return PM_ERR_CUDA; \
  } while (0)
