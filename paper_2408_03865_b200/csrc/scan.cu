// scan.cu -- C ABI of ScanOp_pack (include/pm.h): argument validation,
// workspace / states layout, dispatch to the kernels in scan_fwd.cu and
// scan_bwd.cu.
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "scan_impl.cuh"

namespace {

using namespace pm;

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link
// against libcuda); resolved once.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// A tiled, unswizzled map over a dense tensor; dims innermost first, strides
// in bytes for dims 1..rank-1.  Out-of-range box elements read as zero.
bool encode_map(CUtensorMap* m, CUtensorMapDataType type, int rank, const void* base,
                const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
  const auto enc = tensor_map_encoder();
  if (enc == nullptr || base == nullptr) return false;
  const cuuint32_t ones[4] = {1, 1, 1, 1};
  return enc(m, type, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, ones,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA descriptors of the backward's per-chunk inputs (see ScanBwdArgs).
bool encode_bwd_maps(ScanBwdArgs& a, int N, pm_dtype io, int W) {
  const CUtensorMapDataType ty = io == PM_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const cuuint64_t isz = io == PM_F32 ? 4 : 2, L = a.L, Dn = a.Dn, R = a.R;
  const cuuint64_t dtok[3] = {L, Dn, R}, stok[2] = {L * isz, L * Dn * isz};
  const cuuint32_t btok[3] = {kChunk, (cuuint32_t)W, 1};
  const cuuint64_t dbc[3] = {L, (cuuint64_t)N, R}, sbc[2] = {L * isz, L * N * isz};
  const cuuint32_t bbc[3] = {kChunk, (cuuint32_t)N, 1};
  const cuuint64_t dpos[2] = {L, R}, spos[1] = {L * 4};
  const cuuint32_t bpos[2] = {kChunk, 1};
  const cuuint64_t nch = a.nchunk;
  const cuuint64_t dst[4] = {Dn, (cuuint64_t)N, nch, R},
                   sst[3] = {Dn * 4, Dn * N * 4, Dn * N * nch * 4};
  const cuuint32_t bst[4] = {(cuuint32_t)W, (cuuint32_t)N, 1, 1};
  bool ok = encode_map(&a.tm_u, ty, 3, a.u, dtok, stok, btok) &&
            encode_map(&a.tm_dt, ty, 3, a.dt, dtok, stok, btok) &&
            encode_map(&a.tm_dy, ty, 3, a.dy, dtok, stok, btok) &&
            encode_map(&a.tm_B, ty, 3, a.B, dbc, sbc, bbc) &&
            encode_map(&a.tm_C, ty, 3, a.C, dbc, sbc, bbc) &&
            encode_map(&a.tm_pos, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, a.pos, dpos, spos, bpos) &&
            encode_map(&a.tm_st, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.states, dst, sst, bst);
  if (ok && a.z != nullptr) ok = encode_map(&a.tm_z, ty, 3, a.z, dtok, stok, btok);
  return ok;
}

// bwd workspace = dB/dC partials | param partials | counters of the time
// split | its part lists (2 x R*nslot int4) | part summaries | (recomputed
// states)
size_t ws_bc_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return up256((size_t)n_dblk_bwd(Dn) * R * L * 2 * N * sizeof(float));
}
size_t ws_par_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return up256((size_t)R * n_slots(R, L, Dn) * (N + 2) * Dn * sizeof(float));
}
size_t ws_tsplit_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N) {
  return n_parts(R, L, Dn) > 1 ? 2 * list_bytes(R * n_slots(R, L, Dn)) + psum_bytes(R, Dn, L, N) : 0;
}
size_t bwd_ws_bytes(int64_t R, int64_t Dn, int64_t L, int32_t N, bool recompute) {
  return ws_bc_bytes(R, Dn, L, N) + ws_par_bytes(R, Dn, L, N) + 256 + ws_tsplit_bytes(R, Dn, L, N) +
         (recompute ? up256(state_bytes(R, Dn, L, N)) : 0);
}

// persistent schedule of a forward whose states buffer is `states`
void set_schedule(ScanFwdArgs& a, float* states, int64_t R, int64_t Dn, int64_t L, int32_t N) {
  Sched sc = sched_of(states, R, Dn, L, N);
  a.items = sc.sorted;
  a.counter = sc.counters;
  a.done = sc.done;
  a.n_items = (int)(R * n_seg(L));
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

pm_status pm_selective_scan_fwd_ex(const void* u, const void* dt, const float* A,
                                   const void* B, const void* C, const float* Dskip,
                                   const float* dt_bias, int32_t dt_softplus, int32_t zoh,
                                   const int32_t* pos, const void* z, const float* h0, void* out,
                                   float* states,
                                   float* h_last, float* decay, int64_t R, int64_t Dn, int64_t L,
                                   int32_t N,
                                   pm_dtype io, pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!u || !dt || !A || !B || !C || !pos || (!out && !states && !h_last && !decay))
    return PM_ERR_INVALID_ARG;
  for (const void* p : {u, dt, B, C, z, (const void*)out})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)A, (const void*)Dskip, (const void*)dt_bias, (const void*)pos,
                        (const void*)h0, (const void*)h_last, (const void*)decay})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  if (!aligned16(states)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && aligned16(u) && aligned16(dt) && aligned16(B) &&
                   aligned16(C) && aligned16(out) && aligned16(z);
  ScanFwdArgs a{u, dt, A, B, C, Dskip, dt_bias, pos, out, states, nullptr, nullptr, nullptr, 0,
                (int)R, (int)Dn, (int)L, n_seg(L), n_chunks(L), dt_softplus ? 1 : 0,
                z, h0, h_last, decay, zoh ? 1 : 0};
  if (states != nullptr)  // persistent longest-first schedule lives in the states buffer
    set_schedule(a, states, R, Dn, L, N);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return run_scan_fwd(a, (int)N, vec, io, s);
}

pm_status pm_selective_scan_fwd(const void* u, const void* dt, const float* A, const void* B,
                                const void* C, const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos, void* y, float* states,
                                int64_t R, int64_t Dn, int64_t L, int32_t N, pm_dtype io,
                                pm_stream_t stream) {
  if (!y && !states) return PM_ERR_INVALID_ARG;
  return pm_selective_scan_fwd_ex(u, dt, A, B, C, Dskip, dt_bias, dt_softplus, 0, pos, nullptr,
                                  nullptr, y, states, nullptr, nullptr, R, Dn, L, N, io, stream);
}

}  // extern "C"

namespace {
// The backward.  pdl: the caller (this library) has enqueued the forward that
// fills `states` directly before this call on the same stream, so the
// backward may launch programmatically behind it (pm.h).
pm_status bwd_impl(const void* u, const void* dt, const float* A, const void* B, const void* C,
                   const float* Dskip, const float* dt_bias, int32_t dt_softplus, int32_t zoh,
                   const int32_t* pos, const void* z, const float* h0, float* states,
                   const void* dout, const float* dh_last, void* du, void* ddt, float* dA,
                   float* dB, float* dC, float* dD, float* ddt_bias, void* dz, float* dh0,
                   void* workspace, size_t ws_bytes, int64_t R, int64_t Dn, int64_t L, int32_t N,
                   pm_dtype io, pm_stream_t stream, bool pdl) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (!u || !dt || !A || !B || !C || !pos || !dout || !du || !ddt || !dA || !dB || !dC ||
      (z != nullptr) != (dz != nullptr))
    return PM_ERR_INVALID_ARG;
  const bool recompute = states == nullptr;
  if (!workspace || ws_bytes < bwd_ws_bytes(R, Dn, L, N, recompute)) return PM_ERR_WORKSPACE;
  if (!aligned16(workspace) || !aligned16(states)) return PM_ERR_ALIGN;
  for (const void* p : {u, dt, B, C, z, dout, (const void*)du, (const void*)ddt, (const void*)dz})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)A, (const void*)Dskip, (const void*)dt_bias, (const void*)pos,
                        (const void*)dA, (const void*)dB, (const void*)dC, (const void*)dD,
                        (const void*)ddt_bias, (const void*)h0, (const void*)dh_last,
                        (const void*)dh0})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  const int isz = io == PM_F32 ? 4 : 2;
  const bool vec = (L * isz) % 16 == 0 && Dn % 4 == 0 && aligned16(u) && aligned16(dt) &&
                   aligned16(B) && aligned16(C) && aligned16(dout) && aligned16(du) &&
                   aligned16(ddt) && aligned16(z) && aligned16(dz) && aligned16(pos);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  float* ws_bc = reinterpret_cast<float*>(w);
  w += ws_bc_bytes(R, Dn, L, N);
  float* ws_par = reinterpret_cast<float*>(w);
  w += ws_par_bytes(R, Dn, L, N);
  int* counter = reinterpret_cast<int*>(w);
  w += 256;
  const int nparts = n_parts(R, L, Dn), nslot = n_slots(R, L, Dn);
  int4* part_lists = nparts > 1 ? reinterpret_cast<int4*>(w) : nullptr;
  float* psum_b = nparts > 1 ? reinterpret_cast<float*>(w + 2 * list_bytes(R * nslot)) : nullptr;
  w += ws_tsplit_bytes(R, Dn, L, N);
  const float* stp = states;
  if (recompute) {
    float* st_ws = reinterpret_cast<float*>(w);
    ScanFwdArgs fa{u, dt, A, B, C, Dskip, dt_bias, pos, nullptr, st_ws, nullptr, nullptr, nullptr, 0,
                   (int)R, (int)Dn, (int)L, n_seg(L), n_chunks(L), dt_softplus ? 1 : 0,
                   nullptr, h0, nullptr, nullptr, zoh ? 1 : 0};
    set_schedule(fa, st_ws, R, Dn, L, N);
    const bool fvec = (L * isz) % 16 == 0 && aligned16(u) && aligned16(dt) && aligned16(B) &&
                      aligned16(C);
    pm_status fs = run_scan_fwd(fa, (int)N, fvec, io, s);
    if (fs != PM_OK) return fs;
    stp = st_ws;
    pdl = true;  // the library's own forward is the preceding launch
  }
  // the length-sorted segment list, work counters and per-segment done
  // counts written by the forward pass (in the states buffer)
  const Sched sc = sched_of(const_cast<float*>(stp), R, Dn, L, N);
  ScanBwdArgs a{u, dt, A, B, C, Dskip, dt_bias, pos, stp, dout, du, ddt, ws_bc, ws_par,
                sc.sorted, sc.counters + 1, sc.done, (int)(R * n_seg(L)),
                (int)R, (int)Dn, (int)L, n_seg(L), n_chunks(L), dt_softplus ? 1 : 0,
                z, h0, dh_last, dz, dh0, zoh ? 1 : 0};
  a.pdl = pdl ? 1 : 0;
  if (nparts > 1) {
    // time split: own part list and work counters (in the workspace), no
    // wait on the forward's per-segment release counts, no programmatic
    // launch; the pre-pass writes every part's summary
    a.items = part_lists + (list_bytes(R * nslot) / 16);  // sorted list
    a.counter = counter;
    a.done = nullptr;
    a.pdl = 0;
    a.nseg = nslot;
    a.n_items = (int)(R * nslot);
    a.nparts = nparts;
    a.psum = psum_b;
    const bool pvec = (L * isz) % 16 == 0 && aligned16(dt) && aligned16(C) && aligned16(z) &&
                      aligned16(dout);
    const pm_status ps = run_part_bwd_pre(a, part_lists, const_cast<int4*>(a.items), counter,
                                          (int)N, pvec, io, s);
    if (ps != PM_OK) return ps;
  }
  // TMA for the per-chunk inputs when the vector path applies (row strides
  // are then multiples of 16 bytes); cp.async otherwise.  PM_NO_TMA=1 forces
  // cp.async (A/B measurements).
  // The wide backward (scan_bwd2.cu, two channels per thread) serves N = 16
  // on the TMA path without the gate or ZOH; PM_BWD_WIDE=0 forces the
  // one-channel-per-thread kernel (A/B).
  const char* we = getenv("PM_BWD_WIDE");
  const bool tma = vec && Dn % 4 == 0 && getenv("PM_NO_TMA") == nullptr;
  a.wide = tma && N == 16 && z == nullptr && !zoh && a.items != nullptr &&
           !(we != nullptr && atoi(we) == 0) ? 1 : 0;
  a.use_tma = tma && encode_bwd_maps(a, (int)N, io, a.wide ? kWideCh : kBwdCh) ? 1 : 0;
  if (!a.use_tma) a.wide = 0;
  return run_scan_bwd(a, (int)N, vec, io, dA, dB, dC, dD, ddt_bias, s);
}

struct Span {
  const void* p;
  size_t n;
};
bool overlap(Span a, Span b) {
  if (a.p == nullptr || b.p == nullptr || a.n == 0 || b.n == 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a.p), b0 = reinterpret_cast<uintptr_t>(b.p);
  return a0 < b0 + b.n && b0 < a0 + a.n;
}
}  // namespace

extern "C" {

pm_status pm_selective_scan_bwd_ex(const void* u, const void* dt, const float* A, const void* B,
                                   const void* C, const float* Dskip, const float* dt_bias,
                                   int32_t dt_softplus, int32_t zoh, const int32_t* pos,
                                   const void* z,
                                   const float* h0, float* states, const void* dout,
                                   const float* dh_last, void* du, void* ddt, float* dA,
                                   float* dB, float* dC, float* dD, float* ddt_bias, void* dz,
                                   float* dh0, void* workspace, size_t ws_bytes, int64_t R,
                                   int64_t Dn, int64_t L, int32_t N, pm_dtype io,
                                   pm_stream_t stream) {
  return bwd_impl(u, dt, A, B, C, Dskip, dt_bias, dt_softplus, zoh, pos, z, h0, states, dout,
                  dh_last, du, ddt, dA, dB, dC, dD, ddt_bias, dz, dh0, workspace, ws_bytes, R, Dn,
                  L, N, io, stream, false);
}

pm_status pm_selective_scan_fwd_bwd(const void* u, const void* dt, const float* A, const void* B,
                                    const void* C, const float* Dskip, const float* dt_bias,
                                    int32_t dt_softplus, int32_t zoh, const int32_t* pos,
                                    const void* z, const float* h0, void* out, float* states,
                                    float* h_last, float* decay, const void* dout,
                                    const float* dh_last, void* du, void* ddt, float* dA,
                                    float* dB, float* dC, float* dD, float* ddt_bias, void* dz,
                                    float* dh0, void* workspace, size_t ws_bytes, int64_t R,
                                    int64_t Dn, int64_t L, int32_t N, pm_dtype io,
                                    pm_stream_t stream) {
  pm_status st = check_common(R, Dn, L, N, io);
  if (st != PM_OK) return st;
  if (states == nullptr) return PM_ERR_INVALID_ARG;
  // The backward may start before the forward has finished: none of its
  // outputs may overlap a forward output or an input, and no forward output
  // may be an input of the backward.
  const size_t isz = io == PM_F32 ? 4 : 2;
  const size_t tok = (size_t)R * Dn * L * isz, bc = (size_t)R * N * L, rdn = (size_t)R * Dn * N * 4;
  const Span fwd_out[] = {{out, tok}, {h_last, rdn}, {decay, rdn},
                          {states, state_bytes(R, Dn, L, N)}};
  const Span bwd_out[] = {{du, tok}, {ddt, tok}, {dA, (size_t)Dn * N * 4}, {dB, bc * 4},
                          {dC, bc * 4}, {dD, (size_t)Dn * 4}, {ddt_bias, (size_t)Dn * 4},
                          {dz, tok}, {dh0, rdn}, {workspace, ws_bytes}};
  const Span inputs[] = {{u, tok}, {dt, tok}, {A, (size_t)Dn * N * 4}, {B, bc * isz},
                         {C, bc * isz}, {Dskip, (size_t)Dn * 4}, {dt_bias, (size_t)Dn * 4},
                         {pos, (size_t)R * L * 4}, {z, tok}, {h0, rdn}, {dout, tok},
                         {dh_last, rdn}};
  for (const Span& o : bwd_out) {
    for (const Span& f : fwd_out)
      if (overlap(o, f)) return PM_ERR_INVALID_ARG;
    for (const Span& i : inputs)
      if (overlap(o, i)) return PM_ERR_INVALID_ARG;
  }
  for (const Span& f : fwd_out)
    for (const Span& i : inputs)
      if (overlap(f, i)) return PM_ERR_INVALID_ARG;
  // validate the backward's arguments before the forward is enqueued
  if (!dout || !du || !ddt || !dA || !dB || !dC || (z != nullptr) != (dz != nullptr))
    return PM_ERR_INVALID_ARG;
  if (!workspace || ws_bytes < bwd_ws_bytes(R, Dn, L, N, false)) return PM_ERR_WORKSPACE;
  if (!aligned16(workspace)) return PM_ERR_ALIGN;
  for (const void* p : {dout, (const void*)du, (const void*)ddt, (const void*)dz})
    if (!elem_aligned(p, io)) return PM_ERR_ALIGN;
  for (const void* p : {(const void*)dA, (const void*)dB, (const void*)dC, (const void*)dD,
                        (const void*)ddt_bias, (const void*)dh_last, (const void*)dh0})
    if (p && (reinterpret_cast<uintptr_t>(p) & 3u)) return PM_ERR_ALIGN;
  st = pm_selective_scan_fwd_ex(u, dt, A, B, C, Dskip, dt_bias, dt_softplus, zoh, pos, z, h0, out,
                                states, h_last, decay, R, Dn, L, N, io, stream);
  if (st != PM_OK) return st;
  return bwd_impl(u, dt, A, B, C, Dskip, dt_bias, dt_softplus, zoh, pos, z, h0, states, dout,
                  dh_last, du, ddt, dA, dB, dC, dD, ddt_bias, dz, dh0, workspace, ws_bytes, R, Dn,
                  L, N, io, stream, true);
}

pm_status pm_selective_scan_bwd(const void* u, const void* dt, const float* A, const void* B,
                                const void* C, const float* Dskip, const float* dt_bias,
                                int32_t dt_softplus, const int32_t* pos, float* states,
                                const void* dy, void* du, void* ddt, float* dA, float* dB,
                                float* dC, float* dD, float* ddt_bias, void* workspace,
                                size_t ws_bytes, int64_t R, int64_t Dn, int64_t L, int32_t N,
                                pm_dtype io, pm_stream_t stream) {
  return pm_selective_scan_bwd_ex(u, dt, A, B, C, Dskip, dt_bias, dt_softplus, 0, pos, nullptr,
                                  nullptr, states, dy, nullptr, du, ddt, dA, dB, dC, dD, ddt_bias,
                                  nullptr, nullptr, workspace, ws_bytes, R, Dn, L, N, io, stream);
}

}  // extern "C"
