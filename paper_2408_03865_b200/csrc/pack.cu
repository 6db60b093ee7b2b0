// pack.cu -- pm_plan_fifo / pm_plan_greedy (host) and pm_pack (device
// scatter) -- sec 3.1 P:120 and sec 5 P:273 of arXiv 2408.03865.
//
// The plan is a host decision (it only reads lengths).  The scatter is one
// kernel: each CTA copies one sequence's records into its slot range and
// writes position_indices 0..len-1; a second kernel zero-fills each row's
// padding tail (data = 0, pos = 0: reading Q8).  The per-sequence plan is
// passed as kernel parameters (<= 32 KiB per launch on sm_70+ with CUDA
// >= 12.1), so no device workspace and no host synchronisation are needed.
#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace pm {

constexpr int kPackBatch = 1000;

struct PackItem {
  int64_t src_tok;   // first token of the sequence in src
  int64_t dst_slot;  // row * pack_len + offset
  int64_t len;
};
struct PackBatchParams {
  PackItem item[kPackBatch];
  int n;
};
struct PadItem {
  int64_t slot;  // first padding slot
  int64_t len;   // number of padding slots
};
struct PadBatchParams {
  PadItem item[kPackBatch];
  int n;
};
static_assert(sizeof(PackBatchParams) < 32000, "kernel parameter limit");

__global__ void __launch_bounds__(256)
pack_scatter_kernel(const __grid_constant__ PackBatchParams p, const uint8_t* __restrict__ src,
                    uint8_t* __restrict__ dst, int32_t* __restrict__ pos, int64_t rec) {
  const PackItem it = p.item[blockIdx.x];
  const int64_t nbytes = it.len * rec;
  const uint8_t* s = src + it.src_tok * rec;
  uint8_t* d = dst + it.dst_slot * rec;
  const bool v16 = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15u) == 0;
  const bool v4 = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 3u) == 0;
  int64_t done = 0;
  if (v16) {
    const int64_t n16 = nbytes / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
      reinterpret_cast<uint4*>(d)[i] = __ldg(reinterpret_cast<const uint4*>(s) + i);
    done = n16 * 16;
  } else if (v4) {
    const int64_t n4 = nbytes / 4;
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(d)[i] = __ldg(reinterpret_cast<const uint32_t*>(s) + i);
    done = n4 * 4;
  }
  for (int64_t i = done + threadIdx.x; i < nbytes; i += blockDim.x) d[i] = s[i];
  for (int64_t i = threadIdx.x; i < it.len; i += blockDim.x) pos[it.dst_slot + i] = (int32_t)i;
}

__global__ void __launch_bounds__(256)
pack_pad_kernel(const __grid_constant__ PadBatchParams p, uint8_t* __restrict__ dst,
                int32_t* __restrict__ pos, int64_t rec) {
  const PadItem it = p.item[blockIdx.x];
  uint8_t* d = dst + it.slot * rec;
  for (int64_t i = threadIdx.x; i < it.len * rec; i += blockDim.x) d[i] = 0;
  for (int64_t i = threadIdx.x; i < it.len; i += blockDim.x) pos[it.slot + i] = 0;
}

}  // namespace pm

namespace {

pm_status check_lens(const int32_t* lens, int64_t n, int64_t cap) {
  if (!lens || n < 1 || cap < 1) return PM_ERR_INVALID_ARG;
  for (int64_t i = 0; i < n; ++i)
    if (lens[i] < 1 || lens[i] > cap) return PM_ERR_CAPACITY;
  return PM_OK;
}

// FIFO seal: open a new row exactly when the next sequence does not fit.
int64_t plan_fifo(const int32_t* lens, int64_t n, int64_t cap, int64_t* row, int64_t* off) {
  int64_t r = 0, used = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i > 0 && used + lens[i] > cap) {
      ++r;
      used = 0;
    }
    if (row) row[i] = r;
    if (off) off[i] = used;
    used += lens[i];
  }
  return r + 1;
}

// First-fit-decreasing ("local greedy ... sorts") with a
// max-segment-tree over row free space: O(n log n).
int64_t plan_greedy(const int32_t* lens, int64_t n, int64_t cap, int64_t* row, int64_t* off) {
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return lens[a] > lens[b]; });
  int64_t size = 1;
  while (size < n) size <<= 1;
  std::vector<int64_t> tree(2 * size, cap);  // free space of rows (all rows open)
  std::vector<int64_t> used(size, 0);
  int64_t rows = 0;
  for (int64_t s = 0; s < n; ++s) {
    const int64_t i = order[s], need = lens[i];
    int64_t node = 1;  // leftmost leaf with free >= need (always exists: row n-1 is empty)
    while (node < size) node = (tree[2 * node] >= need) ? 2 * node : 2 * node + 1;
    const int64_t r = node - size;
    if (row) row[i] = r;
    if (off) off[i] = used[r];
    used[r] += need;
    rows = std::max(rows, r + 1);
    tree[node] -= need;
    for (node >>= 1; node >= 1; node >>= 1) tree[node] = std::max(tree[2 * node], tree[2 * node + 1]);
  }
  return rows;
}

pm_status scatter(const int32_t* lens, int64_t n, int64_t cap, const int64_t* row, const int64_t* off,
                  int64_t n_rows, const void* src, int64_t rec, void* dst, int32_t* pos,
                  cudaStream_t s) {
  using namespace pm;
  PackBatchParams pb;
  int64_t tok = 0;
  pb.n = 0;
  std::vector<int64_t> used(n_rows, 0);
  for (int64_t i = 0; i < n; ++i) {
    pb.item[pb.n++] = PackItem{tok, row[i] * cap + off[i], lens[i]};
    tok += lens[i];
    used[row[i]] = std::max(used[row[i]], off[i] + lens[i]);
    if (pb.n == kPackBatch || i == n - 1) {
      pack_scatter_kernel<<<pb.n, 256, 0, s>>>(pb, static_cast<const uint8_t*>(src),
                                                static_cast<uint8_t*>(dst), pos, rec);
      PM_LAUNCH_CHECK();
      pb.n = 0;
    }
  }
  // padding: everything in a row that no sequence covers.  Plans from
  // plan_fifo/plan_greedy are left-packed, so it is the tail [used, cap).
  PadBatchParams pp;
  pp.n = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    if (used[r] < cap) pp.item[pp.n++] = PadItem{r * cap + used[r], cap - used[r]};
    if (pp.n == kPackBatch || (r == n_rows - 1 && pp.n > 0)) {
      pack_pad_kernel<<<pp.n, 256, 0, s>>>(pp, static_cast<uint8_t*>(dst), pos, rec);
      PM_LAUNCH_CHECK();
      pp.n = 0;
    }
  }
  return PM_OK;
}

// A caller plan must be left-packed per row (sequences tile [0, used)).
pm_status check_plan(const int32_t* lens, int64_t n, int64_t cap, const int64_t* row,
                     const int64_t* off, int64_t n_rows) {
  std::vector<std::pair<int64_t, int64_t>> seg;  // (slot, len)
  seg.reserve(n);
  for (int64_t i = 0; i < n; ++i) {
    if (row[i] < 0 || row[i] >= n_rows || off[i] < 0 || off[i] + lens[i] > cap) return PM_ERR_SHAPE;
    seg.emplace_back(row[i] * cap + off[i], lens[i]);
  }
  std::sort(seg.begin(), seg.end());
  int64_t cur_row = -1, next = 0;
  for (auto& s : seg) {
    const int64_t r = s.first / cap, o = s.first % cap;
    if (r != cur_row) {
      cur_row = r;
      next = 0;
    }
    if (o != next) return PM_ERR_SHAPE;  // gap or overlap
    next = o + s.second;
  }
  return PM_OK;
}

}  // namespace

extern "C" {

pm_status pm_plan_fifo(const int32_t* lens, int64_t n, int64_t cap, int64_t* row, int64_t* off,
                       int64_t* n_rows_out) {
  pm_status st = check_lens(lens, n, cap);
  if (st != PM_OK) return st;
  if (!n_rows_out) return PM_ERR_INVALID_ARG;
  *n_rows_out = plan_fifo(lens, n, cap, row, off);
  return PM_OK;
}

pm_status pm_plan_greedy(const int32_t* lens, int64_t n, int64_t cap, int64_t* row, int64_t* off,
                         int64_t* n_rows_out) {
  pm_status st = check_lens(lens, n, cap);
  if (st != PM_OK) return st;
  if (!n_rows_out) return PM_ERR_INVALID_ARG;
  *n_rows_out = plan_greedy(lens, n, cap, row, off);
  return PM_OK;
}

pm_status pm_pack(const int32_t* lens, int64_t n, int64_t cap, const void* src, int64_t rec,
                  void* dst, int32_t* pos, int64_t max_rows, int64_t* n_rows_out, int64_t* row_out,
                  int64_t* off_out, pm_stream_t stream) {
  pm_status st = check_lens(lens, n, cap);
  if (st != PM_OK) return st;
  if (!n_rows_out) return PM_ERR_INVALID_ARG;
  std::vector<int64_t> row(n), off(n);
  const int64_t nr = plan_fifo(lens, n, cap, row.data(), off.data());
  if (dst == nullptr && pos == nullptr) {  // query mode
    *n_rows_out = nr;
    if (row_out) std::copy(row.begin(), row.end(), row_out);
    if (off_out) std::copy(off.begin(), off.end(), off_out);
    return PM_OK;
  }
  if (!src || !dst || !pos || rec < 1) return PM_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(pos) & 3u) return PM_ERR_ALIGN;
  if (nr > max_rows) return PM_ERR_CAPACITY;
  st = scatter(lens, n, cap, row.data(), off.data(), nr, src, rec, dst, pos,
               reinterpret_cast<cudaStream_t>(stream));
  if (st != PM_OK) return st;
  *n_rows_out = nr;
  if (row_out) std::copy(row.begin(), row.end(), row_out);
  if (off_out) std::copy(off.begin(), off.end(), off_out);
  return PM_OK;
}

pm_status pm_pack_planned(const int32_t* lens, int64_t n, int64_t cap, const int64_t* row,
                          const int64_t* off, int64_t n_rows, const void* src, int64_t rec,
                          void* dst, int32_t* pos, pm_stream_t stream) {
  pm_status st = check_lens(lens, n, cap);
  if (st != PM_OK) return st;
  if (!row || !off || n_rows < 1 || !src || !dst || !pos || rec < 1) return PM_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(pos) & 3u) return PM_ERR_ALIGN;
  st = check_plan(lens, n, cap, row, off, n_rows);
  if (st != PM_OK) return st;
  return scatter(lens, n, cap, row, off, n_rows, src, rec, dst, pos,
                 reinterpret_cast<cudaStream_t>(stream));
}

const char* pm_status_string(pm_status s) {
  switch (s) {
    case PM_OK: return "ok";
    case PM_ERR_INVALID_ARG: return "invalid argument";
    case PM_ERR_CAPACITY: return "sequence exceeds pack capacity";
    case PM_ERR_SHAPE: return "shape mismatch";
    case PM_ERR_DTYPE: return "unsupported dtype";
    case PM_ERR_ALIGN: return "misaligned pointer";
    case PM_ERR_UNSUPPORTED: return "unsupported parameter (K or N)";
    case PM_ERR_CUDA: return "CUDA launch failure";
    case PM_ERR_WORKSPACE: return "workspace missing or too small";
  }
  return "unknown status";
}

const char* pm_version(void) { return "libpm 0.1 (sm_100a)"; }

}  // extern "C"
