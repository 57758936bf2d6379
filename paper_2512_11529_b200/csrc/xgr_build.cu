// xgr_mask_build: device construction of the legal-item trie.
//
// PAPER.md L361 (section 6.1): "xBeam generates an item mask based on the pre-built valid item
// vocabulary"; L371: "the mask is stored in a dense format and pre-generated during model
// loading ... during the final decode step, each beam only contains few candidate tokens ...
// xBeam stores the relevant positions in a sparse format". Here the dense/sparse choice is made
// per node (reading R17): a node with >= V/16 children keeps a V-bit bitmap (plus a
// rank directory for O(1) child ids); every node's children are also a contiguous, sorted run of
// next-level labels, which is the sparse list.
//
// Pipeline (all on device, once per catalogue): pack each ND-tuple into a uint64 key (w bits per
// token, most significant first) -> radix sort -> unique -> for each level d, segment starts of
// the d-token prefixes give node ids (lexicographic), labels, first_child offsets; child counts
// give the dense set; bitmaps are filled from the labels.
#include <cub/cub.cuh>

#include <string>
#include <vector>

#include "xgr_internal.cuh"

namespace xgr {

void trie_free(TrieHost& t) {
  for (auto& L : t.lv) {
    t.al.put(L.first_child);
    t.al.put(L.label);
    t.al.put(L.dense_slot);
    t.al.put(L.bitmap);
    t.al.put(L.rankdir);
    L = LevelHost();
  }
  t.bytes = 0;
}

TrieDev trie_dev(const TrieHost& t) {
  TrieDev d;
  memset(&d, 0, sizeof(d));
  d.V = t.V;
  d.nd = t.nd;
  d.W = t.W;
  d.R = t.R;
  for (int i = 0; i <= t.nd; ++i) {
    d.lv[i].first_child = t.lv[i].first_child;
    d.lv[i].label = t.lv[i].label;
    d.lv[i].dense_slot = t.lv[i].dense_slot;
    d.lv[i].bitmap = t.lv[i].bitmap;
    d.lv[i].rankdir = t.lv[i].rankdir;
    d.lv[i].n_nodes = t.lv[i].n_nodes;
    d.lv[i].n_dense = t.lv[i].n_dense;
    d.lv[i].max_children = t.lv[i].max_children;
  }
  return d;
}

namespace {

__global__ void k_pack(const int32_t* __restrict__ items, int64_t n, int nd, int w, int V,
                       uint64_t* __restrict__ keys, uint32_t* __restrict__ err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
  bool bad = false;
  for (int d = 0; d < nd; ++d) {
    int32_t t = items[i * nd + d];
    bad |= (t < 0) | (t >= V);
    k = (k << w) | (uint64_t)(uint32_t)(t & ((1 << w) - 1));
  }
  if (bad) atomicOr(err, 1u);
  keys[i] = k;
}

// starts[i] = 1 iff key i begins a new prefix of the level (shift = w * (nd - d))
__global__ void k_starts(const uint64_t* __restrict__ keys, int64_t n, int shift,
                         uint32_t* __restrict__ starts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  starts[i] = (i == 0) ? 1u : (uint32_t)((keys[i] >> shift) != (keys[i - 1] >> shift));
}

// At each start of a level-d node: its label, its parent (level d-1 node id), and, if it is the
// first child of that parent, the parent's first_child entry.
__global__ void k_level(const uint64_t* __restrict__ keys, int64_t n, int shift_d, int shift_p,
                        int w, const uint32_t* __restrict__ id_d, const uint32_t* __restrict__ id_p,
                        uint16_t* __restrict__ label, uint32_t* __restrict__ parent,
                        uint32_t* __restrict__ fc_p) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = keys[i];
  bool start_d = (i == 0) || ((k >> shift_d) != (keys[i - 1] >> shift_d));
  if (!start_d) return;
  uint32_t j = id_d[i] - 1u;  // inclusive scan of starts -> id + 1
  uint32_t p = id_p ? id_p[i] - 1u : 0u;
  label[j] = (uint16_t)((k >> shift_d) & ((1ull << w) - 1ull));
  parent[j] = p;
  bool start_p = (i == 0) || (shift_p < 64 && (k >> shift_p) != (keys[i - 1] >> shift_p));
  if (shift_p >= 64) start_p = (i == 0);
  if (start_p) fc_p[p] = j;
}

__global__ void k_counts(const uint32_t* __restrict__ fc, int64_t n_nodes, uint32_t thr,
                         uint32_t* __restrict__ dense_flag, int32_t* __restrict__ max_children) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  uint32_t c = fc[i + 1] - fc[i];
  dense_flag[i] = c >= thr ? 1u : 0u;
  atomicMax(max_children, (int32_t)c);
}

__global__ void k_slots(const uint32_t* __restrict__ dense_flag, const uint32_t* __restrict__ excl,
                        int64_t n_nodes, int32_t* __restrict__ slot) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  slot[i] = dense_flag[i] ? (int32_t)excl[i] : -1;
}

__global__ void k_fill_bitmap(const uint16_t* __restrict__ label, const uint32_t* __restrict__ parent,
                              int64_t n_child, const int32_t* __restrict__ pslot, int W,
                              uint32_t* __restrict__ bitmap) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_child) return;
  int32_t s = pslot[parent[j]];
  if (s < 0) return;
  uint32_t v = label[j];
  atomicOr(&bitmap[(size_t)s * W + (v >> 5)], 1u << (v & 31));
}

__global__ void k_rankdir(const uint32_t* __restrict__ bitmap, int64_t n_dense, int W, int R,
                          uint32_t* __restrict__ rankdir) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_dense) return;
  const uint32_t* bm = bitmap + (size_t)s * W;
  uint32_t acc = 0;
  for (int r = 0; r < R; ++r) {
    rankdir[(size_t)s * R + r] = acc;
    for (int q = r * 8; q < min(W, r * 8 + 8); ++q) acc += __popc(bm[q]);
  }
}

inline unsigned grid_for(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

#define BCK(x)                                                                      \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      err = std::string("mask_build: ") + #x + ": " + cudaGetErrorString(e_);       \
      st = (e_ == cudaErrorMemoryAllocation) ? XGR_ERR_OOM : XGR_ERR_CUDA;          \
      goto fail;                                                                    \
    }                                                                               \
  } while (0)

// Builds `out` (freed by the caller with trie_free on any failure). Synchronous on `s`.
xgr_status trie_build(TrieHost& out, const int32_t* h_items, int64_t n, int V, int nd,
                      cudaStream_t s, std::string& err) {
  xgr_status st = XGR_OK;
  int w = 1;
  while ((1 << w) < V) ++w;
  out.V = V;
  out.nd = nd;
  out.w = w;
  out.W = (V + 31) / 32;
  out.R = (V + 255) / 256;

  int32_t* d_items = nullptr;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *starts = nullptr, *id_p = nullptr, *id_d = nullptr, *parent = nullptr, *tmp = nullptr,
           *d_err = nullptr, *d_num = nullptr;
  int32_t* d_maxc = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  int64_t N = 0;
  uint32_t h_err = 0;
  int64_t prev_nodes = 1;

  const int64_t chunk = 1 << 24;
  BCK(out.al.get(&k0, n * sizeof(uint64_t)));
  BCK(out.al.get(&k1, n * sizeof(uint64_t)));
  BCK(out.al.get(&d_items, std::min(n, chunk) * nd * sizeof(int32_t)));
  BCK(out.al.get(&d_err, 2 * sizeof(uint32_t)));
  BCK(out.al.get(&d_maxc, sizeof(int32_t)));
  d_num = d_err + 1;
  BCK(cudaMemsetAsync(d_err, 0, 2 * sizeof(uint32_t), s));
  for (int64_t c0 = 0; c0 < n; c0 += chunk) {
    int64_t m = std::min(chunk, n - c0);
    BCK(cudaMemcpyAsync(d_items, h_items + c0 * nd, m * nd * sizeof(int32_t),
                        cudaMemcpyHostToDevice, s));
    k_pack<<<grid_for(m), 256, 0, s>>>(d_items, m, nd, w, V, k0 + c0, d_err);
    BCK(cudaGetLastError());
  }
  BCK(cudaMemcpyAsync(&h_err, d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  BCK(cudaStreamSynchronize(s));
  out.al.put(d_items);
  d_items = nullptr;
  if (h_err) {
    err = "mask_build: a token is < 0 or >= V";
    st = XGR_ERR_TOKEN_RANGE;
    goto fail;
  }

  // sort + unique
  {
    size_t b1 = 0, b2 = 0, b3 = 0;
    cub::DoubleBuffer<uint64_t> db(k0, k1);
    BCK(cub::DeviceRadixSort::SortKeys(nullptr, b1, db, (int64_t)n, 0, w * nd, s));
    BCK(cub::DeviceSelect::Unique(nullptr, b2, k1, k0, d_num, (int64_t)n, s));
    BCK(cub::DeviceScan::InclusiveSum(nullptr, b3, (uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, s));
    temp_bytes = std::max(b1, std::max(b2, b3));
    BCK(out.al.get(&temp, temp_bytes));
    BCK(cub::DeviceRadixSort::SortKeys(temp, b1, db, (int64_t)n, 0, w * nd, s));
    uint64_t* sorted = db.Current();
    uint64_t* other = db.Alternate();
    BCK(cub::DeviceSelect::Unique(temp, b2, sorted, other, d_num, (int64_t)n, s));
    k0 = other;   // unique keys live here from now on
    k1 = sorted;
    uint32_t hn = 0;
    BCK(cudaMemcpyAsync(&hn, d_num, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    BCK(cudaStreamSynchronize(s));
    N = hn;
  }
  out.al.put(k1);
  k1 = nullptr;
  out.n_items = N;
  out.lv[0].n_nodes = 1;

  BCK(out.al.get(&starts, N * sizeof(uint32_t)));
  BCK(out.al.get(&id_d, N * sizeof(uint32_t)));
  BCK(out.al.get(&id_p, N * sizeof(uint32_t)));
  for (int d = 1; d <= nd; ++d) {
    int shift_d = w * (nd - d);
    int shift_p = (d == 1) ? 64 : w * (nd - d + 1);
    k_starts<<<grid_for(N), 256, 0, s>>>(k0, N, shift_d, starts);
    BCK(cudaGetLastError());
    size_t b3 = temp_bytes;
    BCK(cub::DeviceScan::InclusiveSum(temp, b3, starts, id_d, (int64_t)N, s));
    uint32_t last = 0;
    BCK(cudaMemcpyAsync(&last, id_d + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    BCK(cudaStreamSynchronize(s));
    int64_t nodes = last;
    LevelHost& P = out.lv[d - 1];
    LevelHost& C = out.lv[d];
    C.n_nodes = nodes;
    BCK(out.al.get(&C.label, nodes * sizeof(uint16_t)));
    BCK(out.al.get(&P.first_child, (prev_nodes + 1) * sizeof(uint32_t)));
    out.al.put(parent);
    parent = nullptr;
    BCK(out.al.get(&parent, nodes * sizeof(uint32_t)));
    {
      uint32_t nn = (uint32_t)nodes;
      BCK(cudaMemcpyAsync(P.first_child + prev_nodes, &nn, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    }
    k_level<<<grid_for(N), 256, 0, s>>>(k0, N, shift_d, shift_p, w, id_d, d == 1 ? nullptr : id_p,
                                        C.label, parent, P.first_child);
    BCK(cudaGetLastError());
    // parent level: child counts, dense set, slots
    {
      uint32_t thr = (uint32_t)std::max(1, V / 16);
      out.al.put(tmp);
      tmp = nullptr;
      BCK(out.al.get(&tmp, 2 * (prev_nodes + 1) * sizeof(uint32_t)));
      uint32_t* flag = tmp;
      uint32_t* excl = tmp + prev_nodes + 1;
      BCK(cudaMemsetAsync(d_maxc, 0, sizeof(int32_t), s));
      k_counts<<<grid_for(prev_nodes), 256, 0, s>>>(P.first_child, prev_nodes, thr, flag, d_maxc);
      BCK(cudaGetLastError());
      size_t b4 = 0;
      BCK(cub::DeviceScan::ExclusiveSum(nullptr, b4, flag, excl, (int64_t)prev_nodes + 1, s));
      if (b4 > temp_bytes) {
        out.al.put(temp);
        temp = nullptr;
        temp_bytes = b4;
        BCK(out.al.get(&temp, temp_bytes));
      }
      BCK(cudaMemsetAsync(flag + prev_nodes, 0, sizeof(uint32_t), s));
      b4 = temp_bytes;
      BCK(cub::DeviceScan::ExclusiveSum(temp, b4, flag, excl, (int64_t)prev_nodes + 1, s));
      uint32_t ndense = 0;
      int32_t maxc = 0;
      BCK(cudaMemcpyAsync(&ndense, excl + prev_nodes, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      BCK(cudaMemcpyAsync(&maxc, d_maxc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      BCK(cudaStreamSynchronize(s));
      P.n_dense = ndense;
      P.max_children = maxc;
      if (ndense > 0) {
        BCK(out.al.get(&P.dense_slot, prev_nodes * sizeof(int32_t)));
        k_slots<<<grid_for(prev_nodes), 256, 0, s>>>(flag, excl, prev_nodes, P.dense_slot);
        BCK(cudaGetLastError());
        BCK(out.al.get(&P.bitmap, (size_t)ndense * out.W * sizeof(uint32_t)));
        BCK(cudaMemsetAsync(P.bitmap, 0, (size_t)ndense * out.W * sizeof(uint32_t), s));
        BCK(out.al.get(&P.rankdir, (size_t)ndense * out.R * sizeof(uint32_t)));
        k_fill_bitmap<<<grid_for(nodes), 256, 0, s>>>(C.label, parent, nodes, P.dense_slot, out.W,
                                                      P.bitmap);
        BCK(cudaGetLastError());
        k_rankdir<<<grid_for(ndense, 128), 128, 0, s>>>(P.bitmap, ndense, out.W, out.R, P.rankdir);
        BCK(cudaGetLastError());
      }
    }
    std::swap(id_d, id_p);
    prev_nodes = nodes;
  }
  BCK(cudaStreamSynchronize(s));
  {
    int64_t bytes = 0;
    for (int d = 0; d <= nd; ++d) {
      const LevelHost& L = out.lv[d];
      if (L.first_child) bytes += (L.n_nodes + 1) * 4;
      if (L.label) bytes += L.n_nodes * 2;
      if (L.dense_slot) bytes += L.n_nodes * 4;
      bytes += L.n_dense * (int64_t)(out.W + out.R) * 4;
    }
    out.bytes = bytes;
  }

fail:
  out.al.put(d_items);
  out.al.put(k0);
  out.al.put(k1);
  out.al.put(starts);
  out.al.put(id_p);
  out.al.put(id_d);
  out.al.put(parent);
  out.al.put(tmp);
  out.al.put(d_err);
  out.al.put(d_maxc);
  out.al.put(temp);
  return st;
}

}  // namespace xgr
