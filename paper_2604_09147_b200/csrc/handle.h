// handle.h — the library-owned state behind hh_handle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace hh {

// Device buffer owned by a handle (freed in the destructor).
struct DBuf {
  void *p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  ~DBuf() { reset(); }
  void alloc(size_t n) {
    reset();
    if (n == 0) n = 16;
    HH_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

template <class T> void h2d(DBuf &b, const std::vector<T> &v, cudaStream_t s) {
  b.alloc(v.size() * sizeof(T));
  if (!v.empty()) HH_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

// Phase-1 work item: a contiguous, 16-B aligned window of one W arena plus the entries
// (column groups) it holds.  Phase-2 work: per leaf, a list of column chunks.
struct P1Item {
  int64_t src;        // byte offset in W[tag] (multiple of 16)
  uint32_t nbytes;    // multiple of 16
  uint16_t tag, pad;
  uint32_t e0, e1;    // entries [e0, e1)
};
struct P1Entry {
  uint32_t soff;      // byte offset of the first column inside the staged window
  uint32_t nrows;     // column length (rows of W_b, or a row piece)
  uint32_t ncols;
  uint32_t pad;
  int64_t x0;         // v index (tree position) of row 0
  int64_t out;        // z index of the first column (>= 0) or ~slot for a partial piece
};
struct P2Chunk {
  int64_t src;        // byte offset (multiple of 16) in U[tag] or D
  uint32_t nbytes;    // multiple of 16
  uint32_t lead;      // bytes skipped at the start of the window
  uint32_t ncols;
  uint16_t tag;       // 0..3, dense uses 0 (fp64) with arena flag
  uint16_t dense;     // 1 -> dense arena
  int64_t vbeg;       // v index of column 0's vector entry
};
struct P2Leaf {
  int64_t r0;         // first tree position
  int32_t nr;         // rows
  int32_t pad;
  int64_t c0, c1;     // chunks [c0, c1)
};
struct Combine {      // z[zi] = sum_{s in [s0, s1)} partial[s]
  int64_t zi;
  int64_t s0, s1;
};

}  // namespace hh

struct hh_matrix {
  // parameters
  int32_t d = 0, L = 0, s = 0;
  int64_t N = 0;
  hh_kernel kernel{};
  double eps = 0, eta = 0;
  int32_t leaf_size = 0;
  uint32_t pset = 0;
  bool ledger = false;
  int64_t ncell = 0;
  // tree
  std::vector<int64_t> leaf_start;        // host copy [ncell+1]
  hh::DBuf d_perm;                        // int32 [N]
  // blocks (host SoA, canonical order)
  std::vector<uint8_t> level, kind, tag, storage;
  std::vector<int64_t> tgt, src;
  std::vector<int32_t> rank, kfinal;
  std::vector<int64_t> zoff, w_off, ucol, d_off;
  std::vector<double> nb2, tot, maxabs;
  std::vector<int64_t> u_leaf_off;        // [4*(ncell+1)]
  std::vector<int64_t> d_leaf_off;        // [ncell+1]
  double norm2 = 0;
  int64_t ztotal = 0;
  // arenas
  hh::DBuf W[4], U[4], D;
  int64_t w_bytes[4] = {0, 0, 0, 0}, u_bytes[4] = {0, 0, 0, 0}, d_bytes = 0;
  // matvec plan
  hh::DBuf p1_items, p1_entries, p2_chunks, p2_leaves, combines;
  int64_t n_p1_items = 0, n_p2_leaves = 0, n_combines = 0, n_partials = 0;
  hh::DBuf v;        // [(N + ztotal) * 16] doubles
  hh::DBuf partial;  // [n_partials * 16] doubles
  hh::DBuf hx, hy;   // staging for hh_matvec_host
  // optional per-phase timing of the matvec (hh_matvec_profile)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // 4 per matvec chunk: start, after gather, after phase 1, after phase 2
  // statistics
  hh_info_t info{};
  ~hh_matrix() {
    for (auto e : prof_ev) cudaEventDestroy(e);
  }
};
