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

// W panels: for each (tag, level, source cluster J) the tag's low-rank blocks
// with source J, in target order, form one |J| x P_J panel (P_J = sum of their ranks) split
// into column tiles of width <= W_CT, each stored row-major and 16-B aligned.
constexpr int W_CT = 248;  // row stride = 24 (fp32) / 28 (16-bit) banks mod 32: conflict-free 4-row DMMA fragments

// Phase-1 work item: a row range of one column tile of one W panel.  Tiles taller than
// P1_ROWS are cut into row pieces whose partial column sums go to a workspace and are added
// in piece order by a combine pass (load balance for HODLR-level panels).
constexpr int P1_ROWS = 4096;
struct P1Tile {
  int64_t src;        // byte offset of the tile in W[tag] (multiple of 16)
  int64_t x0;         // v index (tree position) of the tile's row 0
  int64_t zbase;      // index into zmap of the tile's column 0
  int64_t pbase;      // -1: write z; else partial index of column 0 of this piece
  int32_t n;          // rows of this piece
  int32_t r0;         // first row of this piece inside the tile
  int16_t ct;         // columns (1..W_CT)
  int16_t tag;
  int32_t pad;
};
struct P1Combine {    // z[zmap[zbase + c]] = sum_{q < npieces} partial[pbase + q * ct + c]
  int64_t zbase, pbase;
  int32_t ct, npieces;
};
// Phase-2 work: per leaf R, a list of segments; a segment is `ncols` contiguous |R|-row
// columns (column-major) of U[tag] or of the dense arena, multiplied by v[vbeg ...].
struct P2Seg {
  int64_t src;        // byte offset of column 0 in U[tag] (or D); multiple of the element size
  int64_t vbeg;       // v index of column 0's vector entry (z for U, x~ for dense)
  int32_t ncols;
  int16_t tag;        // 0..NTAG-1 (dense: 0)
  int16_t dense;      // 1 -> dense arena
};
struct P2Leaf {
  int64_t r0;         // first tree position
  int32_t nr;         // rows
  int32_t pad;
  int64_t s0, s1;     // segments [s0, s1)
};

// Stage plan of the single-RHS product: every shared-memory stage the
// persistent kernels will stream — one window of a W tile (phase 1) or of a leaf's U / dense
// segment (phase 2) with its vector slice — is precomputed at build time: the two bulk-copy
// windows (StageCopy) and the descriptor the consumers read (StageMeta).  The producer thread
// then only waits for a free stage and issues three bulk copies (factor window, vector window,
// descriptor); computing the windows on the fly cost it ~250 dependent instructions per stage,
// which bounded the small-leaf workloads (2D: ~7 KiB per stage).
struct StageMeta {     // 64 B, read by the consumers from the stage's descriptor slot
  int32_t kind;        // 0 = work, 1 = end of stream
  int32_t wlead;       // bytes between the staged window start and element 0
  int32_t xlead;
  int32_t r0, r1;      // phase 1: rows [r0, r1) of the tile;  phase 2: columns [r0, r1) of the segment
  int32_t flags;       // phase 2: bit 0 = last stage of the leaf
  int32_t a, b;        // phase 1: ct, tag;  phase 2: nr, tag | dense << 8
  int64_t p, q;        // phase 1: zbase, rows of the piece;  phase 2: leaf r0, -
  int64_t pb;          // phase 1: partial index of column 0 (row-split tile) or -1
  int64_t pad;
};
static_assert(sizeof(StageMeta) == 64, "stage descriptor slot");
struct StageCopy {     // 32 B: 16-B aligned enclosing windows (bytes may be 0: no copy)
  uint64_t wsrc, xsrc;
  uint32_t wbytes, xbytes;
  uint32_t pad[2];
};
static_assert(sizeof(StageCopy) == 32, "stage copy record");
struct StageItem {     // 48 B: an item's stages [s0, s1) and its first copy record (no dependent load)
  int64_t s0, s1;
  StageCopy first;
};
static_assert(sizeof(StageItem) == 48, "stage item record");
// single-RHS stage geometries (matvec.cu Geo<1, PH, GV>): factor bytes, vector entries, ring depth.
// GV 1 (twice the stages at half the size) serves plans whose windows are mostly small.
struct StageGeo {
  int wdata, xelems, stages;
};
constexpr StageGeo kStageGeo[2] = {{32768, 512, 2}, {16384, 256, 4}};

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
  bool tie16 = false;   // HH_TIE_FP16
  int64_t ncell = 0;
  // tree
  std::vector<int64_t> leaf_start;        // host copy [ncell+1]
  hh::DBuf d_perm;                        // int32 [N]
  // blocks (host SoA, canonical order)
  std::vector<uint8_t> level, kind, tag, storage;
  std::vector<int64_t> tgt, src;
  std::vector<int32_t> rank, kfinal;
  std::vector<int64_t> zoff, w_off, wcol, wpanel, ucol, d_off;
  std::vector<double> nb2, tot, maxabs;
  std::vector<int64_t> u_leaf_off;        // [NTAG*(ncell+1)]
  std::vector<int64_t> d_leaf_off;        // [ncell+1]
  double norm2 = 0;
  int64_t ztotal = 0;
  // arenas
  hh::DBuf W[hh::NTAG], U[hh::NTAG], D;
  int64_t w_bytes[hh::NTAG] = {}, u_bytes[hh::NTAG] = {}, d_bytes = 0;
  // matvec plan
  hh::DBuf p1_tiles, zmap, p2_segs, p2_leaves, p2_leaves_mo, p1_comb, partial;  // leaves: LPT / Morton order
  int64_t n_p1_tiles = 0, n_p2_leaves = 0, n_p1_comb = 0, n_partial = 0;
  // stage plan of the single-RHS product: per phase the items' stage ranges (item order), copy
  // records and descriptors; geom = stage geometry per phase (kStageGeo index)
  hh::DBuf st_item[2], st_copy[2], st_meta[2];
  int geom[2] = {0, 0};
  hh::DBuf v;        // [(N + ztotal) * 16] doubles (+ slack for 16-B aligned superset copies)
  hh::DBuf ctr;      // work counters of the persistent matvec kernels (zeroed by the gather)
  struct LaunchCfg {  // per RHS-chunk width (1, 2, 4, 8, 16): set once, reused by every hh_matvec
    bool ready = false;
    int nsm = 0, grid1 = 0, grid2 = 0;
  } lcfg[3][5];  // [working precision][width]
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
