// build.h — declarations shared by the build-pipeline translation units.
#pragma once
#include <vector>

#include "handle.h"

namespace hh {

constexpr int KMAX = 4096;  // sketch width limit (HODLR-level blocks at eps=1e-6 reach ranks of ~10^3)

struct CompressJob {
  int64_t block;  // index into the handle's block table
  int32_t k;      // sketch width
};

struct CompressResult {
  int32_t p, k;
  double nb2, tot, R, maxabs;
  int32_t ok;
};

// Pass-2 output placement (device pointers).
struct Arenas {
  uint8_t *W[NTAG];
  uint8_t *U[NTAG];
  const int64_t *u_leaf_off;  // [NTAG][ncell+1]
  const int64_t *leaf_start;  // [ncell+1]
  const int32_t *leaf_of;     // [N] tree position -> leaf cell
  int64_t ncell;
};

// Whole-GPU compression of one large, wide-sketch block (compress_big.cu): cuBLAS/cuSOLVER
// handles and workspaces kept across the blocks of one hh_build.
struct BigCtx {
  struct Impl;
  Impl *p;
  BigCtx();
  ~BigCtx();
  BigCtx(const BigCtx &) = delete;
  BigCtx &operator=(const BigCtx &) = delete;
};
bool use_big_path(int64_t m, int64_t n, int k);
void run_compress_big(hh_matrix *H, const double *pts, const CompressJob &job, bool write, const Arenas *ar,
                      CompressResult &res, cudaStream_t st, BigCtx &ctx);

KernelFn make_kernel_fn(const hh_kernel &kk);
void build_tree(hh_matrix *H, const double *P, cudaStream_t st, DBuf &pts_tree);
void build_partition(hh_matrix *H);
void run_compress(hh_matrix *H, const double *pts, const std::vector<CompressJob> &jobs, bool write,
                  const Arenas *ar, std::vector<CompressResult> &res, cudaStream_t st, size_t ws_budget);
void run_dense(hh_matrix *H, const double *pts, const std::vector<int64_t> &blocks, bool fill, cudaStream_t st);
void assign_tags(hh_matrix *H);
void compute_layout(hh_matrix *H);
void cluster_range(const hh_matrix *H, int l, int64_t m, int64_t &a, int64_t &n);
void build_plan(hh_matrix *H, std::vector<P1Tile> &tiles, std::vector<int32_t> &zmap, std::vector<P1Combine> &comb,
                int64_t &npartial, std::vector<P2Seg> &segs, std::vector<P2Leaf> &leaves,
                std::vector<P2Leaf> &leaves_morton);
// Stage plan of the single-RHS product (handle.h StageMeta / StageCopy): needs the arenas and
// the workspace H->v allocated (absolute device addresses); chooses H->geom per phase.
void build_stage_plan(hh_matrix *H, const std::vector<P1Tile> &tiles, const std::vector<P2Seg> &segs,
                      const std::vector<P2Leaf> &leaves, std::vector<StageItem> (&item)[2],
                      std::vector<StageCopy> (&copy)[2], std::vector<StageMeta> (&meta)[2]);
void run_matvec(hh_matrix *H, const double *x, double *y, int nrhs, cudaStream_t st, int wp = 0);
void print_build_profile();

}  // namespace hh
