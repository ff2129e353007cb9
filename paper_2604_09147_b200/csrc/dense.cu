// dense.cu — dense blocks: leaf diagonals (Alg. 1 last loop; stored in
// working precision fp64) and, for pure H_s, dense leaf neighbours
// (PAPER.md:580-588).  Entries f(||x_i - x_j||) with the singular-diagonal rule (G18):
// a zero distance gives 0 for singular kernels and f(0) = 1 otherwise.
#include <vector>

#include "build.h"

namespace hh {

struct DJob {
  int64_t i0, j0;
  int32_t m, n;
  int64_t off;   // byte offset into the dense arena (fill) or -1
};

namespace {
__global__ void k_dense(const DJob *jobs, const double *__restrict__ pts, int64_t N, int d, KernelFn K, uint8_t *arena,
                        double *tot, unsigned long long *coincident) {
  const DJob J = jobs[blockIdx.x];
  __shared__ double red[8];
  double s = 0.0;
  unsigned long long co = 0;
  const int64_t mn = (int64_t)J.m * J.n;
  for (int64_t e = threadIdx.x; e < mn; e += blockDim.x) {
    const int64_t i = e % J.m, j = e / J.m;
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      double t = __dsub_rn(pts[k * N + J.i0 + i], pts[k * N + J.j0 + j]);
      r2 = __fma_rn(t, t, r2);
    }
    if (r2 == 0.0 && J.i0 + i != J.j0 + j) ++co;
    const double v = kernel_eval(K, r2);
    s = __fma_rn(v, v, s);
    if (arena) reinterpret_cast<double *>(arena + J.off)[e] = v;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  if (co) atomicAdd(coincident, co);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    tot[blockIdx.x] = t;
  }
}
}  // namespace

// Evaluates the dense blocks `blocks` (indices into H's table): writes ||block||_F^2 into
// H->tot and, when `fill`, the entries (fp64, column-major) into the dense arena.
void run_dense(hh_matrix *H, const double *pts, const std::vector<int64_t> &blocks, bool fill, cudaStream_t st) {
  if (blocks.empty()) return;
  std::vector<DJob> jobs(blocks.size());
  for (size_t i = 0; i < blocks.size(); ++i) {
    const int64_t b = blocks[i];
    const int sh = H->d * (H->L - H->level[b]);
    DJob &J = jobs[i];
    J.i0 = H->leaf_start[H->tgt[b] << sh];
    J.m = (int32_t)(H->leaf_start[(H->tgt[b] + 1) << sh] - J.i0);
    J.j0 = H->leaf_start[H->src[b] << sh];
    J.n = (int32_t)(H->leaf_start[(H->src[b] + 1) << sh] - J.j0);
    J.off = fill ? H->d_off[b] : -1;
  }
  DBuf dj, dt, dc;
  h2d(dj, jobs, st);
  dt.alloc(sizeof(double) * jobs.size());
  dc.alloc(sizeof(unsigned long long));
  HH_CUDA(cudaMemsetAsync(dc.p, 0, 8, st));
  const KernelFn K = make_kernel_fn(H->kernel);
  for (size_t b0 = 0; b0 < jobs.size(); b0 += 1u << 20) {
    const unsigned nb = (unsigned)std::min<size_t>(1u << 20, jobs.size() - b0);
    k_dense<<<nb, 256, 0, st>>>(dj.as<DJob>() + b0, pts, H->N, H->d, K, fill ? H->D.as<uint8_t>() : nullptr,
                                dt.as<double>() + b0, dc.as<unsigned long long>());
    HH_LAUNCHED();
  }
  std::vector<double> t(jobs.size());
  unsigned long long co = 0;
  HH_CUDA(cudaMemcpyAsync(t.data(), dt.p, sizeof(double) * t.size(), cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaMemcpyAsync(&co, dc.p, 8, cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < blocks.size(); ++i) H->tot[blocks[i]] = t[i];
  if (!fill) H->info.n_coincident += (int64_t)co;
}

}  // namespace hh
