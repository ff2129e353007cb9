// tree.cu — §8(a) row a1: root cube, depth rule, Morton order on the device.
//
// balanced 2^d-tree; a leaf holds at most n_max points.  Readings
// (DESIGN.md §3): G1 depth = smallest L with every leaf <= n_max; G2 root cube = bounding
// cube of the points; G3 cell c_k = min(2^L-1, floor(ldexp((x_k - lo_k)/side, L))) (IEEE
// subtract + divide, exact ldexp / floor — no contraction possible); G4 Morton digits with
// axis 0 least significant, stable order (ties by original index).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "build.h"

namespace hh {

namespace {

__global__ void k_minmax(const double *__restrict__ P, int64_t N, int d, double *out, int *bad) {
  // out[blockIdx.x * 2d + k] = min, out[... + d + k] = max
  __shared__ double smin[3][256], smax[3][256];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int nf = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < d; ++k) {
      double v = P[i * d + k];
      if (!isfinite(v)) nf = 1;
      mn[k] = fmin(mn[k], v);
      mx[k] = fmax(mx[k], v);
    }
  }
  if (nf) atomicOr(bad, 1);
  for (int k = 0; k < d; ++k) {
    smin[k][threadIdx.x] = mn[k];
    smax[k][threadIdx.x] = mx[k];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < d; ++k) {
        smin[k][threadIdx.x] = fmin(smin[k][threadIdx.x], smin[k][threadIdx.x + s]);
        smax[k][threadIdx.x] = fmax(smax[k][threadIdx.x], smax[k][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < d; ++k) {
      out[blockIdx.x * 2 * d + k] = smin[k][0];
      out[blockIdx.x * 2 * d + d + k] = smax[k][0];
    }
}

struct Cube {
  double lo[3];
  double side;
};

__device__ __forceinline__ uint64_t morton_key(const double *x, int d, const Cube &C, int L) {
  uint64_t key = 0;
  const int64_t cmax = (1ll << L) - 1;
  for (int k = 0; k < d; ++k) {
    double t = __ddiv_rn(__dsub_rn(x[k], C.lo[k]), C.side);
    int64_t c = (int64_t)floor(ldexp(t, L));
    if (c > cmax) c = cmax;
    if (c < 0) c = 0;  // cannot happen (x >= lo), kept for safety
    for (int b = 0; b < L; ++b) key |= (uint64_t)((c >> b) & 1) << (b * d + k);
  }
  return key;
}

__global__ void k_hist(const double *__restrict__ P, int64_t N, int d, Cube C, int L, int *hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[morton_key(P + i * d, d, C, L)], 1);
}

__global__ void k_max(const int *h, int64_t n, int *out) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, h[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_keys(const double *__restrict__ P, int64_t N, int d, Cube C, int L, uint64_t *key, int32_t *idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = morton_key(P + i * d, d, C, L);
    idx[i] = (int32_t)i;
  }
}

__global__ void k_gather_pts(const double *__restrict__ P, int64_t N, int d, const int32_t *__restrict__ perm, double *pt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = perm[t];
    for (int k = 0; k < d; ++k) pt[k * N + t] = P[i * d + k];
  }
}

// flag = 1 if some run of equal sorted keys is longer than n_max (key[i] == key[i + n_max])
__global__ void k_long_run(const uint64_t *__restrict__ key, int64_t N, int nmax, int *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + nmax < N; i += (int64_t)gridDim.x * blockDim.x)
    if (key[i] == key[i + nmax]) *flag = 1;
}

inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

}  // namespace

constexpr int MAX_CELL_BITS = 26;

// Builds H->L, leaf_start, perm; returns tree-ordered points (SoA, d x N) in pts_tree.
void build_tree(hh_matrix *H, const double *P, cudaStream_t st, DBuf &pts_tree) {
  const int64_t N = H->N;
  const int d = H->d;
  // a1.1 bounding cube (min / max are order independent -> deterministic)
  const int nb = grid_for(N);
  DBuf part, bad;
  part.alloc(sizeof(double) * nb * 2 * d);
  bad.alloc(sizeof(int));
  HH_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  k_minmax<<<nb, 256, 0, st>>>(P, N, d, part.as<double>(), bad.as<int>());
  HH_LAUNCHED();
  std::vector<double> hp(nb * 2 * d);
  int hbad = 0;
  HH_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaStreamSynchronize(st));
  HH_REQUIRE(!hbad, HH_ENUMERIC, "non-finite point coordinate");
  Cube C{};
  double side = 0.0;
  for (int k = 0; k < d; ++k) {
    double mn = INFINITY, mx = -INFINITY;
    for (int b = 0; b < nb; ++b) {
      mn = std::min(mn, hp[b * 2 * d + k]);
      mx = std::max(mx, hp[b * 2 * d + d + k]);
    }
    C.lo[k] = mn;
    side = std::max(side, mx - mn);
  }
  if (side == 0.0) side = 1.0;
  C.side = side;
  // a1.2 depth rule: smallest L with max leaf count <= n_max
  DBuf hist, mx;
  mx.alloc(sizeof(int));
  int L = 0;
  for (;; ++L) {
    HH_REQUIRE((int64_t)d * L <= 62, HH_EDEPTH, "d*L exceeds 62 bits before every leaf holds <= leaf_size points");
    if (d * L > MAX_CELL_BITS) {
      // beyond this build's cell limit: report HH_EDEPTH when even the deepest 62-bit keys
      // leave more than leaf_size points in one cell (e.g. duplicated points), else unsupported
      const int Lmax = 62 / d;
      DBuf k1, k2, ix, flag, tb;
      k1.alloc(sizeof(uint64_t) * N);
      k2.alloc(sizeof(uint64_t) * N);
      ix.alloc(sizeof(int32_t) * N);
      flag.alloc(sizeof(int));
      HH_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
      k_keys<<<grid_for(N), 256, 0, st>>>(P, N, d, C, Lmax, k1.as<uint64_t>(), ix.as<int32_t>());
      HH_LAUNCHED();
      size_t tmp = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tmp, k1.as<uint64_t>(), k2.as<uint64_t>(), (int)N, 0, d * Lmax, st);
      tb.alloc(tmp);
      HH_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, tmp, k1.as<uint64_t>(), k2.as<uint64_t>(), (int)N, 0, d * Lmax, st));
      k_long_run<<<grid_for(N), 256, 0, st>>>(k2.as<uint64_t>(), N, H->leaf_size, flag.as<int>());
      HH_LAUNCHED();
      int hf = 0;
      HH_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      HH_CUDA(cudaStreamSynchronize(st));
      HH_REQUIRE(!hf, HH_EDEPTH, "d*L exceeds 62 bits before every leaf holds <= leaf_size points (duplicated points)");
      HH_REQUIRE(false, HH_EUNSUPPORTED, "more than 2^26 leaf cells needed");
    }
    const int64_t ncell = 1ll << (d * L);
    hist.alloc(sizeof(int) * ncell);
    HH_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(int) * ncell, st));
    HH_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), st));
    k_hist<<<grid_for(N), 256, 0, st>>>(P, N, d, C, L, hist.as<int>());
    HH_LAUNCHED();
    k_max<<<grid_for(ncell), 256, 0, st>>>(hist.as<int>(), ncell, mx.as<int>());
    HH_LAUNCHED();
    int hm = 0;
    HH_CUDA(cudaMemcpyAsync(&hm, mx.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    HH_CUDA(cudaStreamSynchronize(st));
    if (hm <= H->leaf_size) break;
  }
  H->L = L;
  H->ncell = 1ll << (d * L);
  // leaf offsets = exclusive scan of the final histogram
  std::vector<int> hh(H->ncell);
  HH_CUDA(cudaMemcpyAsync(hh.data(), hist.p, sizeof(int) * H->ncell, cudaMemcpyDeviceToHost, st));
  // a1.3 Morton keys + stable radix sort (ties keep original index order)
  DBuf keys, keys2, idx, perm;
  keys.alloc(sizeof(uint64_t) * N);
  keys2.alloc(sizeof(uint64_t) * N);
  idx.alloc(sizeof(int32_t) * N);
  H->d_perm.alloc(sizeof(int32_t) * N);
  k_keys<<<grid_for(N), 256, 0, st>>>(P, N, d, C, L, keys.as<uint64_t>(), idx.as<int32_t>());
  HH_LAUNCHED();
  if (d * L > 0) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.as<uint64_t>(), keys2.as<uint64_t>(), idx.as<int32_t>(),
                                    H->d_perm.as<int32_t>(), (int)N, 0, d * L, st);
    DBuf tbuf;
    tbuf.alloc(tmp);
    HH_CUDA(cub::DeviceRadixSort::SortPairs(tbuf.p, tmp, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                            idx.as<int32_t>(), H->d_perm.as<int32_t>(), (int)N, 0, d * L, st));
    count_launch(d * L / 8 + 1);
    HH_CUDA(cudaStreamSynchronize(st));
  } else {
    HH_CUDA(cudaMemcpyAsync(H->d_perm.p, idx.p, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
  }
  HH_CUDA(cudaStreamSynchronize(st));
  H->leaf_start.assign(H->ncell + 1, 0);
  for (int64_t m = 0; m < H->ncell; ++m) H->leaf_start[m + 1] = H->leaf_start[m] + hh[m];
  HH_REQUIRE(H->leaf_start[H->ncell] == N, HH_ECUDA, "leaf histogram does not sum to N");
  // tree-ordered points, structure of arrays
  pts_tree.alloc(sizeof(double) * N * d);
  k_gather_pts<<<grid_for(N), 256, 0, st>>>(P, N, d, H->d_perm.as<int32_t>(), pts_tree.as<double>());
  HH_LAUNCHED();
}

}  // namespace hh
