// compress_big.cu — §8(a) row a3 for blocks whose sketch is wide AND whose clusters are
// large (HODLR-level siblings, finer neighbours at coarse switch levels): the batched
// one-CTA-per-block pipeline of compress.cu would spend minutes on them (its per-block QR and
// Jacobi run on a single SM).  Same algorithm and same decision rule as compress.cu
// (randomized range finder + exact residual, G26), whole-GPU per block:
//   A  = entries of the block, formed explicitly in HBM (|I| x |J| fp64)   own kernel
//   Y  = A Omega        (Omega: the same counter hash as compress.cu)       cuBLAS DGEMM
//   Q  = qr(Y)                                                             cuSOLVER geqrf/orgqr
//   Z  = A^T Q                                                             cuBLAS DGEMM
//   R  = ||A - Q Z^T||_F^2, tot = ||A||_F^2 (fixed-order reductions)        DGEMM + own kernel
//   Z  = Uz S Vz^T  (so Q^T A = Vz S Uz^T)                                 cuSOLVER gesvd
//   U  = Q Vz[:, :p],  W = Z Vz[:, :p] = Uz S                              cuBLAS DGEMM
// cuBLAS / cuSOLVER are deterministic for fixed sizes on one device, so pass 2 (which writes
// the rounded factors) reproduces pass 1 bit for bit, as the batched path does.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "build.h"

namespace hh {

#define HH_BLAS(call)                                                                              \
  do {                                                                                             \
    cublasStatus_t s__ = (call);                                                                   \
    if (s__ != CUBLAS_STATUS_SUCCESS)                                                              \
      throw ::hh::Error(s__ == CUBLAS_STATUS_ALLOC_FAILED ? HH_ENOMEM : HH_ECUDA,                  \
                        std::string(#call) + ": cublas status " + std::to_string((int)s__));       \
  } while (0)
#define HH_SOLVER(call)                                                                            \
  do {                                                                                             \
    cusolverStatus_t s__ = (call);                                                                 \
    if (s__ != CUSOLVER_STATUS_SUCCESS)                                                            \
      throw ::hh::Error(s__ == CUSOLVER_STATUS_ALLOC_FAILED ? HH_ENOMEM : HH_ECUDA,                \
                        std::string(#call) + ": cusolver status " + std::to_string((int)s__));     \
  } while (0)

struct BigCtx::Impl {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t sol = nullptr;
  DBuf A, Om, Q, Z, Zc, VT, S, Uf, Wf, tau, work, info, red;
  ~Impl() {
    if (blas) cublasDestroy(blas);
    if (sol) cusolverDnDestroy(sol);
  }
};

BigCtx::BigCtx() : p(new Impl) {}
BigCtx::~BigCtx() { delete p; }

namespace {

__device__ __forceinline__ uint32_t mix32b(uint32_t x) {  // identical to compress.cu's hash
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ double omega(uint64_t gid, uint32_t j, uint32_t c) {
  uint32_t h = mix32b((uint32_t)gid * 0x9E3779B1u ^ (uint32_t)(gid >> 32) * 0x85EBCA77u ^ j * 0xC2B2AE3Du);
  h = mix32b(h ^ (c + 0x27D4EB2Fu) * 0x165667B1u);
  return (double)(int32_t)h * 0x1p-31;
}

__global__ void k_entries(double *A, const double *__restrict__ pts, int64_t N, int d, int64_t i0, int64_t j0,
                          int64_t m, int64_t n, KernelFn K) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(pts[k * N + i0 + i], pts[k * N + j0 + j]);
      r2 = __fma_rn(t, t, r2);
    }
    A[e] = kernel_eval(K, r2);
  }
}

__global__ void k_omega(double *Om, int64_t n, int k, uint64_t gid) {
  const int64_t total = n * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    Om[e] = omega(gid, (uint32_t)(e % n), (uint32_t)(e / n));
}

// Deterministic sum of squares: block b sums the fixed chunk [b*chunk, (b+1)*chunk) with a
// fixed thread/tree order; then one block sums the partials in index order.
constexpr int RB = 1024, RT = 256;
__global__ void k_sumsq_part(const double *a, int64_t count, double *part) {
  const int64_t chunk = (count + RB - 1) / RB;
  const int64_t s = blockIdx.x * chunk, e = min(count, s + chunk);
  double acc = 0.0;
  for (int64_t i = s + threadIdx.x; i < e; i += RT) acc = __fma_rn(a[i], a[i], acc);
  __shared__ double sh[RT];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = RT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_sum_final(const double *part, double *out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < RB; ++i) s += part[i];
    *out = s;
  }
}
__global__ void k_maxabs_part(const double *a, int64_t count, double *part) {
  const int64_t chunk = (count + RB - 1) / RB;
  const int64_t s = blockIdx.x * chunk, e = min(count, s + chunk);
  double mx = 0.0;
  for (int64_t i = s + threadIdx.x; i < e; i += RT) mx = fmax(mx, fabs(a[i]));
  __shared__ double sh[RT];
  sh[threadIdx.x] = mx;
  __syncthreads();
  for (int o = RT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_max_final(const double *part, double *out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < RB; ++i) s = fmax(s, part[i]);
    *out = s;
  }
}

__device__ __forceinline__ void store_tag(uint8_t *base, int64_t elem, int tag, double v) {
  switch (tag) {
    case TAG_FP64: reinterpret_cast<double *>(base)[elem] = v; break;
    case TAG_FP32: reinterpret_cast<uint32_t *>(base)[elem] = to_fp32_bits(v); break;
    case TAG_FP16: reinterpret_cast<uint16_t *>(base)[elem] = to_fp16_bits(v); break;
    case TAG_BF16: reinterpret_cast<uint16_t *>(base)[elem] = to_bf16_bits(v); break;
    case TAG_Q43: base[elem] = to_q43_bits(v); break;
    case TAG_BF24: {
      const uint32_t b = to_bf24_bits(v);
      base[3 * elem] = (uint8_t)b;
      base[3 * elem + 1] = (uint8_t)(b >> 8);
      base[3 * elem + 2] = (uint8_t)(b >> 16);
      break;
    }
    default: {  // fp48
      const uint64_t b = to_fp48_bits(v);
      uint16_t *h = reinterpret_cast<uint16_t *>(base) + 3 * elem;
      h[0] = (uint16_t)b;
      h[1] = (uint16_t)(b >> 16);
      h[2] = (uint16_t)(b >> 32);
    }
  }
}

// W (n x p, col-major fp64) -> columns wcol.. of the block's source panel (row-major tiles)
__global__ void k_store_w(const double *W, int64_t n, int p, uint8_t *arena, int64_t w_off, int64_t wcol,
                          int64_t wP, int64_t wts, int tag) {
  const int64_t total = n * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, c = e / n;
    const int64_t pc = wcol + c, t = pc / W_CT, j = pc - t * W_CT;
    const int64_t ct = min((int64_t)W_CT, wP - t * W_CT);
    store_tag(arena + w_off + t * wts, i * ct + j, tag, W[e]);
  }
}

// U (m x p, col-major fp64) -> rows of the target's leaf streams
__global__ void k_store_u(const double *U, int64_t m, int p, int64_t i0, uint8_t *arena, int tag, int64_t ucol,
                          Arenas ar) {
  const int64_t total = m * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, c = e / m;
    const int64_t pos = i0 + i;
    const int32_t R = ar.leaf_of[pos];
    const int64_t r0 = ar.leaf_start[R], nr = ar.leaf_start[R + 1] - r0;
    const int64_t off = ar.u_leaf_off[(int64_t)tag * (ar.ncell + 1) + R];
    store_tag(arena + off, (ucol + c) * nr + (pos - r0), tag, U[e]);
  }
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (n + 255) / 256)); }

}  // namespace

bool use_big_path(int64_t m, int64_t n, int k) {
  // a single-CTA Householder QR of an m x k panel costs ~2 m k^2 flops on one SM; the
  // threshold can be lowered (HH_BIG_FLOPS) so tests exercise this path on small inputs
  static const double thr = getenv("HH_BIG_FLOPS") ? atof(getenv("HH_BIG_FLOPS")) : 2.0e9;
  return (double)std::max(m, n) * (double)k * (double)k > thr;
}

void run_compress_big(hh_matrix *H, const double *pts, const CompressJob &job, bool write, const Arenas *ar,
                      CompressResult &res, cudaStream_t st, BigCtx &ctx) {
  BigCtx::Impl &c = *ctx.p;
  if (!c.blas) {
    HH_BLAS(cublasCreate(&c.blas));
    HH_SOLVER(cusolverDnCreate(&c.sol));
  }
  HH_BLAS(cublasSetStream(c.blas, st));
  HH_SOLVER(cusolverDnSetStream(c.sol, st));
  const int64_t b = job.block;
  int64_t i0, m, j0, n;
  cluster_range(H, H->level[b], H->tgt[b], i0, m);
  cluster_range(H, H->level[b], H->src[b], j0, n);
  const int k = (int)std::min<int64_t>(job.k, std::min(m, n));
  const KernelFn K = make_kernel_fn(H->kernel);
  auto grow = [](DBuf &buf, size_t bytes) {
    if (buf.bytes < bytes) buf.alloc(bytes);
  };
  {
    // the block is held explicitly in HBM: refuse (instead of failing in cudaMalloc) when it
    // and the sketch buffers do not fit in the free device memory
    const size_t need = sizeof(double) * ((size_t)m * n + 4 * (size_t)n * k + (size_t)m * k + (size_t)k * k);
    size_t held = c.A.bytes + c.Om.bytes + c.Q.bytes + c.Z.bytes + c.Zc.bytes + c.VT.bytes, fr = 0, tot = 0;
    HH_CUDA(cudaMemGetInfo(&fr, &tot));
    HH_REQUIRE(need <= fr + held, HH_EUNSUPPORTED,
               "block " + std::to_string(m) + " x " + std::to_string(n) + " needs " +
                   std::to_string(need >> 20) + " MiB for whole-GPU compression, more than the free device memory");
  }
  grow(c.A, sizeof(double) * m * n);
  grow(c.Om, sizeof(double) * n * k);
  grow(c.Q, sizeof(double) * m * k);
  grow(c.Z, sizeof(double) * n * k);
  grow(c.Zc, sizeof(double) * n * k);
  grow(c.VT, sizeof(double) * k * k);
  grow(c.S, sizeof(double) * k);
  grow(c.tau, sizeof(double) * k);
  grow(c.info, sizeof(int) * 4);
  grow(c.red, sizeof(double) * (RB + 8));
  double *A = c.A.as<double>(), *Om = c.Om.as<double>(), *Q = c.Q.as<double>(), *Z = c.Z.as<double>();
  double *Zc = c.Zc.as<double>(), *VT = c.VT.as<double>(), *S = c.S.as<double>(), *red = c.red.as<double>();
  const double one = 1.0, zero = 0.0, mone = -1.0;

  k_entries<<<grid_for(m * n), 256, 0, st>>>(A, pts, H->N, H->d, i0, j0, m, n, K);
  HH_LAUNCHED();
  double host[3] = {0, 0, 0};  // tot, R, maxabs
  k_sumsq_part<<<RB, RT, 0, st>>>(A, m * n, red);
  HH_LAUNCHED();
  k_sum_final<<<1, 32, 0, st>>>(red, red + RB);
  HH_LAUNCHED();
  HH_CUDA(cudaMemcpyAsync(&host[0], red + RB, sizeof(double), cudaMemcpyDeviceToHost, st));
  k_omega<<<grid_for(n * k), 256, 0, st>>>(Om, n, k, (uint64_t)b);
  HH_LAUNCHED();
  // Y = A Omega (into Q), Q = qr(Y)
  HH_BLAS(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)m, k, (int)n, &one, A, (int)m, Om, (int)n, &zero, Q,
                      (int)m));
  int lw1 = 0, lw2 = 0, lw3 = 0;
  HH_SOLVER(cusolverDnDgeqrf_bufferSize(c.sol, (int)m, k, Q, (int)m, &lw1));
  HH_SOLVER(cusolverDnDorgqr_bufferSize(c.sol, (int)m, k, k, Q, (int)m, c.tau.as<double>(), &lw2));
  HH_SOLVER(cusolverDnDgesvd_bufferSize(c.sol, (int)n, k, &lw3));
  grow(c.work, sizeof(double) * (size_t)std::max({lw1, lw2, lw3, 1}));
  double *work = c.work.as<double>();
  int *info = c.info.as<int>();
  HH_SOLVER(cusolverDnDgeqrf(c.sol, (int)m, k, Q, (int)m, c.tau.as<double>(), work, lw1, info));
  HH_SOLVER(cusolverDnDorgqr(c.sol, (int)m, k, k, Q, (int)m, c.tau.as<double>(), work, lw2, info + 1));
  // Z = A^T Q
  HH_BLAS(cublasDgemm(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, k, (int)m, &one, A, (int)m, Q, (int)m, &zero, Z,
                      (int)n));
  HH_CUDA(cudaMemcpyAsync(Zc, Z, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
  // SVD of Z (n x k, n >= k): rows of VT are the left singular vectors of Q^T A = Z^T
  HH_SOLVER(cusolverDnDgesvd(c.sol, 'N', 'A', (int)n, k, Zc, (int)n, S, nullptr, 1, VT, k, work, lw3, nullptr,
                             info + 2));
  if (!write) {
    // explicit residual E = A - Q Z^T (A is not needed afterwards in pass 1)
    HH_BLAS(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)m, (int)n, k, &mone, Q, (int)m, Z, (int)n, &one, A,
                        (int)m));
    k_sumsq_part<<<RB, RT, 0, st>>>(A, m * n, red);
    HH_LAUNCHED();
    k_sum_final<<<1, 32, 0, st>>>(red, red + RB + 1);
    HH_LAUNCHED();
    HH_CUDA(cudaMemcpyAsync(&host[1], red + RB + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  std::vector<double> s(k);
  int hinfo[4] = {0, 0, 0, 0};
  HH_CUDA(cudaMemcpyAsync(s.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaMemcpyAsync(hinfo, info, sizeof(int) * 3, cudaMemcpyDeviceToHost, st));
  HH_CUDA(cudaStreamSynchronize(st));
  HH_REQUIRE(hinfo[0] == 0 && hinfo[1] == 0 && hinfo[2] == 0, HH_ENUMERIC, "cuSOLVER QR/SVD failed on a block");
  const double tot = host[0], R = host[1];
  res = CompressResult{};
  res.k = k;
  res.tot = tot;
  res.R = R;
  int p = 0;
  if (write) {
    p = H->rank[b];
    res.ok = 1;
  } else if (tot == 0.0) {
    p = 0;
    res.ok = 1;
  } else {
    // the decision of compress.cu:k_decide (tail(p) = R + sum_{j >= p} s_j^2, from the smallest)
    const double thr = (H->eps * H->eps) * tot, delta = 1e-9;
    int best = -1;
    double t = R;
    if (t <= thr) best = k;
    for (int q = k - 1; q >= 0 && best == q + 1; --q) {
      t += s[q] * s[q];
      if (t <= thr) best = q;
    }
    const bool full = k >= std::min(m, n);
    if (best < 0 && full) best = k;
    bool exact = false;
    if (best == 0) {
      exact = true;
    } else if (best > 0) {
      double tprev = R;
      for (int j = k - 1; j >= best - 1; --j) tprev += s[j] * s[j];
      exact = (tprev - R > thr * (1.0 + delta)) && (R <= 1e-10 * tot);
    }
    res.ok = (best >= 0) && (full || exact);
    p = best;
  }
  res.p = p;
  // a not-ok decision is retried with a wider sketch, except at the sketch limit where the
  // caller accepts it (counted as inexact): its nb2 / maxabs must then be the real ones
  if (p <= 0 || (!res.ok && k < KMAX)) {
    res.nb2 = 0.0;
    res.maxabs = 0.0;
    return;
  }
  double nb2 = 0.0;
  for (int j = 0; j < p; ++j) nb2 = std::fma(s[j], s[j], nb2);
  res.nb2 = nb2;
  // factors: U = Q Vz[:, :p] (m x p), W = Z Vz[:, :p] (n x p); Vz[:, :p] = (first p rows of VT)^T
  grow(c.Uf, sizeof(double) * m * p);
  grow(c.Wf, sizeof(double) * n * p);
  double *Uf = c.Uf.as<double>(), *Wf = c.Wf.as<double>();
  HH_BLAS(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)m, p, k, &one, Q, (int)m, VT, k, &zero, Uf, (int)m));
  HH_BLAS(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, p, k, &one, Z, (int)n, VT, k, &zero, Wf, (int)n));
  if (!write) {
    k_maxabs_part<<<RB, RT, 0, st>>>(Uf, m * p, red);
    HH_LAUNCHED();
    k_max_final<<<1, 32, 0, st>>>(red, red + RB + 2);
    HH_LAUNCHED();
    k_maxabs_part<<<RB, RT, 0, st>>>(Wf, n * p, red);
    HH_LAUNCHED();
    k_max_final<<<1, 32, 0, st>>>(red, red + RB + 3);
    HH_LAUNCHED();
    double mx[2];
    HH_CUDA(cudaMemcpyAsync(mx, red + RB + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    HH_CUDA(cudaStreamSynchronize(st));
    res.maxabs = std::max(mx[0], mx[1]);
  } else {
    const int tag = H->tag[b];
    const int64_t wts = align_up(n * W_CT * tag_bytes(tag));
    k_store_w<<<grid_for(n * p), 256, 0, st>>>(Wf, n, p, ar->W[tag], H->w_off[b], H->wcol[b], H->wpanel[b], wts, tag);
    HH_LAUNCHED();
    k_store_u<<<grid_for(m * p), 256, 0, st>>>(Uf, m, p, i0, ar->U[tag], tag, H->ucol[b], *ar);
    HH_LAUNCHED();
    // pass 2 reports the same maxabs check as the batched path (determinism guard)
    k_maxabs_part<<<RB, RT, 0, st>>>(Uf, m * p, red);
    HH_LAUNCHED();
    k_max_final<<<1, 32, 0, st>>>(red, red + RB + 2);
    HH_LAUNCHED();
    k_maxabs_part<<<RB, RT, 0, st>>>(Wf, n * p, red);
    HH_LAUNCHED();
    k_max_final<<<1, 32, 0, st>>>(red, red + RB + 3);
    HH_LAUNCHED();
    double mx[2];
    HH_CUDA(cudaMemcpyAsync(mx, red + RB + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    HH_CUDA(cudaStreamSynchronize(st));
    res.maxabs = std::max(mx[0], mx[1]);
  }
}

}  // namespace hh
