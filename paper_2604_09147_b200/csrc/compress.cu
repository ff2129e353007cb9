// compress.cu — §8(a) rows a3/a4: on-the-fly kernel entries + rank-revealing compression.
//
// Target: the truncated-SVD rank
//     p = min{p : sum_{k>p} sigma_k(A)^2 <= eps^2 ||A||_F^2}
// of every admissible block A (|I| x |J|, entries generated from the points),
// factors U (orthonormal) and W = A^T U, and ||H~_b||^2 = sum_{k<=p} sigma_k^2 (Alg. 4,
// PAPER.md:1327-1392).
//
// Device algorithm (not the paper's — the paper runs a full SVD in MATLAB):
//   Y = A Omega (Omega: k counter-hashed uniform columns)       fused entry-eval GEMM
//   Q = qr(Y) (Householder, explicit Q)                         CTA per block
//   Z = A^T Q                                                   fused entry-eval GEMM
//   T = R-factor of qr(Z);  Q^T A = Z^T = T^T P^T               CTA per block
//   T^T = Ut S J^T  by one-sided (Hestenes) Jacobi              CTA per block, smem
//   R = ||A - Q Z^T||_F^2 and tot = ||A||_F^2 from the ENTRIES  fused entry-eval GEMM
//   tail(p) = R + sum_{j>=p} s_j^2 (summed from the smallest) is exactly the error of the
//   rank-p factorization U = Q Ut_p, W = Z Ut_p; it exceeds the SVD tail by at most R,
//   so the rank equals the SVD rank unless the SVD decision is within R of its threshold.
//   A block is accepted when R <= 1e-9 eps^2 tot (or k = min(|I|,|J|)); else k doubles.
// Every kernel is deterministic (fixed reduction orders, no atomics in the arithmetic), so
// the second pass (which writes the rounded factors into the arenas once tags and layout
// are known) reproduces the first pass bit for bit.
#include <algorithm>
#include <cstring>
#include <vector>

#include "build.h"

namespace hh {

struct CBlk {
  int64_t i0, j0;      // first tree position of target / source cluster
  int32_t m, n, k, p;  // sizes, sketch width, rank (pass 2: known)
  int64_t oy, oq, oz, ozc, ot, os, otau;  // workspace offsets (doubles)
  int64_t task0;       // first resid task
  int64_t gid;         // block id (RNG stream)
  // pass-2 output placement
  int64_t w_off, ucol;  // W panel byte offset; first column inside the target's leaf streams
  int64_t wcol, wP, wts; // column inside the W panel, panel width, full-tile stride (bytes)
  int32_t tag, pad;
  // results
  double R, tot, nb2, maxabs;
  int32_t ok, pfound;
};

struct Task {
  int32_t blk;   // index into batch
  int32_t r0;    // first row of the tile
};

namespace {

constexpr int THREADS = 256;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {  // "lowbias32" integer finaliser
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

// Sketch matrix Omega(j, c) of block gid: a counter-based hash, uniform on [-1, 1) in steps of
// 2^-31; pure function of (gid, j, c) so pass 2 reproduces pass 1 bit for bit.
__device__ __forceinline__ double hash_uniform(uint64_t gid, uint32_t j, uint32_t c) {
  uint32_t h = mix32((uint32_t)gid * 0x9E3779B1u ^ (uint32_t)(gid >> 32) * 0x85EBCA77u ^ j * 0xC2B2AE3Du);
  h = mix32(h ^ (c + 0x27D4EB2Fu) * 0x165667B1u);
  return (double)(int32_t)h * 0x1p-31;
}

__device__ __forceinline__ double entry(const KernelFn &K, const double *pts, int64_t N, int d, int64_t a, int64_t b) {
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = __dsub_rn(pts[k * N + a], pts[k * N + b]);
    r2 = __fma_rn(t, t, r2);
  }
  return kernel_eval(K, r2);
}

// ---------------------------------------------------------------- fused entry GEMM
// mode 0: Y[:, c] = sum_j A(i, j) Omega(j, c)   rows = target cluster, cols = source
// mode 1: Z[:, c] = sum_i A(i, j) Q(i, c)       rows = source cluster, cols = target
constexpr int GT_M = 64, GT_K = 16;

// GT_N = sketch columns per CTA tile (32, 48 or 64: blocks are launched by sketch-width bucket)
template <int MODE, int GT_N>
__global__ void __launch_bounds__(THREADS) k_gemm_gen(const Task *__restrict__ tasks, CBlk *blks, double *ws,
                                                      const double *__restrict__ pts, int64_t N, int d, KernelFn K) {
  constexpr int TC = GT_N / 16;  // output columns per thread
  const Task T = tasks[blockIdx.x];
  const CBlk &B = blks[T.blk];
  const int rows = MODE == 0 ? B.m : B.n;
  const int cols = MODE == 0 ? B.n : B.m;
  const int64_t rbase = MODE == 0 ? B.i0 : B.j0;
  const int64_t cbase = MODE == 0 ? B.j0 : B.i0;
  const int k = B.k;
  const int c0 = blockIdx.y * GT_N;
  if (c0 >= k) return;
  __shared__ __align__(16) double As[GT_K][GT_M + 2];  // +2: 16-B aligned rows for 128-bit loads
  __shared__ __align__(16) double Xs[GT_K][GT_N + 2];
  __shared__ double rp[3][GT_M];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 4 x 4 outputs each
  for (int i = tid; i < GT_M * d; i += THREADS) {
    int r = i % GT_M, kk = i / GT_M;
    int64_t row = T.r0 + r;
    rp[kk][r] = row < rows ? pts[kk * N + rbase + row] : 0.0;
  }
  double acc[4][TC] = {};
  const double *X = ws + (MODE == 0 ? 0 : B.oq);
  for (int j0 = 0; j0 < cols; j0 += GT_K) {
    __syncthreads();
    // A tile: GT_M x GT_K entries, 4 per thread
    for (int e = tid; e < GT_M * GT_K; e += THREADS) {
      int r = e % GT_M, jj = e / GT_M;
      int64_t row = T.r0 + r, col = j0 + jj;
      double v = 0.0;
      if (row < rows && col < cols) {
        double r2 = 0.0;
        for (int kk = 0; kk < d; ++kk) {
          double t = __dsub_rn(rp[kk][r], pts[kk * N + cbase + col]);
          r2 = __fma_rn(t, t, r2);
        }
        v = kernel_eval(K, r2);
      }
      As[jj][r] = v;
    }
    for (int e = tid; e < GT_K * GT_N; e += THREADS) {
      int jj = e % GT_K, cc = e / GT_K;
      int col = j0 + jj, c = c0 + cc;
      double v = 0.0;
      if (col < cols && c < k) {
        if (MODE == 0)
          v = hash_uniform((uint64_t)B.gid, (uint32_t)col, (uint32_t)c);
        else
          v = X[(int64_t)c * cols + col];  // Q is |I| x k col-major (ld = m = cols)
      }
      Xs[jj][cc] = v;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < GT_K; ++jj) {
      double a[4], x[TC];
#pragma unroll
      for (int q = 0; q < 4; q += 2) {
        const double2 t = *reinterpret_cast<const double2 *>(&As[jj][ty * 4 + q]);
        a[q] = t.x;
        a[q + 1] = t.y;
      }
      if constexpr (TC % 2 == 0) {
#pragma unroll
        for (int q = 0; q < TC; q += 2) {
          const double2 t = *reinterpret_cast<const double2 *>(&Xs[jj][tx * TC + q]);
          x[q] = t.x;
          x[q + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < TC; ++q) x[q] = Xs[jj][tx * TC + q];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[r][c] = __fma_rn(a[r], x[c], acc[r][c]);
    }
  }
  double *Y = ws + (MODE == 0 ? B.oy : B.oz);
  double *Y2 = ws + B.ozc;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int64_t row = T.r0 + ty * 4 + r;
    if (row >= rows) continue;
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      int cc = c0 + tx * TC + c;
      if (cc >= k) continue;
      Y[(int64_t)cc * rows + row] = acc[r][c];
      if (MODE == 1) Y2[(int64_t)cc * rows + row] = acc[r][c];
    }
  }
}

// ---------------------------------------------------------------- block reductions
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*red)[NV], double *out, int nv) {
  // fixed-order: warp butterfly, then warps summed in index order by thread q
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[q] = x;
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp][q] = v[q];
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int w = 0; w < THREADS / 32; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- Householder QR
// A (m x k, col-major, ld m) in place: R in the upper triangle, reflector vectors below.
// SMEM: the m x k panel is copied to shared memory, factored there and (FORM_Q) turned into
// Q in place (the dorg2r order: j = k-1 .. 0), then written back once — every Householder
// step then costs shared-memory instead of L2 latency.  Used when m k doubles fit.
constexpr int QR_SMEM_ELEMS = 13824;  // 108 KiB: two CTAs per SM
template <bool FORM_Q, bool SMEM>
__global__ void __launch_bounds__(THREADS) k_qr(CBlk *blks, const int32_t *__restrict__ order, double *ws, int which) {
  extern __shared__ double qsm[];
  CBlk &B = blks[order[blockIdx.x]];
  const int m = which == 0 ? B.m : B.n;
  const int k = B.k;
  double *Ag = ws + (which == 0 ? B.oy : B.ozc);
  double *A = SMEM ? qsm : Ag;
  double *tau = ws + B.otau;
  __shared__ double red[THREADS / 32][8];
  __shared__ double bc[8];
  __shared__ double sc[4];
  const int tid = threadIdx.x;
  if (SMEM) {
    for (int64_t e = tid; e < (int64_t)m * k; e += THREADS) A[e] = Ag[e];
    __syncthreads();
  }
  for (int j = 0; j < k; ++j) {
    double *aj = A + (int64_t)j * m;
    double v1[1] = {0.0};
    for (int i = j + 1 + tid; i < m; i += THREADS) v1[0] = __fma_rn(aj[i], aj[i], v1[0]);
    block_sum<1>(v1, (double(*)[1])red, bc, 1);
    if (tid == 0) {
      double xn2 = bc[0], alpha = aj[j], t = 0.0, beta = alpha, scale = 0.0;
      if (xn2 != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      sc[0] = t;
      sc[1] = scale;
      sc[2] = beta;
      tau[j] = t;
    }
    __syncthreads();
    const double t = sc[0], scale = sc[1];
    if (t != 0.0)
      for (int i = j + 1 + tid; i < m; i += THREADS) aj[i] *= scale;
    __syncthreads();
    if (tid == 0) aj[j] = sc[2];
    if (t != 0.0) {
      for (int c0 = j + 1; c0 < k; c0 += 8) {
        const int nc = min(8, k - c0);
        double w[8] = {};
        for (int i = j + 1 + tid; i < m; i += THREADS) {
          double v = aj[i];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < nc) w[q] = __fma_rn(v, A[(int64_t)(c0 + q) * m + i], w[q]);
        }
        block_sum<8>(w, red, bc, nc);
        // w_q = tau (a_{j,c} + v^T a_c), formed before row j of a_c is updated
        if (tid < nc) bc[tid] = t * (bc[tid] + A[(int64_t)(c0 + tid) * m + j]);
        __syncthreads();
        for (int i = j + tid; i < m; i += THREADS) {
          double v = (i == j) ? 1.0 : aj[i];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < nc) A[(int64_t)(c0 + q) * m + i] -= v * bc[q];
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (SMEM) {
    if (FORM_Q) {
      // in place: A <- H_0 ... H_{k-1} [I; 0] (reflector j lives below the diagonal of column j)
      for (int j = k - 1; j >= 0; --j) {
        const double t = tau[j];
        for (int c0 = j + 1; c0 < k; c0 += 8) {  // apply H_j to columns j+1.. (rows j..m)
          const int nc = min(8, k - c0);
          double w[8] = {};
          for (int i = j + 1 + tid; i < m; i += THREADS) {
            const double v = A[(int64_t)j * m + i];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nc) w[q] = __fma_rn(v, A[(int64_t)(c0 + q) * m + i], w[q]);
          }
          block_sum<8>(w, red, bc, nc);
          if (tid < nc) bc[tid] = t * (bc[tid] + A[(int64_t)(c0 + tid) * m + j]);
          __syncthreads();
          for (int i = j + tid; i < m; i += THREADS) {
            const double v = (i == j) ? 1.0 : A[(int64_t)j * m + i];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nc) A[(int64_t)(c0 + q) * m + i] -= v * bc[q];
          }
          __syncthreads();
        }
        for (int i = tid; i < m; i += THREADS) {  // column j of Q
          double *a = A + (int64_t)j * m;
          a[i] = i < j ? 0.0 : (i == j ? 1.0 - t : -t * a[i]);
        }
        __syncthreads();
      }
      double *Q = ws + B.oq;
      for (int64_t e = tid; e < (int64_t)m * k; e += THREADS) Q[e] = A[e];
    } else {
      for (int64_t e = tid; e < (int64_t)m * k; e += THREADS) Ag[e] = A[e];
    }
    return;
  }
  if (!FORM_Q) return;
  // explicit Q = H_0 ... H_{k-1} [I; 0] by backward accumulation (into oq)
  double *Q = ws + B.oq;
  for (int64_t e = tid; e < (int64_t)m * k; e += THREADS) {
    int64_t i = e % m, c = e / m;
    Q[e] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const double *aj = A + (int64_t)j * m;
    for (int c0 = j; c0 < k; c0 += 8) {
      const int nc = min(8, k - c0);
      double w[8] = {};
      for (int i = j + tid; i < m; i += THREADS) {
        double v = (i == j) ? 1.0 : aj[i];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < nc) w[q] = __fma_rn(v, Q[(int64_t)(c0 + q) * m + i], w[q]);
      }
      block_sum<8>(w, red, bc, nc);
      for (int i = j + tid; i < m; i += THREADS) {
        double v = (i == j) ? 1.0 : aj[i];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < nc) Q[(int64_t)(c0 + q) * m + i] -= v * (t * bc[q]);
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- Hestenes Jacobi
// M = T^T (k x k) where T = upper triangle of the QR of Z (stored in Zc, ld n).
// Output: s (descending) at os, Ut (k x k, columns = left singular vectors of T^T) at ot.
constexpr int JAC_SMEM_K = 168;   // 168^2 doubles = 220.5 KiB of shared memory
// JT threads per block (JT/32 rotation pairs in flight); launched per k-bucket so that small
// cores get small CTAs and small shared memory (several blocks per SM).
template <int JT>
__global__ void __launch_bounds__(JT) k_jacobi(CBlk *blks, const int32_t *__restrict__ order, double *ws) {
  extern __shared__ double smem[];
  CBlk &B = blks[order[blockIdx.x]];
  const int k = B.k, n = B.n;
  double *M = (k <= JAC_SMEM_K) ? smem : ws + B.oy;  // Y no longer needed (Q formed)
  const double *R = ws + B.ozc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t e = tid; e < (int64_t)k * k; e += JT) {
    int i = (int)(e % k), j = (int)(e / k);
    M[e] = (j <= i) ? R[(int64_t)i * n + j] : 0.0;  // M[i][j] = T[j][i]
  }
  __shared__ int rot;
  __syncthreads();
  const int kk = (k + 1) & ~1;
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rot = 0;
    __syncthreads();
    int myrot = 0;
    for (int r = 0; r < kk - 1; ++r) {
      for (int q = warp; q < kk / 2; q += JT / 32) {
        auto player = [&](int pos) { return pos == 0 ? 0 : (pos - 1 + r) % (kk - 1) + 1; };
        int a = player(q), b = player(kk - 1 - q);
        if (a >= k || b >= k) continue;
        double *ca = M + (int64_t)a * k, *cb = M + (int64_t)b * k;
        double al = 0, be = 0, ga = 0;
        for (int i = lane; i < k; i += 32) {
          double x = ca[i], y = cb[i];
          al = __fma_rn(x, x, al);
          be = __fma_rn(y, y, be);
          ga = __fma_rn(x, y, ga);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          double zeta = (be - al) / (2.0 * ga);
          double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < k; i += 32) {
            double x = ca[i], y = cb[i];
            ca[i] = c * x - s * y;
            cb[i] = s * x + c * y;
          }
          myrot = 1;
        }
      }
      __syncthreads();
    }
    if (myrot && lane == 0) atomicOr(&rot, 1);
    __syncthreads();
    if (rot == 0) break;
    __syncthreads();
  }
  // column norms -> sigma; sort descending (ties by index); normalise
  double *sig = ws + B.os;
  double *Ut = ws + B.ot;
  double *norms = ws + B.otau;  // tau no longer needed
  for (int j = warp; j < k; j += JT / 32) {
    double s = 0;
    for (int i = lane; i < k; i += 32) s = __fma_rn(M[(int64_t)j * k + i], M[(int64_t)j * k + i], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) norms[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < k; j += JT) {
    double nj = norms[j];
    int rk = 0;
    for (int i = 0; i < k; ++i) {
      double ni = norms[i];
      rk += (ni > nj) || (ni == nj && i < j);
    }
    sig[rk] = nj;
    norms[k + j] = (double)rk;  // stash rank (tau area has >= 2k doubles)
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)k * k; e += JT) {
    int i = (int)(e % k), j = (int)(e / k);
    int rk = (int)norms[k + j];
    double nj = norms[j];
    Ut[(int64_t)rk * k + i] = nj > 0.0 ? M[e] / nj : 0.0;
  }
}

// ---------------------------------------------------------------- residual energy
// per task (block, 32-row tile of I): sum over the tile of (A - Q Z^T)^2 and A^2
constexpr int RT_M = 32, RT_N = 32, RT_K = 32;

__global__ void __launch_bounds__(THREADS) k_resid(const Task *__restrict__ tasks, const CBlk *blks, const double *ws,
                                                   const double *__restrict__ pts, int64_t N, int d, KernelFn K,
                                                   double *part) {
  const Task T = tasks[blockIdx.x];
  const CBlk &B = blks[T.blk];
  const int m = B.m, n = B.n, k = B.k;
  const double *Q = ws + B.oq, *Z = ws + B.oz;
  __shared__ double Qs[RT_K][RT_M + 1];
  __shared__ double Zs[RT_K][RT_N + 1];
  __shared__ double rp[3][RT_M];
  __shared__ double red[THREADS / 32][2];
  const int tid = threadIdx.x;
  for (int i = tid; i < RT_M * d; i += THREADS) {
    int r = i % RT_M, kk = i / RT_M;
    rp[kk][r] = (T.r0 + r < m) ? pts[kk * N + B.i0 + T.r0 + r] : 0.0;
  }
  // thread -> (row r = tid % 32, cols c = tid / 32 + 8 q, q < 4)
  const int r = tid % RT_M, cg = tid / RT_M;
  double e2 = 0.0, a2 = 0.0;
  for (int j0 = 0; j0 < n; j0 += RT_N) {
    double s[4] = {0, 0, 0, 0};
    for (int c0 = 0; c0 < k; c0 += RT_K) {
      __syncthreads();
      for (int e = tid; e < RT_K * RT_M; e += THREADS) {
        int rr = e % RT_M, cc = e / RT_M;
        Qs[cc][rr] = (T.r0 + rr < m && c0 + cc < k) ? Q[(int64_t)(c0 + cc) * m + T.r0 + rr] : 0.0;
        Zs[cc][rr] = (j0 + rr < n && c0 + cc < k) ? Z[(int64_t)(c0 + cc) * n + j0 + rr] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int cc = 0; cc < RT_K; ++cc) {
        double qv = Qs[cc][r];
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = __fma_rn(qv, Zs[cc][cg + 8 * q], s[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t col = j0 + cg + 8 * q;
      if (T.r0 + r < m && col < n) {
        double r2 = 0.0;
        for (int kk = 0; kk < d; ++kk) {
          double t = __dsub_rn(rp[kk][r], pts[kk * N + B.j0 + col]);
          r2 = __fma_rn(t, t, r2);
        }
        double a = kernel_eval(K, r2);
        double e = a - s[q];
        e2 = __fma_rn(e, e, e2);
        a2 = __fma_rn(a, a, a2);
      }
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) {
    red[warp][0] = e2;
    red[warp][1] = a2;
  }
  __syncthreads();
  if (tid == 0) {
    double se = 0, sa = 0;
    for (int w = 0; w < THREADS / 32; ++w) {
      se += red[w][0];
      sa += red[w][1];
    }
    part[2 * blockIdx.x] = se;
    part[2 * blockIdx.x + 1] = sa;
  }
}

// ---------------------------------------------------------------- decision
__global__ void k_decide(CBlk *blks, int nb, const double *ws, const double *part, double eps, double delta) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  CBlk &B = blks[b];
  const int ntask = (B.m + RT_M - 1) / RT_M;
  double R = 0, tot = 0;
  for (int t = 0; t < ntask; ++t) {
    R += part[2 * (B.task0 + t)];
    tot += part[2 * (B.task0 + t) + 1];
  }
  B.R = R;
  B.tot = tot;
  const double *s = ws + B.os;
  const int k = B.k;
  const double thr = (eps * eps) * tot;
  if (tot == 0.0) {
    B.pfound = 0;
    B.nb2 = 0;
    B.ok = 1;
    return;
  }
  int best = -1;
  double t = R;
  if (t <= thr) best = k;
  for (int p = k - 1; p >= 0 && best == p + 1; --p) {
    t += s[p] * s[p];
    if (t <= thr) best = p;
  }
  const bool full = k >= min(B.m, B.n);
  if (best < 0 && full) best = k;
  B.pfound = best;
  double nb2 = 0;
  for (int j = 0; j < max(best, 0); ++j) nb2 = __fma_rn(s[j], s[j], nb2);
  B.nb2 = nb2;
  // Exactness of the decision: the SVD tail satisfies gpu_tail(q) - R <= tail(q) <= gpu_tail(q)
  // for every q (interlacing of sigma(Q^T A) with sigma(A)).  Hence the SVD rank equals
  // `best` when gpu_tail(best - 1) - R > thr, i.e. R is below the gap at the decision; a
  // relative guard of 1e-9 absorbs rounding.  R <= 1e-10 tot keeps nb2 (which feeds the
  // precision tag, Eq. 4.4) accurate to 1e-10.  Otherwise the sketch is widened.
  bool exact = false;
  if (best == 0) {
    exact = true;
  } else if (best > 0) {
    double tprev = R;  // gpu_tail(best - 1) = R + sum_{j >= best-1} s_j^2
    for (int j = k - 1; j >= best - 1; --j) tprev += s[j] * s[j];
    exact = (tprev - R > thr * (1.0 + delta)) && (R <= 1e-10 * tot);
  }
  B.ok = (best >= 0) && (full || exact);
}

// ---------------------------------------------------------------- factors
// U = Q Ut[:, :p] (m x p), W = Z Ut[:, :p] (n x p).  Pass 1: max |entry|.  Pass 2: round to
// the block's tag and store (W: columns wcol.. of its source panel, row-major column tiles;
// U rows into the target's leaf streams).
__device__ __forceinline__ void store_tagged(uint8_t *base, int64_t elem, int tag, double v) {
  switch (tag) {
    case TAG_FP64:
      reinterpret_cast<double *>(base)[elem] = v;
      break;
    case TAG_FP32:
      reinterpret_cast<uint32_t *>(base)[elem] = to_fp32_bits(v);
      break;
    case TAG_FP16:
      reinterpret_cast<uint16_t *>(base)[elem] = to_fp16_bits(v);
      break;
    case TAG_BF16:
      reinterpret_cast<uint16_t *>(base)[elem] = to_bf16_bits(v);
      break;
    case TAG_Q43:
      base[elem] = to_q43_bits(v);
      break;
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

constexpr int FC = 32;  // output columns per pass

__global__ void __launch_bounds__(THREADS) k_factors(CBlk *blks, const double *ws, int write, Arenas ar) {
  CBlk &B = blks[blockIdx.x];
  const int p = B.pfound, k = B.k;
  if (p <= 0) {
    if (threadIdx.x == 0) B.maxabs = 0.0;
    return;
  }
  __shared__ double Us[FC][161];
  __shared__ double red[THREADS / 32];
  const double *Ut = ws + B.ot;
  double mx = 0.0;
  for (int side = 0; side < 2; ++side) {
    const int rows = side == 0 ? B.m : B.n;
    const double *S = ws + (side == 0 ? B.oq : B.oz);
    for (int i0 = 0; i0 < rows; i0 += THREADS) {
      const int i = i0 + threadIdx.x;
      const bool valid = i < rows;
      for (int c0 = 0; c0 < p; c0 += FC) {
        const int nc = min(FC, p - c0);
        double acc[FC];
#pragma unroll
        for (int q = 0; q < FC; ++q) acc[q] = 0.0;
        for (int kt0 = 0; kt0 < k; kt0 += 160) {
          const int kn = min(160, k - kt0);
          __syncthreads();
          for (int e = threadIdx.x; e < FC * kn; e += THREADS) {
            int t = e % kn, q = e / kn;
            Us[q][t] = (q < nc) ? Ut[(int64_t)(c0 + q) * k + kt0 + t] : 0.0;
          }
          __syncthreads();
          if (valid)
            for (int t = 0; t < kn; ++t) {
              double sv = S[(int64_t)(kt0 + t) * rows + i];
#pragma unroll
              for (int q = 0; q < FC; ++q) acc[q] = __fma_rn(sv, Us[q][t], acc[q]);
            }
        }
        if (!valid) continue;
        for (int q = 0; q < nc; ++q) {
          mx = fmax(mx, fabs(acc[q]));
          if (write) {
            const int c = c0 + q;
            if (side == 1) {
              const int64_t pc = B.wcol + c, t = pc / W_CT, j = pc - t * W_CT;
              const int64_t ct = min((int64_t)W_CT, B.wP - t * W_CT);
              store_tagged(ar.W[B.tag] + B.w_off + t * B.wts, (int64_t)i * ct + j, B.tag, acc[q]);
            } else {
              const int64_t pos = B.i0 + i;
              const int32_t R = ar.leaf_of[pos];
              const int64_t r0 = ar.leaf_start[R], nr = ar.leaf_start[R + 1] - r0;
              const int64_t off = ar.u_leaf_off[(int64_t)B.tag * (ar.ncell + 1) + R];
              store_tagged(ar.U[B.tag] + off, (B.ucol + c) * nr + (pos - r0), B.tag, acc[q]);
            }
          }
        }
      }
    }
  }
  // block max (order independent)
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0;
    for (int w = 0; w < THREADS / 32; ++w) v = fmax(v, red[w]);
    B.maxabs = v;
  }
}

}  // namespace

// --------------------------------------------------------------------- host driver
// QR launches: blocks whose panel fits shared memory take the SMEM kernel (one launch sized to
// the largest of them), the rest the global-memory kernel.
static void launch_qr(const std::vector<CBlk> &blks, int nb, DBuf &ordb, int which, CBlk *db, double *ws,
                      cudaStream_t st) {
  std::vector<int32_t> ord;
  int nsm = 0;
  int64_t mk_max = 0;
  for (int i = 0; i < nb; ++i) {
    const int64_t mk = (int64_t)(which == 0 ? blks[i].m : blks[i].n) * blks[i].k;
    if (mk <= QR_SMEM_ELEMS) {
      ord.push_back(i);
      ++nsm;
      mk_max = std::max(mk_max, mk);
    }
  }
  for (int i = 0; i < nb; ++i) {
    const int64_t mk = (int64_t)(which == 0 ? blks[i].m : blks[i].n) * blks[i].k;
    if (mk > QR_SMEM_ELEMS) ord.push_back(i);
  }
  h2d(ordb, ord, st);
  const int32_t *od = ordb.as<int32_t>();
  if (nsm > 0) {
    const size_t sm = sizeof(double) * (size_t)mk_max;
    if (which == 0) {
      HH_CUDA(cudaFuncSetAttribute(k_qr<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * QR_SMEM_ELEMS)));
      k_qr<true, true><<<nsm, THREADS, sm, st>>>(db, od, ws, which);
    } else {
      HH_CUDA(cudaFuncSetAttribute(k_qr<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * QR_SMEM_ELEMS)));
      k_qr<false, true><<<nsm, THREADS, sm, st>>>(db, od, ws, which);
    }
    HH_LAUNCHED();
  }
  if (nb - nsm > 0) {
    if (which == 0)
      k_qr<true, false><<<nb - nsm, THREADS, 0, st>>>(db, od + nsm, ws, which);
    else
      k_qr<false, false><<<nb - nsm, THREADS, 0, st>>>(db, od + nsm, ws, which);
    HH_LAUNCHED();
  }
}

KernelFn make_kernel_fn(const hh_kernel &kk) {
  KernelFn K{};
  K.kind = kk.kind;
  K.scale = kk.scale;
  if (kk.kind == HH_K_GAUSS) K.c = -1.0 / (2.0 * kk.scale * kk.scale);
  if (kk.kind == HH_K_EXP) K.c = -1.0 / kk.scale;
  return K;
}

// Runs the compression pipeline on `jobs` (pass 1: results only; pass 2: also write the
// rounded factors).  Returns one result per job.
// Optional build profile (HH_PROFILE_BUILD=1): per-stage device time accumulated over batches.
static const char *kStage[8] = {"gemm_Y", "qr_Y", "gemm_Z", "qr_Z", "jacobi", "resid", "decide", "factors"};
double g_stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
int64_t g_stage_batches = 0;
void print_build_profile() {
  fprintf(stderr, "[hh build profile] batches=%lld", (long long)g_stage_batches);
  for (int i = 0; i < 8; ++i) fprintf(stderr, " %s=%.1fms", kStage[i], g_stage_ms[i]);
  fprintf(stderr, "\n");
}

void run_compress(hh_matrix *H, const double *pts, const std::vector<CompressJob> &jobs, bool write,
                  const Arenas *ar, std::vector<CompressResult> &res, cudaStream_t st, size_t ws_budget) {
  static const bool prof = getenv("HH_PROFILE_BUILD") != nullptr;
  cudaEvent_t ev[9];
  if (prof)
    for (int i = 0; i < 9; ++i) HH_CUDA(cudaEventCreate(&ev[i]));
  auto mark = [&](int i) {
    if (prof) HH_CUDA(cudaEventRecord(ev[i], st));
  };
  res.assign(jobs.size(), CompressResult{});
  const KernelFn K = make_kernel_fn(H->kernel);
  const double delta = 1e-9;
  DBuf wsb, blkb, taskb, partb, ordb, ordq_y, ordq_z;
  size_t ws_cap = 0;
  size_t pos = 0;
  std::vector<CBlk> blks;
  std::vector<Task> tasks;
  auto cluster = [&](int l, int64_t m, int64_t &a, int64_t &n) {
    const int sh = H->d * (H->L - l);
    a = H->leaf_start[m << sh];
    n = H->leaf_start[(m + 1) << sh] - a;
  };
  while (pos < jobs.size()) {
    // assemble a batch within the workspace budget
    blks.clear();
    tasks.clear();
    int64_t off = 0;
    size_t end = pos;
    while (end < jobs.size() && blks.size() < 65536) {
      const CompressJob &J = jobs[end];
      const int64_t b = J.block;
      CBlk c{};
      int64_t mi, ni;
      cluster(H->level[b], H->tgt[b], c.i0, mi);
      cluster(H->level[b], H->src[b], c.j0, ni);
      c.m = (int)mi;
      c.n = (int)ni;
      c.k = std::min<int>(J.k, std::min(c.m, c.n));
      const int64_t need = (2 * (int64_t)c.m + 2 * (int64_t)c.n) * c.k + (int64_t)c.k * c.k + 3 * (int64_t)c.k + 8;
      if (!blks.empty() && (size_t)(off + need) * 8 > ws_budget) break;
      c.oy = off;
      c.oq = c.oy + (int64_t)c.m * c.k;
      c.oz = c.oq + (int64_t)c.m * c.k;
      c.ozc = c.oz + (int64_t)c.n * c.k;
      c.ot = c.ozc + (int64_t)c.n * c.k;
      c.os = c.ot + (int64_t)c.k * c.k;
      c.otau = c.os + c.k;
      off = c.otau + 2 * c.k + 8;
      c.gid = b;
      c.task0 = 0;
      if (write) {  // pass 2: rank known from pass 1 (bitwise-identical pipeline)
        c.pfound = H->rank[b];
        c.tag = H->tag[b];
        c.w_off = H->w_off[b];
        c.ucol = H->ucol[b];
        c.wcol = H->wcol[b];
        c.wP = H->wpanel[b];
        c.wts = align_up((int64_t)c.n * W_CT * tag_bytes(c.tag));
      }
      blks.push_back(c);
      ++end;
    }
    const int nb = (int)blks.size();
    // tasks: target-row tiles (mode 0 / resid), source-row tiles (mode 1)
    // GEMM tasks grouped by sketch-width bucket (k <= 32, <= 48, > 48: 64-column tiles)
    std::vector<Task> tA, tB, tR;
    int nA[3] = {0, 0, 0}, nB[3] = {0, 0, 0}, kmxb[3] = {0, 0, 0};
    auto kb = [](int k) { return k <= 32 ? 0 : k <= 48 ? 1 : 2; };
    for (int bkt = 0; bkt < 3; ++bkt)
      for (int i = 0; i < nb; ++i) {
        if (kb(blks[i].k) != bkt) continue;
        kmxb[bkt] = std::max(kmxb[bkt], blks[i].k);
        for (int r = 0; r < blks[i].m; r += GT_M, ++nA[bkt]) tA.push_back(Task{i, r});
      }
    for (int bkt = 0; bkt < 3; ++bkt)
      for (int i = 0; i < nb; ++i) {
        if (kb(blks[i].k) != bkt) continue;
        for (int r = 0; r < blks[i].n; r += GT_M, ++nB[bkt]) tB.push_back(Task{i, r});
      }
    for (int i = 0; i < nb; ++i) {
      blks[i].task0 = (int64_t)tR.size();
      for (int r = 0; r < blks[i].m; r += RT_M) tR.push_back(Task{i, r});
    }
    if ((size_t)off * 8 > ws_cap) {
      ws_cap = std::max((size_t)off * 8, std::min<size_t>(ws_budget, (size_t)off * 8 * 2));
      wsb.alloc(ws_cap);
    }
    h2d(blkb, blks, st);
    std::vector<Task> all;
    all.insert(all.end(), tA.begin(), tA.end());
    all.insert(all.end(), tB.begin(), tB.end());
    all.insert(all.end(), tR.begin(), tR.end());
    h2d(taskb, all, st);
    partb.alloc(sizeof(double) * 2 * std::max<size_t>(1, tR.size()));
    const Task *dA = taskb.as<Task>(), *dB = dA + tA.size(), *dR = dB + tB.size();
    double *ws = wsb.as<double>();
    CBlk *db = blkb.as<CBlk>();
    // fused entry GEMMs per sketch-width bucket (MODE 0: Y = A Omega, MODE 1: Z = A^T Q)
    auto gemm = [&](int mode, const Task *tasks, const int *cnt) {
      size_t base = 0;
      for (int bkt = 0; bkt < 3; ++bkt) {
        const int gy = bkt < 2 ? 1 : (kmxb[2] + 63) / 64;
        for (size_t t0 = 0; t0 < (size_t)cnt[bkt]; t0 += 65535) {
          dim3 g((unsigned)std::min<size_t>(65535, cnt[bkt] - t0), gy);
          const Task *tp = tasks + base + t0;
          if (mode == 0) {
            if (bkt == 0) k_gemm_gen<0, 32><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
            else if (bkt == 1) k_gemm_gen<0, 48><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
            else k_gemm_gen<0, 64><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
          } else {
            if (bkt == 0) k_gemm_gen<1, 32><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
            else if (bkt == 1) k_gemm_gen<1, 48><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
            else k_gemm_gen<1, 64><<<g, THREADS, 0, st>>>(tp, db, ws, pts, H->N, H->d, K);
          }
          HH_LAUNCHED();
        }
        base += cnt[bkt];
      }
    };
    mark(0);
    gemm(0, dA, nA);
    mark(1);
    launch_qr(blks, nb, ordq_y, 0, db, ws, st);
    mark(2);
    // Z = A^T Q (and a copy for the R-only QR)
    gemm(1, dB, nB);
    mark(3);
    launch_qr(blks, nb, ordq_z, 1, db, ws, st);
    mark(4);
    {
      // k-buckets: (k <= 32: 256 threads), (<= 64: 512), (<= 96: 512), (<= 168: 1024, smem),
      // (> 168: 1024, global) — small cores get small CTAs / smem so several share an SM
      std::vector<int32_t> ord;
      int cnt[5] = {0, 0, 0, 0, 0}, kmx[5] = {0, 0, 0, 0, 0};
      auto bucket = [](int k) { return k <= 32 ? 0 : k <= 64 ? 1 : k <= 96 ? 2 : k <= JAC_SMEM_K ? 3 : 4; };
      for (int bkt = 0; bkt < 5; ++bkt)
        for (int i = 0; i < nb; ++i)
          if (bucket(blks[i].k) == bkt) {
            ord.push_back(i);
            ++cnt[bkt];
            kmx[bkt] = std::max(kmx[bkt], blks[i].k);
          }
      h2d(ordb, ord, st);
      const int32_t *od = ordb.as<int32_t>();
      int start = 0;
      for (int bkt = 0; bkt < 5; ++bkt) {
        if (cnt[bkt] == 0) continue;
        const int jsm = std::min(kmx[bkt], JAC_SMEM_K);
        const size_t jsmem = bkt == 4 ? 0 : sizeof(double) * (size_t)jsm * jsm;
        if (bkt == 0) {
          k_jacobi<256><<<cnt[bkt], 256, jsmem, st>>>(db, od + start, ws);
        } else if (bkt <= 2) {
          HH_CUDA(cudaFuncSetAttribute(k_jacobi<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 96 * 96)));
          k_jacobi<512><<<cnt[bkt], 512, jsmem, st>>>(db, od + start, ws);
        } else {
          HH_CUDA(cudaFuncSetAttribute(k_jacobi<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * JAC_SMEM_K * JAC_SMEM_K)));
          k_jacobi<1024><<<cnt[bkt], 1024, jsmem, st>>>(db, od + start, ws);
        }
        HH_LAUNCHED();
        start += cnt[bkt];
      }
    }
    mark(5);
    if (!write) {  // pass 2 knows the rank: no residual / decision needed
      k_resid<<<(unsigned)tR.size(), THREADS, 0, st>>>(dR, db, ws, pts, H->N, H->d, K, partb.as<double>());
      HH_LAUNCHED();
      mark(6);
      k_decide<<<(nb + 127) / 128, 128, 0, st>>>(db, nb, ws, partb.as<double>(), H->eps, delta);
      HH_LAUNCHED();
    } else {
      mark(6);
    }
    mark(7);
    Arenas a{};
    if (write) a = *ar;
    k_factors<<<nb, THREADS, 0, st>>>(db, ws, write ? 1 : 0, a);
    HH_LAUNCHED();
    mark(8);
    HH_CUDA(cudaMemcpyAsync(blks.data(), blkb.p, sizeof(CBlk) * nb, cudaMemcpyDeviceToHost, st));
    HH_CUDA(cudaStreamSynchronize(st));
    if (prof) {
      for (int i = 0; i < 8; ++i) {
        float ms = 0;
        HH_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        g_stage_ms[i] += ms;
      }
      ++g_stage_batches;
    }
    for (int i = 0; i < nb; ++i) {
      CompressResult &r = res[pos + i];
      const CBlk &c = blks[i];
      r.p = c.pfound;
      r.k = c.k;
      r.nb2 = c.nb2;
      r.tot = c.tot;
      r.R = c.R;
      r.maxabs = c.maxabs;
      r.ok = c.ok;
    }
    pos = end;
  }
}

}  // namespace hh
