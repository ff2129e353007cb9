// matvec.cu — §8(a) rows a7–a10: the hot path  y = H-hat x  (Alg. 3).
//
//   a7  gather:   v[t] = x[perm[t]]  (tree order, RHS-interleaved)
//   a8  phase 1:  z_b = W_b^T x_J  for every low-rank block — streams the W arenas
//   a9  phase 2:  per leaf R (one owner, fixed order, no atomics):
//                 y_R = sum_dense D_RJ x_J + sum_{levels, tags} U_{R,l,g} z_{l,g}
//   a10 scatter:  fused into the phase-2 epilogue, y[perm[t]] = y~[t]
// "Compute in working precision u": stored fp32/fp16/bf16 values are
// up-converted exactly and accumulated in fp64.
//
// Both phases are persistent kernels with a producer warp that streams 16-B aligned arena
// windows into a shared-memory ring with cp.async.bulk (TMA bulk copies, mbarrier
// complete_tx) and 8 consumer warps that compute from shared memory.
#include <algorithm>
#include <vector>

#include "build.h"

namespace hh {

namespace mv {

constexpr int STAGES = 6;
constexpr int STAGE_BYTES = 16384;
constexpr int NCW = 8;                 // consumer warps
constexpr int THREADS = 32 * (NCW + 1);

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory"); }

template <int TAG>
__device__ __forceinline__ double ld_up(const uint8_t *base, int64_t i) {
  if (TAG == TAG_FP64) return reinterpret_cast<const double *>(base)[i];
  if (TAG == TAG_FP32) return (double)reinterpret_cast<const float *>(base)[i];
  if (TAG == TAG_FP16) return (double)__half2float(reinterpret_cast<const __half *>(base)[i]);
  return (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t *>(base)[i]) << 16);
}

// --------------------------------------------------------------------------- gather
template <int NR>
__global__ void k_gather(const int32_t *__restrict__ perm, const double *__restrict__ x, int64_t N, int64_t ldx,
                         double *__restrict__ v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = perm[t];
#pragma unroll
    for (int r = 0; r < NR; ++r) v[t * NR + r] = x[i + r * ldx];
  }
}

// --------------------------------------------------------------------------- phase 1
struct P1Args {
  const P1Item *items;
  const P1Entry *entries;
  int64_t nitems;
  const uint8_t *W[4];
  double *v;          // [x~ (N) ; z] x NR
  double *partial;    // [slots] x NR
  int64_t N;
};

template <int TAG, int NR>
__device__ __forceinline__ void p1_column(const uint8_t *col, int nrows, const double *__restrict__ xv, int lane,
                                          double (&acc)[NR]) {
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  for (int r = lane; r < nrows; r += 32) {
    const double w = ld_up<TAG>(col, r);
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = __fma_rn(w, __ldg(xv + (int64_t)r * NR + q), acc[q]);
  }
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
}

template <int NR>
__global__ void __launch_bounds__(THREADS) k_phase1(P1Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {  // producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int n = 0;
      for (int64_t it = blockIdx.x; it < a.nitems; it += gridDim.x, ++n) {
        const int s = n % STAGES;
        if (n >= STAGES) mbar_wait(&empty[s], ((n / STAGES) & 1) ^ 1);
        const P1Item I = a.items[it];
        mbar_expect_tx(&full[s], I.nbytes);
        bulk_g2s(smem + s * STAGE_BYTES, a.W[I.tag] + I.src, I.nbytes, &full[s], pol);
      }
    }
    return;
  }
  int n = 0;
  for (int64_t it = blockIdx.x; it < a.nitems; it += gridDim.x, ++n) {
    const int s = n % STAGES;
    const P1Item I = a.items[it];
    mbar_wait(&full[s], (n / STAGES) & 1);
    const uint8_t *stage = smem + s * STAGE_BYTES;
    const int w = tag_bytes(I.tag);
    int gc = 0;  // running column counter inside the item; warp gc % NCW owns column gc
    for (uint32_t e = I.e0; e < I.e1; ++e) {
      const P1Entry E = a.entries[e];
      int c = (warp - gc % NCW + NCW) % NCW;
      for (; c < (int)E.ncols; c += NCW) {
        const uint8_t *col = stage + E.soff + (int64_t)c * E.nrows * w;
        const double *xv = a.v + E.x0 * NR;
        double acc[NR];
        switch (I.tag) {
          case TAG_FP64: p1_column<TAG_FP64, NR>(col, E.nrows, xv, lane, acc); break;
          case TAG_FP32: p1_column<TAG_FP32, NR>(col, E.nrows, xv, lane, acc); break;
          case TAG_FP16: p1_column<TAG_FP16, NR>(col, E.nrows, xv, lane, acc); break;
          default: p1_column<TAG_BF16, NR>(col, E.nrows, xv, lane, acc); break;
        }
        if (lane == 0) {
          double *out = E.out >= 0 ? a.v + (a.N + E.out + c) * NR : a.partial + (~E.out) * NR;
#pragma unroll
          for (int q = 0; q < NR; ++q) out[q] = acc[q];
        }
      }
      gc += E.ncols;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

template <int NR>
__global__ void k_combine(const Combine *__restrict__ cm, int64_t n, const double *__restrict__ partial, double *v,
                          int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Combine C = cm[i];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      double s = 0.0;
      for (int64_t k = C.s0; k < C.s1; ++k) s += partial[k * NR + q];
      v[(N + C.zi) * NR + q] = s;
    }
  }
}

// --------------------------------------------------------------------------- phase 2
struct P2Args {
  const P2Leaf *leaves;
  const P2Chunk *chunks;
  int64_t nleaves;
  const uint8_t *U[4];
  const uint8_t *D;
  const double *v;
  const int32_t *perm;
  double *y;
  int64_t ldy;
};

template <int TAG, int NR>
__device__ __forceinline__ void p2_chunk(const uint8_t *stage, const P2Chunk &C, int nr, int rr, int g, int G,
                                         const double *__restrict__ v, double (&acc)[NR]) {
  const uint8_t *base = stage + C.lead;
  const double *vv = v + C.vbeg * NR;
  for (int c = g; c < (int)C.ncols; c += G) {
    const double u = ld_up<TAG>(base, (int64_t)c * nr + rr);
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = __fma_rn(u, __ldg(vv + (int64_t)c * NR + q), acc[q]);
  }
}

template <int NR>
__global__ void __launch_bounds__(THREADS) k_phase2(P2Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  double *red = reinterpret_cast<double *>(empty + STAGES);  // [NCW*32][NR]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int n = 0;
      for (int64_t li = blockIdx.x; li < a.nleaves; li += gridDim.x) {
        const P2Leaf Lf = a.leaves[li];
        for (int64_t ci = Lf.c0; ci < Lf.c1; ++ci, ++n) {
          const int s = n % STAGES;
          if (n >= STAGES) mbar_wait(&empty[s], ((n / STAGES) & 1) ^ 1);
          const P2Chunk C = a.chunks[ci];
          mbar_expect_tx(&full[s], C.nbytes);
          const uint8_t *src = (C.dense ? a.D : a.U[C.tag]) + C.src;
          bulk_g2s(smem + s * STAGE_BYTES, src, C.nbytes, &full[s], pol);
        }
      }
    }
    return;
  }
  const int tid = threadIdx.x;  // 0 .. NCW*32-1
  int n = 0;
  for (int64_t li = blockIdx.x; li < a.nleaves; li += gridDim.x) {
    const P2Leaf Lf = a.leaves[li];
    const int nr = Lf.nr;
    const int G = (NCW * 32) / nr;  // nr <= 256 (leaf_size limit)
    const int rr = tid % nr, g = tid / nr;
    const bool active = g < G;
    double acc[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = 0.0;
    for (int64_t ci = Lf.c0; ci < Lf.c1; ++ci, ++n) {
      const int s = n % STAGES;
      const P2Chunk C = a.chunks[ci];
      mbar_wait(&full[s], (n / STAGES) & 1);
      const uint8_t *stage = smem + s * STAGE_BYTES;
      if (active) {
        switch (C.tag) {
          case TAG_FP64: p2_chunk<TAG_FP64, NR>(stage, C, nr, rr, g, G, a.v, acc); break;
          case TAG_FP32: p2_chunk<TAG_FP32, NR>(stage, C, nr, rr, g, G, a.v, acc); break;
          case TAG_FP16: p2_chunk<TAG_FP16, NR>(stage, C, nr, rr, g, G, a.v, acc); break;
          default: p2_chunk<TAG_BF16, NR>(stage, C, nr, rr, g, G, a.v, acc); break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // fixed-order reduction over column groups, then scatter y[perm[t]] (a10)
#pragma unroll
    for (int q = 0; q < NR; ++q) red[tid * NR + q] = acc[q];
    consumer_sync();
    if (tid < nr) {
      double s[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) s[q] = 0.0;
      for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int q = 0; q < NR; ++q) s[q] += red[(gg * nr + tid) * NR + q];
      const int64_t i = a.perm[Lf.r0 + tid];
#pragma unroll
      for (int q = 0; q < NR; ++q) a.y[i + q * a.ldy] = s[q];
    }
    consumer_sync();
  }
}

}  // namespace mv

size_t p1_smem() { return mv::STAGES * mv::STAGE_BYTES + 2 * mv::STAGES * sizeof(uint64_t); }
size_t p2_smem(int nr) {
  return mv::STAGES * mv::STAGE_BYTES + 2 * mv::STAGES * sizeof(uint64_t) + sizeof(double) * mv::NCW * 32 * nr;
}

template <int NR>
void matvec_chunk(hh_matrix *H, const double *x, double *y, int col0, cudaStream_t st) {
  using namespace mv;
  int dev = 0, nsm = 148;
  HH_CUDA(cudaGetDevice(&dev));
  HH_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double *v = H->v.as<double>();
  cudaEvent_t ev[4];
  auto mark = [&](int i) {
    if (!H->prof) return;
    HH_CUDA(cudaEventCreate(&ev[i]));
    HH_CUDA(cudaEventRecord(ev[i], st));
    H->prof_ev.push_back(ev[i]);
  };
  mark(0);
  // a7 gather
  k_gather<NR><<<nsm * 8, 256, 0, st>>>(H->d_perm.as<int32_t>(), x + (int64_t)col0 * H->N, H->N, H->N, v);
  HH_LAUNCHED();
  mark(1);
  // a8 phase 1
  if (H->n_p1_items > 0) {
    P1Args a{};
    a.items = H->p1_items.as<P1Item>();
    a.entries = H->p1_entries.as<P1Entry>();
    a.nitems = H->n_p1_items;
    for (int g = 0; g < 4; ++g) a.W[g] = H->W[g].as<uint8_t>();
    a.v = v;
    a.partial = H->partial.as<double>();
    a.N = H->N;
    const size_t sm = p1_smem();
    static bool attr1[17] = {};
    if (!attr1[NR]) {
      HH_CUDA(cudaFuncSetAttribute(k_phase1<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr1[NR] = true;
    }
    int per_sm = 0;
    HH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phase1<NR>, THREADS, sm));
    const int64_t grid = std::min<int64_t>(H->n_p1_items, (int64_t)nsm * std::max(1, per_sm));
    k_phase1<NR><<<(unsigned)grid, THREADS, sm, st>>>(a);
    HH_LAUNCHED();
    if (H->n_combines > 0) {
      k_combine<NR><<<nsm * 4, 256, 0, st>>>(H->combines.as<Combine>(), H->n_combines, H->partial.as<double>(), v, H->N);
      HH_LAUNCHED();
    }
  }
  mark(2);
  // a9 + a10 phase 2 with fused scatter
  P2Args b{};
  b.leaves = H->p2_leaves.as<P2Leaf>();
  b.chunks = H->p2_chunks.as<P2Chunk>();
  b.nleaves = H->n_p2_leaves;
  for (int g = 0; g < 4; ++g) b.U[g] = H->U[g].as<uint8_t>();
  b.D = H->D.as<uint8_t>();
  b.v = v;
  b.perm = H->d_perm.as<int32_t>();
  b.y = y + (int64_t)col0 * H->N;
  b.ldy = H->N;
  const size_t sm2 = p2_smem(NR);
  static bool attr2[17] = {};
  if (!attr2[NR]) {
    HH_CUDA(cudaFuncSetAttribute(k_phase2<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    attr2[NR] = true;
  }
  int per_sm2 = 0;
  HH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_phase2<NR>, THREADS, sm2));
  const int64_t grid2 = std::min<int64_t>(H->n_p2_leaves, (int64_t)nsm * std::max(1, per_sm2));
  if (grid2 > 0) {
    k_phase2<NR><<<(unsigned)grid2, THREADS, sm2, st>>>(b);
    HH_LAUNCHED();
  }
  mark(3);
}

void run_matvec(hh_matrix *H, const double *x, double *y, int nrhs, cudaStream_t st) {
  int col = 0;
  while (col < nrhs) {
    const int rem = nrhs - col;
    if (rem >= 16) {
      matvec_chunk<16>(H, x, y, col, st);
      col += 16;
    } else if (rem >= 8) {
      matvec_chunk<8>(H, x, y, col, st);
      col += 8;
    } else if (rem >= 4) {
      matvec_chunk<4>(H, x, y, col, st);
      col += 4;
    } else if (rem >= 2) {
      matvec_chunk<2>(H, x, y, col, st);
      col += 2;
    } else {
      matvec_chunk<1>(H, x, y, col, st);
      col += 1;
    }
  }
}

}  // namespace hh
