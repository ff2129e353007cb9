// matvec.cu — §8(a) rows a7–a10: the hot path  y = H-hat x  (Alg. 3).
//
//   a7  gather:   v[t] = x[perm[t]]  (tree order, RHS-interleaved); also zeroes the work
//                 counters of the two persistent kernels
//   a8  phase 1:  z_b = W_b^T x_J for every low-rank block.  W is stored as per-source
//                 panels: for a source cluster J all blocks b with src J form
//                 one |J| x P_J matrix, cut into column tiles of <= 248 columns stored
//                 row-major.  One work item = one tile (tiles taller than 4096 rows: one
//                 row piece, summed by a fixed-order combine pass); thread c of the CTA owns
//                 tile column c and accumulates it over the rows.
//   a9  phase 2:  per leaf R (one owner, fixed order, no atomics):
//                 y_R = sum_dense D_RJ x_J + sum_{tags, levels} U_{R,l,g} z_{l,g}
//   a10 scatter:  fused into the phase-2 epilogue, y[perm[t]] = y~[t]
// "Compute in working precision u": stored fp32/fp16/bf16 values are
// up-converted exactly and accumulated in fp64.
//
// Both phases are persistent kernels (grid = resident CTAs) that take work items from a
// counter.  One producer thread streams each item through a ring of shared-memory stages
// with cp.async.bulk (TMA bulk copies completing on an mbarrier): the factor window (<= 32
// KiB) AND the matching vector slice (x~ rows for phase 1, z entries for phase 2) plus a
// small descriptor, so the 8 consumer warps never touch global memory in their inner loops.
// Consumers: fp64 FMA (DFMA) at NR = 1, 2, 4; FP64 tensor cores (DMMA) at NR = 8, 16.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "build.h"

namespace hh {

namespace mv {

#ifndef HH_MV_NCW
#define HH_MV_NCW 8
#endif
constexpr int NCW = HH_MV_NCW;         // consumer warps
constexpr int NCT = NCW * 32;          // consumer threads
constexpr int THREADS = NCT + 32;      // + one producer warp
#ifndef HH_MV_MINB
#define HH_MV_MINB 1
#endif
// Stage geometry.  Measured on B200 (profiles/r01_variants.txt): fewer, larger stages with
// more CTAs per SM win — 2 stages of 32 KiB factor data at 3 CTAs/SM for NR <= 2; the
// FP64-bound multi-RHS kernels size the vector slice per phase (see Geo).
#ifndef HH_MV_WDATA
#define HH_MV_WDATA 32768
#endif
#ifndef HH_MV_XDATA
#define HH_MV_XDATA 4096
#endif
#ifndef HH_MV_P2HI
#define HH_MV_P2HI 28672   // phase 2 at NR = 16: 28 KiB factor + 28 KiB z stages, 2 CTAs/SM (measured)
#endif
#ifndef HH_MV_P1HI
#define HH_MV_P1HI 49152  // phase-1 factor bytes per stage at NR = 16 (48 KiB + 8 KiB x~, 2 CTAs/SM, measured)
#endif
#ifndef HH_MV_P1X
#define HH_MV_P1X 8192  // phase-1 x~ bytes per stage at NR = 16 (0: max(NR * 512, 4096))
#endif
#ifndef HH_MV_STAGES
#define HH_MV_STAGES 2
#endif
#ifndef HH_MV_P2STAGES
#define HH_MV_P2STAGES HH_MV_STAGES  // phase-2 ring depth at NR = 16
#endif
#ifndef HH_MV_P2X
#define HH_MV_P2X 28672  // phase-2 z bytes per stage at NR = 16 (0: NR * 2048 / (32768 / P2HI))
#endif
// DMMA K-loops without per-step bounds checks (tail step peeled): measured ~1% faster in
// phase 1, ~2% slower in phase 2 (profiles/r01_variants.txt)
#ifndef HH_MV_P2ALIAS
#define HH_MV_P2ALIAS 1  // phase 2 at NR = 16: the leaf-end reduction reuses the leaf's last stage
#endif
#ifndef HH_MV_PEEL1
#define HH_MV_PEEL1 1
#endif
#ifndef HH_MV_PEEL2
#define HH_MV_PEEL2 0
#endif
constexpr int META = 64;
#ifndef HH_MV_PDL
#define HH_MV_PDL 1  // programmatic dependent launch between the matvec kernels
#endif
#ifndef HH_MV_P2MORTON_NR
#define HH_MV_P2MORTON_NR 8  // phase-2 leaves in Morton order from this RHS width up (z locality in L2)
#endif
#ifndef HH_MV_P2RED
#define HH_MV_P2RED 1  // NR = 1 leaf-end reduction: 0 = one thread per row slot, 1 = lanes per row + shuffles (measured: 1 is 4% faster on the sphere set, neutral elsewhere)
#endif
#ifndef HH_MV_VEC1
#define HH_MV_VEC1 1  // NR = 1 consumers with vector factor loads (0: the round-1 scalar consumers)
#endif

// K-quartered stages for the DMMA consumers (NR = 8, 16).  A DMMA K-step takes four K
// indices, one per lane group kq = lane % 4.  With the window staged as one linear copy the
// four indices are consecutive, so the four kq lanes of a fragment load addresses one
// row (x~ / z: NR * 8 B = 128 B at NR = 16) or one U column (|R| * w B, 128 B for a 32-point
// fp32 leaf) apart — the same shared-memory banks, a 4-way conflict on every fragment load
// (ncu r02f, proxy at 16 RHS: 180 M of 270 M phase-2 wavefronts were conflict replays, the
// LSU pipe 69% busy next to a 75% busy DMMA pipe).  Instead the producer cuts each window's
// K range into four quarters, copies each with its own bulk copy to a shared-memory region
// whose start is skewed by 32 B (8 banks) per quarter, and lane group kq walks quarter kq:
// the four lanes of a fragment row then sit 8 banks apart, the eight rows fill the gaps.
// MEASURED (profiles/r02h_ab_quart_geom.txt, r02h_proxy_nrhs16_quart_ncu.txt): the replays
// disappear (phase-2 wavefronts 270 M -> 91 M, phase 1 172 M -> 73 M) but the kernels do not get
// faster — phase 1 unchanged, phase 2 5-15% slower (eight bulk copies and 7% fewer columns per
// stage, more index arithmetic): the DMMA pipe (83% / 75% issue-busy), not shared memory, is
// the limit.  Kept as an opt-in variant; the default is the linear window.
#ifndef HH_MV_QUART
#define HH_MV_QUART 0
#endif
// byte stride between the quarter regions of a stage: room for the quarter's enclosing 16-B
// aligned window, rounded to the 128-B bank period, plus the 32-B skew
__host__ __device__ constexpr int quarter_stride(int qbytes) { return ((qbytes + 32 + 127) & ~127) + 32; }
// largest quarter (bytes) whose four regions fit a buffer of BUF bytes
constexpr int quarter_max_bytes(int buf) { return ((buf / 4 - 32) / 128) * 128 - 32; }

// FP64 tensor-core (DMMA m8n8k4) consumers for the multi-RHS contractions (NR = 8, 16):
// the phase-1 tile is then D = W^T X (ct x NR) and the phase-2 leaf Y = U Z (nr x NR).
#ifndef HH_MV_MMA
#define HH_MV_MMA 1
#endif
template <int NR> constexpr bool use_mma() { return HH_MV_MMA && (NR == 8 || NR == 16); }
// resident CTAs per SM the register allocation must allow: the DMMA kernels are sized (shared
// memory) for two, which 9 warps reach only at <= 96 registers per thread
// (phase 1 at NR = 8 has 74 KiB of stages: three CTAs, <= 72 registers)
template <int NR, int PH> constexpr int min_ctas() { return use_mma<NR>() ? (NR == 8 && PH == 1 ? 3 : 2) : HH_MV_MINB; }
template <int NR, int WP = 0> constexpr bool quartered() { return HH_MV_QUART && WP == 0 && use_mma<NR>(); }

// Precomputed stage plan for the single-RHS fp64 product (handle.h StageCopy / StageMeta /
// StageItem; built by layout.cpp build_stage_plan): the producer only issues copies.  0 = the
// on-the-fly producer at NR = 1 too (variant builds, A/B).
#ifndef HH_MV_DESC
#define HH_MV_DESC 1
#endif
template <int NR, int WP = 0> constexpr bool planned() { return HH_MV_DESC && NR == 1 && WP == 0; }

// GV = stage geometry variant of the planned product (kStageGeo[GV], chosen per handle and phase)
template <int NR, int PH, int GV = 0> struct Geo {  // PH = phase (1: x~ rows per W row window, 2: z per U column)
  static_assert(GV == 0 || (NR == 1 && HH_MV_DESC), "geometry variants belong to the planned single-RHS product");
  // factor bytes per stage (phase 2 at NR >= 8 may use smaller stages to fit 2 CTAs/SM)
  static constexpr int WDATA = (NR == 1 && HH_MV_DESC) ? kStageGeo[GV].wdata
                               : (PH == 2 && NR >= 16) ? HH_MV_P2HI : (PH == 1 && NR >= 16) ? HH_MV_P1HI : HH_MV_WDATA;
  static constexpr int WBUF = WDATA + 32;                            // + 16-B alignment slack
  // vector bytes per stage: phase 1 needs one NR-vector per W row (a 248-column row is >= 1 KiB
  // of factors), phase 2 one per U column (|R| rows, as little as ~32 elements)
  static constexpr int XDATA =
      (NR == 1 && HH_MV_DESC) ? kStageGeo[GV].xelems * 8
      : NR <= 2 ? HH_MV_XDATA
              : (PH == 1 ? ((NR >= 16 && HH_MV_P1X > 0) ? HH_MV_P1X : (NR * 512 > 4096 ? NR * 512 : 4096))
                         : ((NR >= 16 && HH_MV_P2X > 0) ? HH_MV_P2X : NR * 2048 / (32768 / WDATA)));
  static constexpr int XELEMS = XDATA / 8;                        // doubles (rows x NR)
  static constexpr int XBUF = XDATA + 32;
  static constexpr int STAGE = WBUF + XBUF + META;
  static constexpr int STAGES = (NR == 1 && HH_MV_DESC) ? kStageGeo[GV].stages
                                : (PH == 2 && NR >= 16) ? HH_MV_P2STAGES : HH_MV_STAGES;
  // phase 2 at NR = 16 may reduce in the leaf's last stage (held until the reduction ends)
  static constexpr bool RED_IN_STAGE = PH == 2 && NR >= 16 && HH_MV_P2ALIAS && use_mma<NR>();
  static constexpr size_t red_bytes() {  // phase-2 cross-group reduction buffer
    return use_mma<NR>() ? sizeof(double) * NCW * 4 * (NR / 8) * 32 * 2 : sizeof(double) * NCT * NR * (NR >= 8 ? 2 : 1);
  }
  static constexpr size_t smem(bool red) {
    return (size_t)STAGES * STAGE + 2 * STAGES * sizeof(uint64_t) + (red && !RED_IN_STAGE ? red_bytes() : 0);
  }
};

// Stage descriptor the consumers read from the stage's last 64 bytes (handle.h StageMeta):
// written by the producer thread, or delivered by a bulk copy from the precomputed stage plan.
using Meta = StageMeta;
static_assert(sizeof(Meta) <= META, "meta");

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }
// Programmatic dependent launch: the matvec kernels are launched so that the next one's CTAs
// may be scheduled while the previous one drains (its launch latency and prologue overlap the
// tail); every kernel waits for its predecessor's completion (and memory) before its first
// global access, so the data dependencies are those of plain stream order.
__device__ __forceinline__ void pdl_wait() {
#if HH_MV_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if HH_MV_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Cycle probe of the NR = 1 pipelines (variant builds only, -DHH_MV_PROBE=1; the product build
// compiles none of it): where do the producer thread and a consumer thread spend their time?
// Slots (summed over CTAs): phase p in {1, 2} at base 8 (p - 1):
//   +0 producer cycles in its item loop   +1 of which waiting on empty barriers   +2 stages issued
//   +3 consumer (thread 0) cycles          +4 of which waiting on full barriers    +5 in item-end sections
//   +6 items
#ifndef HH_MV_PROBE
#define HH_MV_PROBE 0
#endif
#if HH_MV_PROBE
__device__ unsigned long long g_probe[16];
__device__ __forceinline__ unsigned long long pclk() { return clock64(); }
#define PROBE(stmt) stmt
#else
#define PROBE(stmt)
#endif

// Copy [src, src + bytes) as the enclosing 16-B aligned window; returns the lead offset.
__device__ __forceinline__ int stage_copy(uint8_t *dst, const uint8_t *src, int64_t bytes, uint64_t *bar,
                                          uint64_t pol, uint32_t &tx) {
  const uintptr_t s = (uintptr_t)src, sa = s & ~(uintptr_t)15, ea = (s + bytes + 15) & ~(uintptr_t)15;
  if (bytes > 0) {
    bulk_g2s(dst, (const void *)sa, (uint32_t)(ea - sa), bar, pol);
    tx += (uint32_t)(ea - sa);
  }
  return (int)(s - sa);
}
// arena base by tag without dynamic indexing of the kernel-parameter array (no local memory)
__device__ __forceinline__ const uint8_t *pick(const uint8_t *const (&arr)[NTAG], int t) {
  return t == 0 ? arr[0] : t == 1 ? arr[1] : t == 2 ? arr[2] : t == 3 ? arr[3] : t == 4 ? arr[4] : t == 5 ? arr[5] : arr[6];
}
__device__ __forceinline__ uint32_t window_bytes(const uint8_t *src, int64_t bytes) {
  const uintptr_t s = (uintptr_t)src;
  return bytes > 0 ? (uint32_t)(((s + bytes + 15) & ~(uintptr_t)15) - (s & ~(uintptr_t)15)) : 0u;
}

template <int TAG> struct Elem;
template <> struct Elem<TAG_FP64> { using T = double; };
template <> struct Elem<TAG_FP32> { using T = float; };
template <> struct Elem<TAG_FP16> { using T = __half; };
template <> struct Elem<TAG_BF16> { using T = uint16_t; };
template <> struct Elem<TAG_Q43> { using T = uint8_t; };
// accessor formats (NEXT-3): the top 3 bytes of an fp32 / top 6 bytes of an fp64
struct B24 { uint8_t b[3]; };
struct B48 { uint16_t h[3]; };
static_assert(sizeof(B24) == 3 && sizeof(B48) == 6, "packed accessor elements");
template <> struct Elem<TAG_BF24> { using T = B24; };
template <> struct Elem<TAG_FP48> { using T = B48; };

// f(std::integral_constant<int, TAG>) for the runtime tag (one branch per storage format)
template <class F>
__device__ __forceinline__ void dispatch_tag(int tag, F &&f) {
  switch (tag) {
    case TAG_FP64: f(std::integral_constant<int, TAG_FP64>{}); break;
    case TAG_FP32: f(std::integral_constant<int, TAG_FP32>{}); break;
    case TAG_FP16: f(std::integral_constant<int, TAG_FP16>{}); break;
    case TAG_BF16: f(std::integral_constant<int, TAG_BF16>{}); break;
    case TAG_Q43: f(std::integral_constant<int, TAG_Q43>{}); break;
    case TAG_BF24: f(std::integral_constant<int, TAG_BF24>{}); break;
    default: f(std::integral_constant<int, TAG_FP48>{}); break;
  }
}

// Tunables (compile-time; scripts/variants.sh builds alternatives side by side).
#ifndef HH_MV_CVT
#define HH_MV_CVT 0      // 0: F2F conversion; 1: bit placement + exact power-of-two DMUL
#endif

// exact up-conversion of a stored element to fp64
template <int TAG>
__device__ __forceinline__ double up(const typename Elem<TAG>::T v) {
  if constexpr (TAG == TAG_FP64) {
    return v;
  } else if constexpr (TAG == TAG_BF24) {  // 1-8-15: the bytes are the top 24 bits of an fp32
    const uint32_t b = (uint32_t)v.b[0] | ((uint32_t)v.b[1] << 8) | ((uint32_t)v.b[2] << 16);
    return (double)__uint_as_float(b << 8);
  } else if constexpr (TAG == TAG_FP48) {  // 1-11-36: the top 48 bits of an fp64
    const uint64_t b = (uint64_t)v.h[0] | ((uint64_t)v.h[1] << 16) | ((uint64_t)v.h[2] << 32);
    return __longlong_as_double((long long)(b << 16));
  } else if constexpr (TAG == TAG_Q43) {
    // q43 byte s|eeee|mmm (bias 7) placed in an fp16's top bits (exponent field 0eeee, mantissa
    // mmm0000000) is the same value scaled by 2^-8, normals and subnormals alike: exact
    const uint32_t b = v;
    return (double)__half2float(__ushort_as_half((unsigned short)(((b & 0x80u) << 8) | ((b & 0x7Fu) << 7)))) * 256.0;
  } else if constexpr (HH_MV_CVT == 1) {
    // place sign / exponent / mantissa bits in an fp64 with the same (unbiased-shifted)
    // exponent field, then rescale by the exact power of two between the two biases
    // (normals, subnormals and zeros are all exact; factors are finite by construction)
    if constexpr (TAG == TAG_FP32) {
      const uint32_t b = __float_as_uint(v);
      return __hiloint2double((int)((b & 0x80000000u) | ((b & 0x7FFFFFFFu) >> 3)), (int)(b << 29)) * 0x1p896;
    } else if constexpr (TAG == TAG_FP16) {
      const uint32_t h = __half_as_ushort(v);
      return __hiloint2double((int)(((h & 0x8000u) << 16) | ((h & 0x7FFFu) << 10)), 0) * 0x1p1008;
    } else {
      const uint32_t h = v;
      return __hiloint2double((int)(((h & 0x8000u) << 16) | ((h & 0x7FFFu) << 13)), 0) * 0x1p896;
    }
  } else {
    if constexpr (TAG == TAG_FP32) return (double)v;
    else if constexpr (TAG == TAG_FP16) return (double)__half2float(v);
    else return (double)__uint_as_float(((uint32_t)v) << 16);
  }
}

// D = A B + D on the FP64 tensor cores: A 8x4 (thread holds A[lane/4][lane%4]), B 4x8
// (thread holds B[lane%4][lane/4]), C/D 8x8 (thread holds row lane/4, columns 2(lane%4)+{0,1}).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Producer of the planned single-RHS product: items from the work counter, for every stage of
// the item three bulk copies (factor window, vector window, 64-B descriptor) completing on the
// stage's full barrier.  The next item record and the next copy record are loaded one ahead.
struct PlanArgs {
  const StageItem *items;
  const StageCopy *copies;
  const StageMeta *metas;
};
__device__ __forceinline__ StageCopy load_copy(const StageCopy *p) {
  const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p)), b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
  StageCopy c;
  c.wsrc = (uint64_t)a.x | ((uint64_t)a.y << 32);
  c.xsrc = (uint64_t)a.z | ((uint64_t)a.w << 32);
  c.wbytes = b.x;
  c.xbytes = b.y;
  return c;
}
template <class G, int PH>
__device__ __forceinline__ void planned_producer(const PlanArgs &pl, int64_t nitems, int *ctr, uint8_t *smem,
                                                 uint64_t *full, uint64_t *empty) {
  const uint64_t pol_w = evict_first_policy(), pol_x = evict_last_policy();
  int n = 0;
  PROBE(unsigned long long pt0 = pclk(); unsigned long long pwait = 0; unsigned long long pitems = 0;)
  int item = atomicAdd(ctr, 1);
  int64_t s0n = 0, s1n = 0;
  StageCopy cn{};
  if (item < nitems) {
    const uint4 r = __ldg(reinterpret_cast<const uint4 *>(pl.items + item));
    s0n = (int64_t)((uint64_t)r.x | ((uint64_t)r.y << 32));
    s1n = (int64_t)((uint64_t)r.z | ((uint64_t)r.w << 32));
    cn = load_copy(&pl.items[item].first);
  }
  while (item < nitems) {
    const int64_t s0 = s0n, s1 = s1n;
    StageCopy c = cn;
    const int nxt = atomicAdd(ctr, 1);
    if (nxt < nitems) {
      const uint4 r = __ldg(reinterpret_cast<const uint4 *>(pl.items + nxt));
      s0n = (int64_t)((uint64_t)r.x | ((uint64_t)r.y << 32));
      s1n = (int64_t)((uint64_t)r.z | ((uint64_t)r.w << 32));
      cn = load_copy(&pl.items[nxt].first);
    }
    StageCopy c1{};
    if (s0 + 1 < s1) c1 = load_copy(pl.copies + s0 + 1);
    PROBE(++pitems;)
    for (int64_t si = s0; si < s1; ++si, ++n) {
      const int s = n % G::STAGES;
      PROBE(const unsigned long long w0 = pclk();)
      if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
      PROBE(pwait += pclk() - w0;)
      uint8_t *st = smem + s * G::STAGE;
      mbar_expect_tx(&full[s], c.wbytes + c.xbytes + (uint32_t)sizeof(StageMeta));
      if (c.wbytes) bulk_g2s(st, reinterpret_cast<const void *>(c.wsrc), c.wbytes, &full[s], pol_w);
      if (c.xbytes) bulk_g2s(st + G::WBUF, reinterpret_cast<const void *>(c.xsrc), c.xbytes, &full[s], pol_x);
      bulk_g2s(st + G::WBUF + G::XBUF, pl.metas + si, (uint32_t)sizeof(StageMeta), &full[s], pol_w);
      c = c1;
      if (si + 2 < s1) c1 = load_copy(pl.copies + si + 2);
    }
    item = nxt;
  }
  PROBE(atomicAdd(&g_probe[8 * (PH - 1)], pclk() - pt0); atomicAdd(&g_probe[8 * (PH - 1) + 1], pwait);
        atomicAdd(&g_probe[8 * (PH - 1) + 2], (unsigned long long)n); atomicAdd(&g_probe[8 * (PH - 1) + 6], pitems);)
  const int s = n % G::STAGES;
  if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
  reinterpret_cast<Meta *>(smem + s * G::STAGE + G::WBUF + G::XBUF)->kind = 1;
  mbar_arrive(&full[s]);
}

// --------------------------------------------------------------------------- working precision
// Alg. 3 "compute in working precision u" with u below fp64 — the paper's
// backward-error study (Thm 4.4).  Reading G27: x and every
// stored factor / dense entry enter rounded once (RNE) to the working format; every
// multiply-add is one FMA rounded to it; partial sums, z and the cross-thread reductions are
// held in it; y returns its working-precision values as fp64.  WP 0 = fp64 is the product path
// (the code below reduces to it exactly), 1 = fp32 (FFMA), 2 = fp16 (HFMA).
template <int WP> struct WpT;
template <> struct WpT<0> { using A = double; };
template <> struct WpT<1> { using A = float; };
template <> struct WpT<2> { using A = __half; };

template <class A> __device__ __forceinline__ A wp_round(double v) {
  if constexpr (std::is_same_v<A, double>) return v;
  else if constexpr (std::is_same_v<A, float>) return __double2float_rn(v);
  else return __double2half(v);  // cvt.rn.f16.f64: one RNE rounding
}
template <class A> __device__ __forceinline__ double wp_out(A v) {
  if constexpr (std::is_same_v<A, __half>) return (double)__half2float(v);
  else return (double)v;
}
template <class A> __device__ __forceinline__ A wp_zero() {
  if constexpr (std::is_same_v<A, __half>) return __ushort_as_half((unsigned short)0);
  else return A(0);
}
template <class A> __device__ __forceinline__ A wp_fma(A a, A b, A c) {
  if constexpr (std::is_same_v<A, double>) return __fma_rn(a, b, c);
  else if constexpr (std::is_same_v<A, float>) return __fmaf_rn(a, b, c);
  else return __hfma(a, b, c);
}
template <class A> __device__ __forceinline__ A wp_add(A a, A b) {
  if constexpr (std::is_same_v<A, double>) return a + b;
  else if constexpr (std::is_same_v<A, float>) return __fadd_rn(a, b);
  else return __hadd(a, b);
}
// a stored element of format TAG as a working-precision operand (one RNE rounding when the
// storage format is wider than the working one; exact otherwise)
template <int TAG, class A> __device__ __forceinline__ A wp_elem(const typename Elem<TAG>::T v) {
  if constexpr (std::is_same_v<A, double>) {
    return up<TAG>(v);
  } else if constexpr (std::is_same_v<A, float>) {
    if constexpr (TAG == TAG_FP64) return __double2float_rn(v);
    else if constexpr (TAG == TAG_FP32) return v;
    else if constexpr (TAG == TAG_FP16) return __half2float(v);
    else if constexpr (TAG == TAG_BF16) return __uint_as_float(((uint32_t)v) << 16);
    else if constexpr (TAG == TAG_FP48) return __double2float_rn(up<TAG>(v));
    else return (float)up<TAG>(v);  // q43, bf24: exact in fp32
  } else {
    if constexpr (TAG == TAG_FP64) return __double2half(v);
    else if constexpr (TAG == TAG_FP32) return __float2half_rn(v);
    else if constexpr (TAG == TAG_FP16) return v;
    else if constexpr (TAG == TAG_BF16) return __float2half_rn(__uint_as_float(((uint32_t)v) << 16));
    else if constexpr (TAG == TAG_BF24) return __float2half_rn((float)up<TAG>(v));
    else if constexpr (TAG == TAG_FP48) return __double2half(up<TAG>(v));
    else {
      const uint32_t b = v;  // q43 values are exact in fp16: bit placement then x 2^8
      return __hmul(__ushort_as_half((unsigned short)(((b & 0x80u) << 8) | ((b & 0x7Fu) << 7))),
                    __ushort_as_half((unsigned short)0x5C00u));
    }
  }
}

// --------------------------------------------------------------------------- gather
template <int NR, int WP = 0>
__global__ void k_gather(const int32_t *__restrict__ perm, const double *__restrict__ x, int64_t N, int64_t ldx,
                         double *__restrict__ v, int *ctr) {
  using A = typename WpT<WP>::A;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x < 2) ctr[threadIdx.x] = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = perm[t];
#pragma unroll
    for (int r = 0; r < NR; ++r) v[t * NR + r] = wp_out<A>(wp_round<A>(x[i + r * ldx]));
  }
}

// a8 (second pass for row-split tiles): z = sum over pieces in piece order (deterministic)
template <int NR, int WP = 0>
__global__ void k_p1_combine(const P1Combine *__restrict__ cm, int64_t ncomb, const int32_t *__restrict__ zmap,
                             const double *__restrict__ partial, double *v, int64_t N) {
  using A = typename WpT<WP>::A;
  pdl_wait();
  pdl_trigger();
  for (int64_t t = blockIdx.x; t < ncomb; t += gridDim.x) {
    const P1Combine C = cm[t];
    for (int c = threadIdx.x; c < C.ct; c += blockDim.x) {
      A s[NR];
#pragma unroll
      for (int k = 0; k < NR; ++k) s[k] = wp_zero<A>();
      for (int q = 0; q < C.npieces; ++q)
#pragma unroll
        for (int k = 0; k < NR; ++k) s[k] = wp_add(s[k], wp_round<A>(partial[(C.pbase + (int64_t)q * C.ct + c) * NR + k]));
      double *out = v + (N + zmap[C.zbase + c]) * NR;
#pragma unroll
      for (int k = 0; k < NR; ++k) out[k] = wp_out<A>(s[k]);
    }
  }
}

// --------------------------------------------------------------------------- phase 1
struct P1Args {
  const P1Tile *tiles;
  const int32_t *zmap;
  double *partial;    // [npartial] x NR partial column sums of row-split tiles
  int64_t ntiles;
  const uint8_t *W[NTAG];
  double *v;          // [x~ (N) ; z] x NR
  int64_t N;
  int *ctr;
  PlanArgs plan;      // planned single-RHS product only
};

// Register blocking: at NR >= 8 each thread owns MB = 2 factor columns (phase 1) or rows
// (phase 2), so every vector entry loaded from shared memory feeds 2 * NR fp64 FMAs.
template <int NR> constexpr int mblock() { return NR >= 8 ? 2 : 1; }

// Strided dot-accumulate over the cnt indices j this thread owns:
//   acc[b][k] += up(e[j * es + b * eo]) * v[j * vs + k]      (b < MB with valid[b])
// One fixed summation order per (b, k) => bitwise reproducible.
template <int TAG, int NR, int MB, class A = double>
__device__ __forceinline__ void block_acc(const typename Elem<TAG>::T *e, const double *v, int cnt, int es, int eo,
                                          int vs, const bool (&valid)[MB], A (&acc)[MB][NR]) {
#pragma unroll 2
  for (int j = 0; j < cnt; ++j) {
    A a[MB];
#pragma unroll
    for (int b = 0; b < MB; ++b) a[b] = valid[b] ? wp_elem<TAG, A>(e[b * eo]) : wp_zero<A>();
    if constexpr (NR % 2 == 0) {  // 16-B aligned vector entries (NR * 8 bytes per index)
      const double2 *v2 = reinterpret_cast<const double2 *>(v);
#pragma unroll
      for (int k2 = 0; k2 < NR / 2; ++k2) {
        const double2 xv = v2[k2];
        const A x0 = wp_round<A>(xv.x), x1 = wp_round<A>(xv.y);  // exact: v holds working-precision values
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          acc[b][2 * k2] = wp_fma(a[b], x0, acc[b][2 * k2]);
          acc[b][2 * k2 + 1] = wp_fma(a[b], x1, acc[b][2 * k2 + 1]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        const A xk = wp_round<A>(v[k]);
#pragma unroll
        for (int b = 0; b < MB; ++b) acc[b][k] = wp_fma(a[b], xk, acc[b][k]);
      }
    }
    e += es;
    v += vs;
  }
}

// Phase-1 DMMA consumer (NR = 8, 16): warp w owns tile columns [32w, 32w + 32) as four
// 8-column M-tiles; each 4-row K-step does 4 x NR/8 DMMAs.  Accumulators persist over the
// tile's row windows; z is written at the last one.
template <int TAG, int NR, int MT>
__device__ __forceinline__ void p1_mma_rows_t(const uint8_t *wst, const double *xst, int nrows, int ct, int col0,
                                              int lane, double (&c)[4][NR / 8][2]) {
  using T = typename Elem<TAG>::T;
  const T *W = reinterpret_cast<const T *>(wst);
  const int kq = lane & 3, mq = lane >> 2;
  bool cv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) cv[mt] = col0 + mt * 8 + mq < ct;
  int k0 = 0;
#if HH_MV_PEEL1
  if (col0 + MT * 8 <= ct) {
    const int kfull = nrows & ~3;
#pragma unroll 2
    for (; k0 < kfull; k0 += 4) {
      const int row = k0 + kq;
      double b[NR / 8];
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) b[nt] = xst[row * NR + nt * 8 + mq];
      const T *wrow = W + row * ct + col0 + mq;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double av = up<TAG>(wrow[mt * 8]);
#pragma unroll
        for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
      }
    }
  }
#endif
#pragma unroll 2
  for (; k0 < nrows; k0 += 4) {
    const int row = k0 + kq;
    const bool rv = row < nrows;
    double b[NR / 8];
#pragma unroll
    for (int nt = 0; nt < NR / 8; ++nt) b[nt] = rv ? xst[row * NR + nt * 8 + mq] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double av = (rv && cv[mt]) ? up<TAG>(W[row * ct + col0 + mt * 8 + mq]) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
    }
  }
}

// K-quartered phase-1 K-loop (HH_MV_QUART): the window's rows [0, nrows) lie in four quarter
// regions of Qr = ceil(nrows / 4) rows each (the last ones shorter or empty); lane group kq
// multiplies row j of quarter kq in K-step j.  wq / xq point at this lane's quarter.
template <int TAG, int NR, int MT>
__device__ __forceinline__ void p1_mma_rows_qt(const uint8_t *wq, const double *xq, int nrq, int Qr, int ct, int col0,
                                               int lane, double (&c)[4][NR / 8][2]) {
  using T = typename Elem<TAG>::T;
  const int mq = lane >> 2;
  const T *W = reinterpret_cast<const T *>(wq) + col0 + mq;
  const double *X = xq + mq;
  bool cv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) cv[mt] = col0 + mt * 8 + mq < ct;
  int j = 0;
  if (col0 + MT * 8 <= ct) {  // whole M-tiles: no column checks on the rows every quarter holds
    const int jfull = __reduce_min_sync(0xffffffffu, nrq);
#pragma unroll 2
    for (; j < jfull; ++j) {
      double b[NR / 8];
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) b[nt] = X[j * NR + nt * 8];
      const T *wrow = W + j * ct;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double av = up<TAG>(wrow[mt * 8]);
#pragma unroll
        for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
      }
    }
  }
#pragma unroll 2
  for (; j < Qr; ++j) {
    const bool rv = j < nrq;
    double b[NR / 8];
#pragma unroll
    for (int nt = 0; nt < NR / 8; ++nt) b[nt] = rv ? X[j * NR + nt * 8] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double av = (rv && cv[mt]) ? up<TAG>(W[j * ct + mt * 8]) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
    }
  }
}

template <int TAG, int NR>
__device__ __forceinline__ void p1_mma_rows_q(const uint8_t *wq, const double *xq, int nrq, int Qr, int ct, int col0,
                                              int lane, double (&c)[4][NR / 8][2]) {
  const int mtiles = min(4, (ct - col0 + 7) >> 3);
  switch (mtiles) {
    case 4: p1_mma_rows_qt<TAG, NR, 4>(wq, xq, nrq, Qr, ct, col0, lane, c); break;
    case 3: p1_mma_rows_qt<TAG, NR, 3>(wq, xq, nrq, Qr, ct, col0, lane, c); break;
    case 2: p1_mma_rows_qt<TAG, NR, 2>(wq, xq, nrq, Qr, ct, col0, lane, c); break;
    default: p1_mma_rows_qt<TAG, NR, 1>(wq, xq, nrq, Qr, ct, col0, lane, c); break;
  }
}

// only the M-tiles that hold columns of the tile are multiplied (MT = 1..4, warp-uniform)
template <int TAG, int NR>
__device__ __forceinline__ void p1_mma_rows(const uint8_t *wst, const double *xst, int nrows, int ct, int col0,
                                            int lane, double (&c)[4][NR / 8][2]) {
  const int mtiles = min(4, (ct - col0 + 7) >> 3);
  switch (mtiles) {
    case 4: p1_mma_rows_t<TAG, NR, 4>(wst, xst, nrows, ct, col0, lane, c); break;
    case 3: p1_mma_rows_t<TAG, NR, 3>(wst, xst, nrows, ct, col0, lane, c); break;
    case 2: p1_mma_rows_t<TAG, NR, 2>(wst, xst, nrows, ct, col0, lane, c); break;
    default: p1_mma_rows_t<TAG, NR, 1>(wst, xst, nrows, ct, col0, lane, c); break;
  }
}

template <int NR, class G>
__device__ __forceinline__ void p1_mma_consumer(const P1Args &a, uint8_t *smem, uint64_t *full, uint64_t *empty,
                                                int warp, int lane) {
  constexpr int NT = NR / 8;
  double c[4][NT][2];
  int32_t zi[4];
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    const uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int ct = m.a, col0 = warp * 32;
    const bool active = col0 < ct;
    if (m.r0 == 0) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) c[mt][nt][0] = c[mt][nt][1] = 0.0;
        const int col = col0 + mt * 8 + (lane >> 2);
        if (col < ct && m.pb < 0) zi[mt] = a.zmap[m.p + col];
      }
    }
    if (active) {
      const int nrows = m.r1 - m.r0;
      if constexpr (quartered<NR>()) {
        // this lane's quarter: rows [kq Qr, kq Qr + nrq) of the window, staged in region kq
        const int kq = lane & 3, Qr = (nrows + 3) >> 2;
        const int nrq = max(0, min(Qr, nrows - kq * Qr));
        const int qw = Qr * ct * tag_bytes(m.b), qx = Qr * NR * 8;
        const uint8_t *wq = st + kq * quarter_stride(qw) + ((m.wlead + kq * qw) & 15);
        const double *xq =
            reinterpret_cast<const double *>(st + G::WBUF + kq * quarter_stride(qx) + ((m.xlead + kq * qx) & 15));
        dispatch_tag(m.b, [&](auto t) { p1_mma_rows_q<decltype(t)::value, NR>(wq, xq, nrq, Qr, ct, col0, lane, c); });
      } else {
        const uint8_t *wst = st + m.wlead;
        const double *xst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
        dispatch_tag(m.b, [&](auto t) { p1_mma_rows<decltype(t)::value, NR>(wst, xst, nrows, ct, col0, lane, c); });
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (m.r1 == m.q && active) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int col = col0 + mt * 8 + (lane >> 2);
        if (col < ct) {
          double *out = (m.pb >= 0 ? a.partial + (m.pb + col) * NR : a.v + (a.N + zi[mt]) * NR) + 2 * (lane & 3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            *reinterpret_cast<double2 *>(out + nt * 8) = make_double2(c[mt][nt][0], c[mt][nt][1]);
        }
      }
    }
  }
}

// ---- NR = 1 (the headline single-RHS product): vector factor loads.  At one RHS every stored
// element costs a load, an exact up-conversion and a DFMA; loading V consecutive elements with
// one 8/16-byte shared-memory access into V independent DFMA chains halves the issued
// instructions per element (ncu r01: 13 thread-instructions per element, 61-68% issue-busy),
// which keeps the kernels HBM-bound when the power cap lowers the SM clock.
// V consecutive stored elements starting at e (aligned to V elements) -> fp64, exactly
template <int TAG, int V>
__device__ __forceinline__ void loadv(const typename Elem<TAG>::T *e, double (&w)[V]) {
  if constexpr (V == 1) {
    w[0] = up<TAG>(e[0]);
  } else if constexpr (TAG == TAG_FP64) {
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const double2 d = *reinterpret_cast<const double2 *>(e + i);
      w[i] = d.x;
      w[i + 1] = d.y;
    }
  } else if constexpr (TAG == TAG_FP32) {
    if constexpr (V == 4) {
      const float4 f = *reinterpret_cast<const float4 *>(e);
      w[0] = f.x; w[1] = f.y; w[2] = f.z; w[3] = f.w;
    } else {
      const float2 f = *reinterpret_cast<const float2 *>(e);
      w[0] = f.x; w[1] = f.y;
    }
  } else if constexpr (TAG == TAG_FP16 || TAG == TAG_BF16) {
    uint32_t u[V / 2];
    if constexpr (V == 4) {
      const uint2 p = *reinterpret_cast<const uint2 *>(e);
      u[0] = p.x; u[1] = p.y;
    } else {
      u[0] = *reinterpret_cast<const uint32_t *>(e);
    }
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      if constexpr (TAG == TAG_FP16) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&u[i]));
        w[2 * i] = f.x; w[2 * i + 1] = f.y;
      } else {
        w[2 * i] = (double)__uint_as_float(u[i] << 16);
        w[2 * i + 1] = (double)__uint_as_float(u[i] & 0xFFFF0000u);
      }
    }
  } else if constexpr (TAG == TAG_BF24) {
    // V elements = 3V bytes, 4-byte (V = 4) / 2-byte (V = 2) aligned: whole words, then shifts
    if constexpr (V == 4) {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(e);
      const uint32_t a = p[0], b = p[1], c = p[2];
      w[0] = (double)__uint_as_float(a << 8);
      w[1] = (double)__uint_as_float(__funnelshift_l(a, b, 16) & 0xFFFFFF00u);  // bytes 3..5
      w[2] = (double)__uint_as_float(__funnelshift_l(b, c, 24) & 0xFFFFFF00u);  // bytes 6..8
      w[3] = (double)__uint_as_float(c & 0xFFFFFF00u);
    } else {
      const uint16_t *p = reinterpret_cast<const uint16_t *>(e);
      const uint32_t a = p[0], b = p[1], c = p[2];  // bytes 0..5
      w[0] = (double)__uint_as_float((a << 8) | (b << 24));
      w[1] = (double)__uint_as_float((b & 0xFF00u) | (c << 16));
    }
  } else if constexpr (TAG == TAG_FP48) {
    // V elements = 6V bytes, 8-byte (V = 4) / 4-byte (V = 2) aligned
    if constexpr (V == 4) {
      const uint64_t *p = reinterpret_cast<const uint64_t *>(e);
      const uint64_t a = p[0], b = p[1], c = p[2];
      w[0] = __longlong_as_double((long long)(a << 16));
      w[1] = __longlong_as_double((long long)(((a >> 48) | (b << 16)) << 16));
      w[2] = __longlong_as_double((long long)((((b >> 32) | (c << 32)) << 16)));
      w[3] = __longlong_as_double((long long)(c & 0xFFFFFFFFFFFF0000ull));
    } else {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(e);
      const uint64_t a = p[0], b = p[1], c = p[2];  // bytes 0..11
      w[0] = __longlong_as_double((long long)(((a | (b << 32)) << 16)));
      w[1] = __longlong_as_double((long long)((((b >> 16) | (c << 16)) << 16)));
    }
  } else {  // q43
    uint32_t u;
    if constexpr (V == 4) u = *reinterpret_cast<const uint32_t *>(e);
    else u = *reinterpret_cast<const uint16_t *>(e);
#pragma unroll
    for (int i = 0; i < V; ++i) w[i] = up<TAG_Q43>((uint8_t)(u >> (8 * i)));
  }
}

// acc[i] += w(row j, element i) * v[j] over the rows j = j0, j0 + jstep, ... < jend this thread
// owns (V chains; e / v point at row j0).  The bound is tested on j itself: no per-stage
// integer division for the trip count (the small-leaf workloads are issue-bound on exactly
// this kind of per-stage overhead, profiles/r02k_probe.txt)
template <int TAG, int V>
__device__ __forceinline__ void vec_acc(const typename Elem<TAG>::T *e, const double *v, int j0, int jend, int jstep,
                                        int es, int vs, double (&acc)[4]) {
#pragma unroll 2
  for (int j = j0; j < jend; j += jstep) {
    double w[V];
    loadv<TAG, V>(e, w);
    const double x = *v;
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = __fma_rn(w[i], x, acc[i]);
    e += es;
    v += vs;
  }
}

template <int V>
__device__ __forceinline__ void vec_acc_tag(int tag, const uint8_t *base, int e0, const double *v, int j0, int jend,
                                            int jstep, int es, int vs, double (&acc)[4]) {
  dispatch_tag(tag, [&](auto t) {
    constexpr int TG = decltype(t)::value;
    vec_acc<TG, V>(reinterpret_cast<const typename Elem<TG>::T *>(base) + e0, v, j0, jend, jstep, es, vs, acc);
  });
}

// Phase-1 consumer at NR = 1: a tile whose width is a multiple of 4 is read as 4-column
// vectors — thread = (column quad cq, row group q), 4 chains; narrower layouts keep one
// column per thread.  The Q row groups of a column (quad) are adjacent lanes, reduced by
// shuffles in a fixed order at the tile's last window.
template <class G>
__device__ __forceinline__ void p1_consumer_nr1(const P1Args &a, uint8_t *smem, uint64_t *full, uint64_t *empty,
                                                int tid, int lane) {
  int cur_ct = -1, V = 1, slots = 1, lq = 0, cs = 0, q = 0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int32_t zi[4] = {0, 0, 0, 0};
  PROBE(unsigned long long ct0 = pclk(); unsigned long long cwait = 0;)
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    PROBE(const unsigned long long w0 = pclk();)
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    PROBE(cwait += pclk() - w0;)
    const uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int ct = m.a;
    if (ct != cur_ct) {  // thread layout of this tile width (recomputed only when it changes)
      cur_ct = ct;
      V = (ct & 3) == 0 ? 4 : 1;
      slots = ct / V;
      lq = 0;  // Q = 2^lq row groups, <= 8, Q * slots <= NCT
      while (lq < 3 && (2 << lq) * slots <= NCT) ++lq;
      cs = tid >> lq;
      q = tid & ((1 << lq) - 1);
    }
    const int Q = 1 << lq;
    const bool active = cs < slots;
    if (m.r0 == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i] = 0.0;
        if (active && i < V && q == 0 && m.pb < 0) zi[i] = a.zmap[m.p + cs * V + i];
      }
    }
    if (active) {
      const uint8_t *wst = st + m.wlead;
      const double *xst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
      const int nrows = m.r1 - m.r0;
      if (V == 4) vec_acc_tag<4>(m.b, wst, q * ct + 4 * cs, xst + q, q, nrows, Q, Q * ct, Q, acc);
      else vec_acc_tag<1>(m.b, wst, q * ct + cs, xst + q, q, nrows, Q, Q * ct, Q, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (m.r1 == m.q) {  // last window of the tile: fixed-order reduction over the Q row groups
      for (int o = 1; o < Q; o <<= 1)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (q == 0 && active) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < V) {
            double *out = m.pb >= 0 ? a.partial + (m.pb + cs * V + i) : a.v + (a.N + zi[i]);
            *out = acc[i];
          }
      }
    }
  }
  PROBE(if (tid == 0) {
    atomicAdd(&g_probe[3], pclk() - ct0);
    atomicAdd(&g_probe[4], cwait);
  })
}

template <int NR, int WP = 0, int GV = 0>
__global__ void __launch_bounds__(THREADS, min_ctas<NR, 1>()) k_phase1(P1Args a) {
  static_assert(WP == 0 || NR <= 4, "reduced working precision runs the FMA consumers (NR <= 4)");
  using G = Geo<NR, 1, GV>;
  using A = typename WpT<WP>::A;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + G::STAGES * G::STAGE);
  uint64_t *empty = full + G::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (warp == NCW) {  // ------------------------------------------------ producer
    if (lane != 0) return;
    if constexpr (planned<NR, WP>()) {
      planned_producer<G, 1>(a.plan, a.ntiles, a.ctr, smem, full, empty);
      return;
    }
    const uint64_t pol_w = evict_first_policy(), pol_x = evict_last_policy();
    int n = 0;
    // the next item index and its descriptor are requested one item ahead, so their latency
    // overlaps the current item's stage issue (small tiles are ~1 us of streaming each)
    PROBE(unsigned long long pt0 = pclk(); unsigned long long pwait = 0; unsigned long long pitems = 0;)
    int item = atomicAdd(a.ctr, 1);
    P1Tile Tn{};
    if (item < a.ntiles) Tn = a.tiles[item];
    while (item < a.ntiles) {
      PROBE(++pitems;)
      const P1Tile T = Tn;
      const int nxt = atomicAdd(a.ctr, 1);
      if (nxt < a.ntiles) Tn = a.tiles[nxt];
      const int w = tag_bytes(T.tag);
      const int rowb = T.ct * w;
      int rs = max(1, min(G::XELEMS / NR, G::WDATA / rowb));
      // DMMA K-steps take 4 rows: whole K-steps per window (49 rows of a 248-column fp32 tile
      // would pad every window's 13th K-step with 3 zero rows, 6% of the issued DMMAs)
      if constexpr (use_mma<NR>() && WP == 0)
        if (rs >= 4) rs &= ~3;
      if constexpr (quartered<NR, WP>()) {  // four quarter regions per buffer; whole K-steps per quarter
        int Q = max(1, min(quarter_max_bytes(G::WBUF) / rowb, quarter_max_bytes(G::XBUF) / (NR * 8)));
        if (Q >= 4) Q &= ~3;  // quarters start 16-B aligned alike => exact 8-bank skew
        rs = 4 * Q;
      }
      const uint8_t *wbase = pick(a.W, T.tag) + T.src + (int64_t)T.r0 * rowb;
      const uint8_t *xbase = reinterpret_cast<const uint8_t *>(a.v + (T.x0 + T.r0) * NR);
      for (int r0 = 0; r0 < T.n; r0 += rs, ++n) {
        const int r1 = min(T.n, r0 + rs);
        const int s = n % G::STAGES;
        PROBE(const unsigned long long w0 = pclk();)
        if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
        PROBE(pwait += pclk() - w0;)
        uint8_t *st = smem + s * G::STAGE;
        const uint8_t *wsrc = wbase + (int64_t)r0 * rowb;
        const int64_t wlen = (int64_t)(r1 - r0) * rowb;
        const uint8_t *xsrc = xbase + (int64_t)r0 * NR * 8;
        const int64_t xlen = (int64_t)(r1 - r0) * NR * 8;
        Meta *m = reinterpret_cast<Meta *>(st + G::WBUF + G::XBUF);
        m->kind = 0;
        m->wlead = (int)((uintptr_t)wsrc & 15);
        m->xlead = (int)((uintptr_t)xsrc & 15);
        m->r0 = r0;
        m->r1 = r1;
        m->a = T.ct;
        m->b = T.tag;
        m->p = T.zbase;
        m->q = T.n;
        m->pb = T.pbase;
        if constexpr (quartered<NR, WP>()) {
          const int nrw = r1 - r0, Qr = (nrw + 3) >> 2;
          const int qw = Qr * rowb, qx = Qr * NR * 8;
          uint32_t exp = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int nq = max(0, min(Qr, nrw - q * Qr));
            exp += window_bytes(wsrc + q * qw, (int64_t)nq * rowb) + window_bytes(xsrc + q * qx, (int64_t)nq * NR * 8);
          }
          mbar_expect_tx(&full[s], exp);
          uint32_t tx = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int nq = max(0, min(Qr, nrw - q * Qr));
            stage_copy(st + q * quarter_stride(qw), wsrc + q * qw, (int64_t)nq * rowb, &full[s], pol_w, tx);
            stage_copy(st + G::WBUF + q * quarter_stride(qx), xsrc + q * qx, (int64_t)nq * NR * 8, &full[s], pol_x, tx);
          }
        } else {
          mbar_expect_tx(&full[s], window_bytes(wsrc, wlen) + window_bytes(xsrc, xlen));
          uint32_t tx = 0;
          stage_copy(st, wsrc, wlen, &full[s], pol_w, tx);
          stage_copy(st + G::WBUF, xsrc, xlen, &full[s], pol_x, tx);
        }
      }
      item = nxt;
    }
    PROBE(if (NR == 1 && WP == 0) {
      atomicAdd(&g_probe[0], pclk() - pt0);
      atomicAdd(&g_probe[1], pwait);
      atomicAdd(&g_probe[2], (unsigned long long)n);
      atomicAdd(&g_probe[6], pitems);
    })
    const int s = n % G::STAGES;
    if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
    reinterpret_cast<Meta *>(smem + s * G::STAGE + G::WBUF + G::XBUF)->kind = 1;
    mbar_arrive(&full[s]);
    return;
  }
  if constexpr (WP == 0 && use_mma<NR>()) {
    p1_mma_consumer<NR, G>(a, smem, full, empty, warp, lane);
    return;
  }
#if HH_MV_VEC1
  if constexpr (WP == 0 && NR == 1) {
    p1_consumer_nr1<G>(a, smem, full, empty, threadIdx.x, lane);
    return;
  }
#endif
  // --------------------------------------------------------------------- consumers
  constexpr int MB = mblock<NR>();
  const int tid = threadIdx.x;
  int cur_ct = -1, slots = 1, Q = 1, cs = 0, q = 0;
  A acc[MB][NR];
  int32_t zi[MB];
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    const uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int ct = m.a;
    if (ct != cur_ct) {  // thread layout of this tile width (recomputed only when it changes)
      cur_ct = ct;
      slots = (ct + MB - 1) / MB;  // thread column slot cs owns columns cs + b * slots
      int lq = 0;                  // Q = 2^lq row groups, <= 8, Q * slots <= NCT (lanes of a column share a warp)
      while (lq < 3 && (2 << lq) * slots <= NCT) ++lq;
      Q = 1 << lq;
      cs = tid >> lq;
      q = tid & (Q - 1);
    }
    const bool active = cs < slots;
    bool valid[MB];
#pragma unroll
    for (int b = 0; b < MB; ++b) valid[b] = active && cs + b * slots < ct;
    if (m.r0 == 0) {
#pragma unroll
      for (int b = 0; b < MB; ++b) {
#pragma unroll
        for (int k = 0; k < NR; ++k) acc[b][k] = wp_zero<A>();
        if (valid[b] && q == 0 && m.pb < 0) zi[b] = a.zmap[m.p + cs + b * slots];
      }
    }
    if (active) {
      const uint8_t *wst = st + m.wlead;
      const double *xst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
      const int nrows = m.r1 - m.r0;
      const int cnt = q < nrows ? (nrows - q + Q - 1) / Q : 0;
      const int e0 = q * ct + cs;
      dispatch_tag(m.b, [&](auto t) {
        constexpr int TG = decltype(t)::value;
        block_acc<TG, NR, MB, A>(reinterpret_cast<const typename Elem<TG>::T *>(wst) + e0, xst + q * NR, cnt, Q * ct,
                                 slots, Q * NR, valid, acc);
      });
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (m.r1 == m.q) {  // last stage of the tile: fixed-order reduction over the Q row groups
      for (int o = 1; o < Q; o <<= 1)
#pragma unroll
        for (int b = 0; b < MB; ++b)
#pragma unroll
          for (int k = 0; k < NR; ++k) acc[b][k] = wp_add(acc[b][k], __shfl_xor_sync(0xffffffffu, acc[b][k], o));
      if (q == 0)
#pragma unroll
        for (int b = 0; b < MB; ++b)
          if (valid[b]) {
            double *out = m.pb >= 0 ? a.partial + (m.pb + cs + b * slots) * NR : a.v + (a.N + zi[b]) * NR;
#pragma unroll
            for (int k = 0; k < NR; ++k) out[k] = wp_out<A>(acc[b][k]);
          }
    }
  }
}

// --------------------------------------------------------------------------- phase 2
struct P2Args {
  const P2Leaf *leaves;
  const P2Seg *segs;
  int64_t nleaves;
  const uint8_t *U[NTAG];
  const uint8_t *D;
  const double *v;
  const int32_t *perm;
  double *y;
  int64_t ldy;
  int *ctr;
  PlanArgs plan;      // planned single-RHS product only
};

// Phase-2 DMMA consumer (NR = 8, 16): the leaf's rows form ceil(nr/8) M-tiles, grouped by
// four (MG groups); warp w takes group w % MG and the K-steps (4 columns) k = w / MG (mod
// KS), KS = NCW / MG.  At the leaf's last window the KS partial tiles of each group are
// summed in a fixed order through shared memory and scattered to y (a10).
template <int TAG, int NR, int MT>
__device__ __forceinline__ void p2_mma_cols_t(const uint8_t *ust, const double *zst, int ncols, int nr, int row0,
                                              int kfirst, int KS, int lane, double (&c)[4][NR / 8][2]) {
  using T = typename Elem<TAG>::T;
  const T *U = reinterpret_cast<const T *>(ust);
  const int kq = lane & 3, mq = lane >> 2;
  bool rv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) rv[mt] = row0 + mt * 8 + mq < nr;
  int k0 = 4 * kfirst;
#if HH_MV_PEEL2
  // whole K-steps: no column checks; rows checked only when the group's last tile is ragged
  const bool rows_full = row0 + MT * 8 <= nr;
  const int kfull = ncols & ~3;
  if (rows_full) {
#pragma unroll 2
    for (; k0 < kfull; k0 += 4 * KS) {
      const int col = k0 + kq;
      double b[NR / 8];
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) b[nt] = zst[col * NR + nt * 8 + mq];
      const T *ucol = U + col * nr + row0 + mq;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double av = up<TAG>(ucol[mt * 8]);
#pragma unroll
        for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
      }
    }
  }
#endif
#pragma unroll 2
  for (; k0 < ncols; k0 += 4 * KS) {
    const int col = k0 + kq;
    const bool cvl = col < ncols;
    double b[NR / 8];
#pragma unroll
    for (int nt = 0; nt < NR / 8; ++nt) b[nt] = cvl ? zst[col * NR + nt * 8 + mq] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double av = (cvl && rv[mt]) ? up<TAG>(U[col * nr + row0 + mt * 8 + mq]) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
    }
  }
}

// K-quartered phase-2 K-loop (HH_MV_QUART): the window's columns [0, ncols) lie in four
// quarter regions of Qc = ceil(ncols / 4) columns; lane group kq multiplies column j of
// quarter kq in K-step j (K-steps j = kfirst, kfirst + KS, ... belong to this warp's K-slice).
template <int TAG, int NR, int MT>
__device__ __forceinline__ void p2_mma_cols_qt(const uint8_t *uq, const double *zq, int ncq, int Qc, int nr, int row0,
                                               int kfirst, int KS, int lane, double (&c)[4][NR / 8][2]) {
  using T = typename Elem<TAG>::T;
  const int mq = lane >> 2;
  const T *U = reinterpret_cast<const T *>(uq) + row0 + mq;
  const double *Z = zq + mq;
  bool rv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) rv[mt] = row0 + mt * 8 + mq < nr;
#pragma unroll 2
  for (int j = kfirst; j < Qc; j += KS) {
    const bool cvl = j < ncq;
    double b[NR / 8];
#pragma unroll
    for (int nt = 0; nt < NR / 8; ++nt) b[nt] = cvl ? Z[j * NR + nt * 8] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double av = (cvl && rv[mt]) ? up<TAG>(U[j * nr + mt * 8]) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NR / 8; ++nt) dmma(c[mt][nt], av, b[nt]);
    }
  }
}

template <int TAG, int NR>
__device__ __forceinline__ void p2_mma_cols_q(const uint8_t *uq, const double *zq, int ncq, int Qc, int nr, int row0,
                                              int tcount, int kfirst, int KS, int lane, double (&c)[4][NR / 8][2]) {
  switch (tcount) {
    case 4: p2_mma_cols_qt<TAG, NR, 4>(uq, zq, ncq, Qc, nr, row0, kfirst, KS, lane, c); break;
    case 3: p2_mma_cols_qt<TAG, NR, 3>(uq, zq, ncq, Qc, nr, row0, kfirst, KS, lane, c); break;
    case 2: p2_mma_cols_qt<TAG, NR, 2>(uq, zq, ncq, Qc, nr, row0, kfirst, KS, lane, c); break;
    default: p2_mma_cols_qt<TAG, NR, 1>(uq, zq, ncq, Qc, nr, row0, kfirst, KS, lane, c); break;
  }
}

// only this group's M-tiles are multiplied (tcount = 1..4, warp-uniform)
template <int TAG, int NR>
__device__ __forceinline__ void p2_mma_cols(const uint8_t *ust, const double *zst, int ncols, int nr, int row0,
                                            int tcount, int kfirst, int KS, int lane, double (&c)[4][NR / 8][2]) {
  switch (tcount) {
    case 4: p2_mma_cols_t<TAG, NR, 4>(ust, zst, ncols, nr, row0, kfirst, KS, lane, c); break;
    case 3: p2_mma_cols_t<TAG, NR, 3>(ust, zst, ncols, nr, row0, kfirst, KS, lane, c); break;
    case 2: p2_mma_cols_t<TAG, NR, 2>(ust, zst, ncols, nr, row0, kfirst, KS, lane, c); break;
    default: p2_mma_cols_t<TAG, NR, 1>(ust, zst, ncols, nr, row0, kfirst, KS, lane, c); break;
  }
}

template <int NR, class G>
__device__ __forceinline__ void p2_mma_consumer(const P2Args &a, uint8_t *smem, uint64_t *full, uint64_t *empty,
                                                double *red, int warp, int lane) {
  constexpr int NT = NR / 8;
  double c[4][NT][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[mt][nt][0] = c[mt][nt][1] = 0.0;
  int kbase = 0;  // K-step parity offset: windows of a leaf continue the K-step numbering
  int cur_nr = -1, MG = 1, KS = 1, mg = 0, ks = 0, tbeg = 0, tcnt = 0;
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    const uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int nr = m.a;
    if (nr != cur_nr) {  // per-leaf warp layout (integer divisions only when the leaf size changes)
      cur_nr = nr;
      const int T = (nr + 7) >> 3;  // 8-row M-tiles of the leaf, dealt to MG groups of <= 4
      MG = (T + 3) >> 2;
      KS = max(1, NCW / MG);
      mg = warp % MG;
      ks = warp / MG;
      tbeg = mg * T / MG;           // balanced: group sizes differ by at most one tile
      tcnt = (mg + 1) * T / MG - tbeg;
    }
    const bool active = warp < MG * KS;
    const int ncols = m.r1 - m.r0;
    if (active) {
      int kfirst = ks - kbase;
      if (kfirst < 0) kfirst += KS;
      if constexpr (quartered<NR>()) {
        // this lane's quarter: columns [kq Qc, kq Qc + ncq) of the window, staged in region kq
        const int kq = lane & 3, Qc = (ncols + 3) >> 2;
        const int ncq = max(0, min(Qc, ncols - kq * Qc));
        const int qu = Qc * nr * tag_bytes(m.b & 0xff), qz = Qc * NR * 8;
        const uint8_t *uq = st + kq * quarter_stride(qu) + ((m.wlead + kq * qu) & 15);
        const double *zq =
            reinterpret_cast<const double *>(st + G::WBUF + kq * quarter_stride(qz) + ((m.xlead + kq * qz) & 15));
        dispatch_tag(m.b & 0xff, [&](auto t) {
          p2_mma_cols_q<decltype(t)::value, NR>(uq, zq, ncq, Qc, nr, tbeg * 8, tcnt, kfirst, KS, lane, c);
        });
      } else {
        const uint8_t *ust = st + m.wlead;
        const double *zst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
        dispatch_tag(m.b & 0xff, [&](auto t) {
          p2_mma_cols<decltype(t)::value, NR>(ust, zst, ncols, nr, tbeg * 8, tcnt, kfirst, KS, lane, c);
        });
      }
    }
    if (KS == 1) {
      kbase = 0;
    } else {
      kbase += (ncols + 3) >> 2;
      while (kbase >= KS) kbase -= KS;
    }
    __syncwarp();
    if (!G::RED_IN_STAGE || !(m.flags & 1))
      if (lane == 0) mbar_arrive(&empty[s]);
    if (m.flags & 1) {
      if constexpr (G::RED_IN_STAGE) {
        static_assert(G::red_bytes() <= (size_t)G::WBUF + G::XBUF, "reduction fits the stage data");
        red = reinterpret_cast<double *>(smem + s * G::STAGE);
        consumer_sync();  // every warp is done with the stage's U / z before it is overwritten
      }
      double *mine = red + (size_t)warp * 4 * NT * 64;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mine[((mt * NT + nt) * 32 + lane) * 2] = c[mt][nt][0];
          mine[((mt * NT + nt) * 32 + lane) * 2 + 1] = c[mt][nt][1];
          c[mt][nt][0] = c[mt][nt][1] = 0.0;
        }
      consumer_sync();
      // every warp finalises some of the MG x 4 x NT output fragments: fixed-order sum over
      // the KS k-slices, then the scatter y[perm[t]] (a10)
      const int T = (nr + 7) >> 3;
      for (int f = warp; f < MG * 4 * NT; f += NCW) {
        const int g = f / (4 * NT), mt = (f / NT) % 4, nt = f % NT;
        const int tb = g * T / MG, tc = (g + 1) * T / MG - tb;  // group g's tiles (as in the layout)
        if (mt >= tc) continue;
        const int r = (tb + mt) * 8 + (lane >> 2);
        if (r >= nr) continue;
        double s0 = 0.0, s1 = 0.0;
        for (int k = 0; k < KS; ++k) {
          const double *src = red + (size_t)(g + k * MG) * 4 * NT * 64 + ((mt * NT + nt) * 32 + lane) * 2;
          s0 += src[0];
          s1 += src[1];
        }
        const int64_t i = a.perm[m.p + r];
        const int64_t col = nt * 8 + 2 * (lane & 3);
        a.y[i + col * a.ldy] = s0;
        a.y[i + (col + 1) * a.ldy] = s1;
      }
      if constexpr (G::RED_IN_STAGE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      consumer_sync();
      if constexpr (G::RED_IN_STAGE)
        if (lane == 0) mbar_arrive(&empty[s]);  // the stage goes back to the producer's TMA
      kbase = 0;
    }
  }
}

// Phase-2 consumer at NR = 1: thread = (row slot rs, column group g); a row slot is V = 4 (|R|
// a multiple of 4), 2 (|R| even) or 1 consecutive rows of the leaf, read with one shared-memory
// access per column (the U slab is column-major, so a slot's rows are adjacent and a warp reads
// one contiguous span); V independent DFMA chains.  At the leaf's last window the Gn group
// partials are summed in a fixed order through that stage's data area (held back from the
// producer until the scatter y[perm[t]] (a10) is done).
template <class G>
__device__ __forceinline__ void p2_consumer_nr1(const P2Args &a, uint8_t *smem, uint64_t *full, uint64_t *empty,
                                                int tid, int lane) {
  static_assert(sizeof(double) * NCT * 4 <= (size_t)G::WBUF, "leaf reduction fits the stage");
  int cur_nr = -1, V = 1, nslots = 1, Gn = 1, rs = 0, g = 0;
  int lt = 0, rr = 0, sub = 0, rsl = 0, ri = 0;  // leaf-end reduction role of this thread
  int64_t cur_leaf = -1, yi = 0;                 // the leaf's first tree position, y index of row rr
  int64_t ys[4] = {0, 0, 0, 0};                  // (HH_MV_P2RED = 0) y indices of this slot's rows
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  PROBE(unsigned long long ct0 = pclk(); unsigned long long cwait = 0; unsigned long long cend = 0;)
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    PROBE(const unsigned long long w0 = pclk();)
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    PROBE(cwait += pclk() - w0;)
    uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int nr = m.a;
    if (nr != cur_nr) {  // per-leaf layout (divisions only when the leaf size changes)
      cur_nr = nr;
      V = (nr & 3) == 0 ? 4 : (nr & 1) == 0 ? 2 : 1;
      nslots = nr / V;
      Gn = NCT / nslots;  // nr <= 256 (leaf_size limit)
      rs = tid % nslots;
      g = tid / nslots;
      // reduction: row rr of the leaf (slot rr / V, element rr % V) is summed by T = 2^lt
      // adjacent lanes (T * nr <= NCT), each over a strided subset of the Gn group partials
      lt = 0;
      while (lt < 5 && (nr << (lt + 1)) <= NCT) ++lt;
      rr = tid >> lt;
      sub = tid & ((1 << lt) - 1);
      rsl = rr / V;
      ri = rr - rsl * V;
    }
    if (m.p != cur_leaf) {  // a new leaf: its scatter indices are fetched now, used at the leaf end
      cur_leaf = m.p;
#if HH_MV_P2RED
      if (rr < nr) yi = a.perm[m.p + rr];
#else
      if (tid < nslots)
        for (int i = 0; i < 4; ++i)
          if (i < V) ys[i] = a.perm[m.p + tid * V + i];
#endif
    }
    if (g < Gn) {
      const uint8_t *ust = st + m.wlead;
      const double *zst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
      const int ncols = m.r1 - m.r0;
      const int e0 = g * nr + rs * V;
      if (V == 4) vec_acc_tag<4>(m.b & 0xff, ust, e0, zst + g, g, ncols, Gn, Gn * nr, Gn, acc);
      else if (V == 2) vec_acc_tag<2>(m.b & 0xff, ust, e0, zst + g, g, ncols, Gn, Gn * nr, Gn, acc);
      else vec_acc_tag<1>(m.b & 0xff, ust, e0, zst + g, g, ncols, Gn, Gn * nr, Gn, acc);
    }
    __syncwarp();
    if (!(m.flags & 1)) {
      if (lane == 0) mbar_arrive(&empty[s]);
      continue;
    }
    // last window of the leaf: fixed-order reduction over the Gn groups in this stage's data
    PROBE(const unsigned long long e0 = pclk();)
    consumer_sync();  // every warp is done with the stage's U / z
    double *red = reinterpret_cast<double *>(st);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      red[tid * 4 + i] = acc[i];
      acc[i] = 0.0;
    }
    consumer_sync();
#if HH_MV_P2RED
    const int T = 1 << lt;
    double sum = 0.0;
    if (rr < nr)
      for (int gg = sub; gg < Gn; gg += T) sum += red[(gg * nslots + rsl) * 4 + ri];
#else
    double sv[4] = {0.0, 0.0, 0.0, 0.0};
    if (tid < nslots)
      for (int gg = 0; gg < Gn; ++gg)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < V) sv[i] += red[(gg * nslots + tid) * 4 + i];
#endif
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    consumer_sync();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage goes back to the producer's TMA
#if HH_MV_P2RED
    // fixed shuffle tree over the T lanes of the row, then the scatter y[perm[t]] (a10)
    for (int o = 1; o < T; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (rr < nr && sub == 0) a.y[yi] = sum;
#else
    if (tid < nslots)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < V) a.y[ys[i]] = sv[i];
#endif
    PROBE(cend += pclk() - e0;)
  }
  PROBE(if (tid == 0) {
    atomicAdd(&g_probe[11], pclk() - ct0);
    atomicAdd(&g_probe[12], cwait);
    atomicAdd(&g_probe[13], cend);
  })
}

template <int NR, int WP = 0, int GV = 0>
__global__ void __launch_bounds__(THREADS, min_ctas<NR, 2>()) k_phase2(P2Args a) {
  static_assert(WP == 0 || NR <= 4, "reduced working precision runs the FMA consumers (NR <= 4)");
  using G = Geo<NR, 2, GV>;
  using A = typename WpT<WP>::A;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + G::STAGES * G::STAGE);
  uint64_t *empty = full + G::STAGES;
  double *red = reinterpret_cast<double *>(empty + G::STAGES);  // [NCT][MB][NR]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (warp == NCW) {  // ------------------------------------------------ producer
    if (lane != 0) return;
    if constexpr (planned<NR, WP>()) {
      planned_producer<G, 2>(a.plan, a.nleaves, a.ctr + 1, smem, full, empty);
      return;
    }
    const uint64_t pol_w = evict_first_policy(), pol_x = evict_last_policy();
    int n = 0;
    // next leaf index / descriptor and the next segment descriptor are fetched one ahead
    // (also fetching the next leaf's first segment descriptor ahead was measured 10-25% SLOWER
    // in phase 2 at one RHS: profiles/r02i_ab_p2prefetch.txt)
    PROBE(unsigned long long pt0 = pclk(); unsigned long long pwait = 0; unsigned long long pitems = 0;)
    int li = atomicAdd(a.ctr + 1, 1);
    P2Leaf Ln{};
    if (li < a.nleaves) Ln = a.leaves[li];
    while (li < a.nleaves) {
      PROBE(++pitems;)
      const P2Leaf Lf = Ln;
      const int nxt = atomicAdd(a.ctr + 1, 1);
      if (nxt < a.nleaves) Ln = a.leaves[nxt];
      P2Seg Sn = a.segs[Lf.s0];
      for (int64_t si = Lf.s0; si < Lf.s1; ++si) {
        const P2Seg S = Sn;
        if (si + 1 < Lf.s1) Sn = a.segs[si + 1];
        const int w = tag_bytes(S.tag);
        const int colb = Lf.nr * w;
        int cs = max(1, min(G::XELEMS / NR, G::WDATA / colb));
        if constexpr (use_mma<NR>() && WP == 0)  // whole 4-column DMMA K-steps per window
          if (cs >= 4) cs &= ~3;
        if constexpr (quartered<NR, WP>()) {  // four quarter regions per buffer; whole K-steps per quarter
          int Q = max(1, min(quarter_max_bytes(G::WBUF) / colb, quarter_max_bytes(G::XBUF) / (NR * 8)));
          if (Q >= 4) Q &= ~3;  // quarters start 16-B aligned alike => exact 8-bank skew
          cs = 4 * Q;
        }
        const uint8_t *ubase = (S.dense ? a.D : pick(a.U, S.tag)) + S.src;
        const uint8_t *zbase = reinterpret_cast<const uint8_t *>(a.v + S.vbeg * NR);
        for (int c0 = 0; c0 < S.ncols; c0 += cs, ++n) {
          const int c1 = min(S.ncols, c0 + cs);
          const int s = n % G::STAGES;
          PROBE(const unsigned long long w0 = pclk();)
          if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
          PROBE(pwait += pclk() - w0;)
          uint8_t *st = smem + s * G::STAGE;
          const uint8_t *usrc = ubase + (int64_t)c0 * colb;
          const int64_t ulen = (int64_t)(c1 - c0) * colb;
          const uint8_t *zsrc = zbase + (int64_t)c0 * NR * 8;
          const int64_t zlen = (int64_t)(c1 - c0) * NR * 8;
          Meta *m = reinterpret_cast<Meta *>(st + G::WBUF + G::XBUF);
          m->kind = 0;
          m->wlead = (int)((uintptr_t)usrc & 15);
          m->xlead = (int)((uintptr_t)zsrc & 15);
          m->r0 = c0;
          m->r1 = c1;
          m->flags = (si + 1 == Lf.s1 && c1 == S.ncols) ? 1 : 0;
          m->a = Lf.nr;
          m->b = S.tag | (S.dense << 8);
          m->p = Lf.r0;
          if constexpr (quartered<NR, WP>()) {
            const int nc = c1 - c0, Qc = (nc + 3) >> 2;
            const int qu = Qc * colb, qz = Qc * NR * 8;
            uint32_t exp = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int nq = max(0, min(Qc, nc - q * Qc));
              exp += window_bytes(usrc + q * qu, (int64_t)nq * colb) + window_bytes(zsrc + q * qz, (int64_t)nq * NR * 8);
            }
            mbar_expect_tx(&full[s], exp);
            uint32_t tx = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int nq = max(0, min(Qc, nc - q * Qc));
              stage_copy(st + q * quarter_stride(qu), usrc + q * qu, (int64_t)nq * colb, &full[s], pol_w, tx);
              stage_copy(st + G::WBUF + q * quarter_stride(qz), zsrc + q * qz, (int64_t)nq * NR * 8, &full[s], pol_x, tx);
            }
          } else {
            mbar_expect_tx(&full[s], window_bytes(usrc, ulen) + window_bytes(zsrc, zlen));
            uint32_t tx = 0;
            stage_copy(st, usrc, ulen, &full[s], pol_w, tx);
            stage_copy(st + G::WBUF, zsrc, zlen, &full[s], pol_x, tx);
          }
        }
      }
      li = nxt;
    }
    PROBE(if (NR == 1 && WP == 0) {
      atomicAdd(&g_probe[8], pclk() - pt0);
      atomicAdd(&g_probe[9], pwait);
      atomicAdd(&g_probe[10], (unsigned long long)n);
      atomicAdd(&g_probe[14], pitems);
    })
    const int s = n % G::STAGES;
    if (n >= G::STAGES) mbar_wait(&empty[s], ((n / G::STAGES) & 1) ^ 1);
    reinterpret_cast<Meta *>(smem + s * G::STAGE + G::WBUF + G::XBUF)->kind = 1;
    mbar_arrive(&full[s]);
    return;
  }
  if constexpr (WP == 0 && use_mma<NR>()) {
    p2_mma_consumer<NR, G>(a, smem, full, empty, red, warp, lane);
    return;
  }
#if HH_MV_VEC1
  if constexpr (WP == 0 && NR == 1) {
    p2_consumer_nr1<G>(a, smem, full, empty, threadIdx.x, lane);
    return;
  }
#endif
  // --------------------------------------------------------------------- consumers
  constexpr int MB = mblock<NR>();
  const int tid = threadIdx.x;
  int cur_nr = -1, nr2 = 1, Gn = 1, rr = 0, g = 0;
  A acc[MB][NR];
#pragma unroll
  for (int b = 0; b < MB; ++b)
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[b][k] = wp_zero<A>();
  for (int n = 0;; ++n) {
    const int s = n % G::STAGES;
    mbar_wait(&full[s], (n / G::STAGES) & 1);
    const uint8_t *st = smem + s * G::STAGE;
    const Meta m = *reinterpret_cast<const Meta *>(st + G::WBUF + G::XBUF);
    if (m.kind) break;
    const int nr = m.a;
    if (nr != cur_nr) {  // thread layout of this leaf size (divisions only when it changes)
      cur_nr = nr;
      nr2 = (nr + MB - 1) / MB;  // thread row slot rr owns rows rr + b * nr2
      Gn = NCT / nr2;            // column groups (nr <= 256: leaf_size limit)
      rr = tid % nr2;
      g = tid / nr2;
    }
    bool valid[MB];
#pragma unroll
    for (int b = 0; b < MB; ++b) valid[b] = g < Gn && rr + b * nr2 < nr;
    if (g < Gn) {
      const uint8_t *ust = st + m.wlead;
      const double *zst = reinterpret_cast<const double *>(st + G::WBUF + m.xlead);
      const int ncols = m.r1 - m.r0;
      const int cnt = g < ncols ? (ncols - g + Gn - 1) / Gn : 0;
      const int e0 = g * nr + rr;
      dispatch_tag(m.b & 0xff, [&](auto t) {
        constexpr int TG = decltype(t)::value;
        block_acc<TG, NR, MB, A>(reinterpret_cast<const typename Elem<TG>::T *>(ust) + e0, zst + g * NR, cnt,
                                 Gn * nr, nr2, Gn * NR, valid, acc);
      });
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (m.flags & 1) {  // last stage of the leaf: fixed-order reduction over groups, scatter (a10)
#pragma unroll
      for (int b = 0; b < MB; ++b)
#pragma unroll
        for (int k = 0; k < NR; ++k) red[(tid * MB + b) * NR + k] = wp_out<A>(acc[b][k]);
      consumer_sync();
      if (tid < nr2) {
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          const int r = tid + b * nr2;
          if (r < nr) {
            A sum[NR];
#pragma unroll
            for (int k = 0; k < NR; ++k) sum[k] = wp_zero<A>();
            for (int gg = 0; gg < Gn; ++gg)
#pragma unroll
              for (int k = 0; k < NR; ++k) sum[k] = wp_add(sum[k], wp_round<A>(red[((gg * nr2 + tid) * MB + b) * NR + k]));
            const int64_t i = a.perm[m.p + r];
#pragma unroll
            for (int k = 0; k < NR; ++k) a.y[i + k * a.ldy] = wp_out<A>(sum[k]);
          }
        }
      }
      consumer_sync();
#pragma unroll
      for (int b = 0; b < MB; ++b)
#pragma unroll
        for (int k = 0; k < NR; ++k) acc[b][k] = wp_zero<A>();
    }
  }
}

}  // namespace mv

// launch with the programmatic-stream-serialization attribute (see pdl_wait)
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = HH_MV_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HH_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

template <int NR, int WP, int GV1, int GV2>
void matvec_chunk_g(hh_matrix *H, const double *x, double *y, int col0, cudaStream_t st) {
  using namespace mv;
  using G1 = Geo<NR, 1, GV1>;
  using G2 = Geo<NR, 2, GV2>;
  // launch geometry (device attributes, smem opt-in, occupancy) once per handle, width and
  // working precision
  hh_matrix::LaunchCfg &L = H->lcfg[WP][NR == 1 ? 0 : NR == 2 ? 1 : NR == 4 ? 2 : NR == 8 ? 3 : 4];
  if (!L.ready) {
    int dev = 0;
    HH_CUDA(cudaGetDevice(&dev));
    HH_CUDA(cudaDeviceGetAttribute(&L.nsm, cudaDevAttrMultiProcessorCount, dev));
    HH_CUDA(cudaFuncSetAttribute(k_phase1<NR, WP, GV1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G1::smem(false)));
    HH_CUDA(cudaFuncSetAttribute(k_phase2<NR, WP, GV2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G2::smem(true)));
    int p1 = 0, p2 = 0;
    HH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, k_phase1<NR, WP, GV1>, THREADS, G1::smem(false)));
    HH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, k_phase2<NR, WP, GV2>, THREADS, G2::smem(true)));
    L.grid1 = (int)std::min<int64_t>(H->n_p1_tiles, (int64_t)L.nsm * std::max(1, p1));
    L.grid2 = (int)std::min<int64_t>(H->n_p2_leaves, (int64_t)L.nsm * std::max(1, p2));
    L.ready = true;
  }
  const int nsm = L.nsm;
  double *v = H->v.as<double>();
  int *ctr = H->ctr.as<int>();
  cudaEvent_t ev[4];
  auto mark = [&](int i) {
    if (!H->prof) return;
    HH_CUDA(cudaEventCreate(&ev[i]));
    HH_CUDA(cudaEventRecord(ev[i], st));
    H->prof_ev.push_back(ev[i]);
  };
  mark(0);
  // a7 gather (+ counter reset)
  launch_pdl(k_gather<NR, WP>, nsm * 8, 256, 0, st, H->d_perm.as<int32_t>(), x + (int64_t)col0 * H->N, H->N, H->N,
             v, ctr);
  HH_LAUNCHED();
  mark(1);
  // a8 phase 1
  if (H->n_p1_tiles > 0) {
    P1Args a{};
    a.tiles = H->p1_tiles.as<P1Tile>();
    a.zmap = H->zmap.as<int32_t>();
    a.partial = H->partial.as<double>();
    a.ntiles = H->n_p1_tiles;
    for (int g = 0; g < NTAG; ++g) a.W[g] = H->W[g].as<uint8_t>();
    a.v = v;
    a.N = H->N;
    a.ctr = ctr;
    a.plan = PlanArgs{H->st_item[0].as<StageItem>(), H->st_copy[0].as<StageCopy>(), H->st_meta[0].as<StageMeta>()};
    launch_pdl(k_phase1<NR, WP, GV1>, (unsigned)L.grid1, THREADS, G1::smem(false), st, a);
    HH_LAUNCHED();
    if (H->n_p1_comb > 0) {
      launch_pdl(k_p1_combine<NR, WP>, (unsigned)std::min<int64_t>(H->n_p1_comb, (int64_t)nsm * 8), 256, 0, st,
                 H->p1_comb.as<P1Combine>(), H->n_p1_comb, a.zmap, a.partial, v, H->N);
      HH_LAUNCHED();
    }
  }
  mark(2);
  // a9 + a10 phase 2 with fused scatter
  P2Args b{};
  b.leaves = (NR >= HH_MV_P2MORTON_NR ? H->p2_leaves_mo : H->p2_leaves).as<P2Leaf>();
  b.segs = H->p2_segs.as<P2Seg>();
  b.nleaves = H->n_p2_leaves;
  for (int g = 0; g < NTAG; ++g) b.U[g] = H->U[g].as<uint8_t>();
  b.D = H->D.as<uint8_t>();
  b.v = v;
  b.perm = H->d_perm.as<int32_t>();
  b.y = y + (int64_t)col0 * H->N;
  b.ldy = H->N;
  b.ctr = ctr;
  b.plan = PlanArgs{H->st_item[1].as<StageItem>(), H->st_copy[1].as<StageCopy>(), H->st_meta[1].as<StageMeta>()};
  if (L.grid2 > 0) {
    launch_pdl(k_phase2<NR, WP, GV2>, (unsigned)L.grid2, THREADS, G2::smem(true), st, b);
    HH_LAUNCHED();
  }
  mark(3);
}

// the planned single-RHS product runs the stage geometry its plan was built for (hh_matrix::geom)
template <int NR, int WP = 0>
void matvec_chunk(hh_matrix *H, const double *x, double *y, int col0, cudaStream_t st) {
  if constexpr (mv::planned<NR, WP>()) {
    const int g1 = H->geom[0], g2 = H->geom[1];
    if (g1 && g2) return matvec_chunk_g<1, 0, 1, 1>(H, x, y, col0, st);
    if (g1) return matvec_chunk_g<1, 0, 1, 0>(H, x, y, col0, st);
    if (g2) return matvec_chunk_g<1, 0, 0, 1>(H, x, y, col0, st);
  }
  matvec_chunk_g<NR, WP, 0, 0>(H, x, y, col0, st);
}

template <int WP>
void run_matvec_wp(hh_matrix *H, const double *x, double *y, int nrhs, cudaStream_t st) {
  // reduced working precision: FMA consumers only, chunks of <= 4 columns
  int col = 0;
  while (col < nrhs) {
    const int rem = nrhs - col;
    if (rem >= 4) {
      matvec_chunk<4, WP>(H, x, y, col, st);
      col += 4;
    } else if (rem >= 2) {
      matvec_chunk<2, WP>(H, x, y, col, st);
      col += 2;
    } else {
      matvec_chunk<1, WP>(H, x, y, col, st);
      col += 1;
    }
  }
}

#if HH_MV_PROBE
}  // namespace hh
// variant builds only: read (and optionally reset) the cycle probe
extern "C" int hh_debug_probe(unsigned long long *out, int reset) {
  if (out && cudaMemcpyFromSymbol(out, hh::mv::g_probe, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(hh::mv::g_probe, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
namespace hh {
#endif

void run_matvec(hh_matrix *H, const double *x, double *y, int nrhs, cudaStream_t st, int wp) {
  if (wp == 1) return run_matvec_wp<1>(H, x, y, nrhs, st);
  if (wp == 2) return run_matvec_wp<2>(H, x, y, nrhs, st);
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
