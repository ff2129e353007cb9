/*
 * hh.h — C-ABI of libhh: adaptive mixed-precision hybrid hierarchical (H_h) matrices on
 * one NVIDIA B200 (sm_100a).  arxiv 2604.09147 ("Adaptive mixed precision H_h matrices").
 *
 * The library builds, on the device, the H_h representation of the kernel matrix
 *     H_ij = f(||x_i - x_j||_2)                                   (Eq. 5.1)
 * of N points in R^d, and applies it:  y = H-hat x                (Alg. 3).
 *
 * Construction (hh_build) follows
 *   - the balanced 2^d-tree
 *   - hybrid admissibility Eq. 3.1: standard below the switch level, weak from it
 *                                                                  PAPER.md:394-403, 552-557
 *   - Alg. 1: every admissible block compressed to relative Frobenius accuracy eps
 *     (rank = truncated-SVD rank), leaf diagonal blocks dense
 *                                                                  PAPER.md:562-619
 *   - Alg. 4: ||H~||^2 from the kept singular values
 *   - Alg. 2 / Eq. 4.4: per-block storage precision, the largest u in the precision set with
 *     u <= eps / (2^{dl/2} xi), xi = ||H~_IJ||/||H~||
 * and packs the factors into per-precision HBM arenas (layout: DESIGN.md §4).  hh_build runs
 * libhh's own kernels and, for large blocks with wide sketches only, cuBLAS DGEMM and
 * cuSOLVER QR/SVD (compress_big.cu); hh_matvec runs only libhh's sm_100a kernels.
 *
 * Conventions shared by every entry point
 *   - Pointers documented as "device" must be cudaMalloc'd (or torch CUDA) memory on the
 *     current device; "host" pointers are ordinary CPU memory (pinned memory is faster).
 *   - Arrays are little-endian, float64 unless stated; N x d point arrays are row-major;
 *     N x nrhs vector blocks are column-major with leading dimension N, ORIGINAL point order.
 *   - Every call returns hh_status; nothing throws or aborts across the ABI.  On a non-OK
 *     status hh_last_error() returns a thread-local message.
 *   - There is no CPU fallback: without a usable CUDA device every call that needs one
 *     returns HH_ECUDA.
 */
#ifndef HH_H
#define HH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hh_matrix *hh_handle;   /* opaque, library-owned */

typedef enum {
  HH_OK = 0,
  HH_EINVAL = 1,        /* invalid argument (see each call) */
  HH_ENOMEM = 2,        /* device or host allocation failed */
  HH_ECUDA = 3,         /* CUDA runtime/kernel error, or no usable device */
  HH_ENUMERIC = 4,      /* non-finite input point / vector / kernel entry */
  HH_EDEPTH = 5,        /* d*L would exceed 62 bits before every leaf holds <= leaf_size points */
  HH_EUNSUPPORTED = 6   /* outside what this build supports (e.g. 2^{dL} > 2^26 leaf cells) */
} hh_status;

/* Kernel functions f(r) (length scale: reading G19).
 * LOG, INV_R, INV_R2 are singular: H_ii = 0.  GAUSS/EXP: H_ii = 1. */
typedef enum {
  HH_K_LOG = 0,     /* log r                    */
  HH_K_INV_R = 1,   /* 1 / r                    */
  HH_K_INV_R2 = 2,  /* 1 / r^2                  */
  HH_K_GAUSS = 3,   /* exp(-r^2 / (2 scale^2))  */
  HH_K_EXP = 4      /* exp(-r / scale)          */
} hh_kernel_kind;

typedef struct {
  int32_t kind;     /* hh_kernel_kind */
  double scale;     /* length scale for GAUSS / EXP; ignored otherwise */
} hh_kernel;

/* precision_set bitmask (Table 1); FP64 (the working precision) is mandatory.
 * NEXT-3 opt-in formats:
 *   HH_P_Q43  Table 1's 8-bit q43 = (1-4-3), e_min -6, e_max 7, x_max 240, u = 2^-4 (reading G12),
 *             1 byte per element with the OCP FP8 E4M3 encoding (identical for |x| <= 240; the
 *             range guard promotes anything that rounds above 240);
 *   HH_P_BF24 / HH_P_FP48  the "memory accessor" continuum of PAPER.md:933 (§4.2 remark after
 *             Eq. 4.4) at byte granularity: bf24 = (1-8-15), u = 2^-16, 3 bytes = the top 24 bits
 *             of an fp32; fp48 = (1-11-36), u = 2^-37, 6 bytes = the top 48 bits of an fp64.
 *             Stored by single RNE rounding, up-converted exactly (reading G28). */
enum { HH_P_FP64 = 1u, HH_P_FP32 = 2u, HH_P_FP16 = 4u, HH_P_BF16 = 8u, HH_P_Q43 = 16u, HH_P_BF24 = 32u,
       HH_P_FP48 = 64u, HH_P_ALL = 127u };
/* tag ids used in exported tables */
enum { HH_TAG_FP64 = 0, HH_TAG_FP32 = 1, HH_TAG_FP16 = 2, HH_TAG_BF16 = 3, HH_TAG_Q43 = 4, HH_TAG_BF24 = 5,
       HH_TAG_FP48 = 6, HH_NTAG = 7 };
/* OR into precision_set: compute ranks / tags / norms / byte ledger only, store no factors
 * (hh_matvec then returns HH_EINVAL).  Used for storage ratios of configurations that do
 * not fit in HBM (uniform-fp64 H_s at N = 2^20). */
#define HH_LEDGER_ONLY (1u << 16)
/* OR into precision_set (NEXT-3, bits-aware tie rule): when Eq. 4.4 admits bf16 it also admits
 * fp16 (smaller u, same 16 bits); the paper keeps the largest u (bf16) —
 * with this flag the block is stored in fp16 (3 more mantissa bits) unless an entry would
 * overflow fp16, in which case bf16 stays.  Requires both HH_P_FP16 and HH_P_BF16. */
#define HH_TIE_FP16 (1u << 17)

/* switch_level: 0..L is Eq. 3.1 read literally (0 = HODLR); HH_SWITCH_NONE = pure H_s
 * (Alg. 1 with ell = L: dense leaf neighbours; in mixed precision a leaf neighbour is stored
 * low-rank iff that is smaller in bits). */
#define HH_SWITCH_NONE (-1)

/* Block kinds (exported tables) */
enum { HH_KIND_FAR = 0, HH_KIND_NBR = 1, HH_KIND_SIB = 2, HH_KIND_LNBR = 3, HH_KIND_DIAG = 4 };
enum { HH_STORE_LR = 0, HH_STORE_DENSE = 1 };

/*
 * hh_build — construct H-hat on the device.
 *   points        device, N x d row-major float64, finite.  Read during the call only.
 *   N, d          N >= 1, 1 <= d <= 3 in this build (HH_EUNSUPPORTED otherwise).
 *   kernel        see hh_kernel.
 *   eps           target accuracy, 2^-53 < eps < 1 ("u < eps").
 *   eta           admissibility parameter > 0 (Eq. 2.1); eta^2 within 1e-12 of an
 *                 integer is snapped to it.
 *   leaf_size     n_max >= 1: depth L = smallest L with every leaf holding <= n_max points.
 *   switch_level  0..L, or HH_SWITCH_NONE.  > L -> HH_EINVAL.
 *   precision_set bitmask of HH_P_*, must contain HH_P_FP64; may OR HH_LEDGER_ONLY.
 *   cuda_stream   cudaStream_t (NULL = legacy default stream).  hh_build synchronises it.
 *   out           receives the handle on HH_OK (unchanged otherwise).
 * Ownership: the handle owns every device allocation it makes — the per-tag factor arenas and
 * the dense arena (hh_info_t: w_bytes, u_bytes, d_bytes), the block and plan tables, the matvec
 * workspace ([x~ ; z] for 16 right-hand sides) and the precomputed stage plan of the single-RHS
 * product (96 bytes per streamed shared-memory stage, about 0.35% of the stored bytes) — until
 * hh_free.  Nothing is allocated inside hh_matvec.
 * Sketch limit: the device compressor widens a block's randomized sketch until its rank decision
 * provably equals the truncated-SVD decision (G26).  If a block reaches the 4096-column
 * limit (below min(|I|, |J|)) with a decision that is valid (the explicit residual meets eps) but
 * not proved minimal, the rank is accepted and counted in hh_info_t.n_inexact.
 * Errors: HH_EUNSUPPORTED if a block's rank exceeds 4096 columns (no sketch of <= 4096 columns
 * meets eps), or a whole-GPU-path block needs more device memory than is free, HH_EINVAL (bad argument), HH_ENUMERIC (non-finite point or kernel entry, e.g.
 * log of a zero distance between distinct points is mapped to 0 and counted — not an
 * error — but an overflowing entry is), HH_EDEPTH, HH_ENOMEM (arenas exceed free HBM),
 * HH_ECUDA.
 */
hh_status hh_build(const double *points, int64_t N, int32_t d, hh_kernel kernel, double eps,
                   double eta, int32_t leaf_size, int32_t switch_level, uint32_t precision_set,
                   void *cuda_stream, hh_handle *out);

/*
 * hh_matvec — y = H-hat x (Alg. 3), fp64 working precision.
 *   x      device, N x nrhs column-major (ld = N), original point order.  Not modified.
 *   y      device, same layout; overwritten; must not overlap x.
 *   nrhs   >= 1 (processed in chunks of <= 16 columns).
 *   stream cudaStream_t; the call only enqueues work (asynchronous w.r.t. the host).
 * The result is bitwise reproducible: no atomics, fixed summation order.
 * Concurrent calls on one handle are not allowed (shared workspace).
 * Errors: HH_EINVAL (NULL pointers, nrhs < 1, x == y, ledger-only handle), HH_ECUDA.
 */
hh_status hh_matvec(hh_handle H, const double *x, double *y, int32_t nrhs, void *cuda_stream);

/*
 * hh_matvec_wp — Alg. 3 in a lower working precision u (NEXT-3: the backward-error study of
 * PAPER.md:1266-1285, Thm 4.4 at PAPER.md:1028-1040, "this u may differ from the u used in
 * Alg. 2").  Reading G27: x and every stored factor / dense entry enter rounded
 * once (RNE) to the working format (exact when the storage format is narrower), every
 * multiply-add is one fused multiply-add rounded to it, z and all partial sums are held in it,
 * and y receives its working-precision values as float64.  The summation order is the
 * library's (fixed, deterministic; the paper fixes none).  Arguments as hh_matvec;
 * working_precision = HH_WP_FP64 (identical to hh_matvec), HH_WP_FP32 or HH_WP_FP16.  Reduced
 * precisions run chunks of <= 4 columns on the FMA pipes (no FP64 tensor cores).
 * Errors: as hh_matvec; HH_EINVAL for an unknown working_precision.
 */
enum { HH_WP_FP64 = 0, HH_WP_FP32 = 1, HH_WP_FP16 = 2 };
hh_status hh_matvec_wp(hh_handle H, const double *x, double *y, int32_t nrhs, int32_t working_precision,
                       void *cuda_stream);

/*
 * hh_matvec_host — same product with HOST x and y: copies x host->device, runs hh_matvec
 * and copies y device->host on `stream`, then synchronises it (the end-to-end path).
 */
hh_status hh_matvec_host(hh_handle H, const double *x_host, double *y_host, int32_t nrhs,
                         void *cuda_stream);

/*
 * hh_matvec_profile / hh_matvec_timing — optional per-phase device timing of hh_matvec (used
 * by bench.py for the roofline).  While enabled, every hh_matvec records CUDA events on the
 * caller's stream around its gather (a7), phase 1 (a8, incl. the combine of split columns)
 * and phase 2 (a9 + fused scatter a10).  hh_matvec_timing synchronises on the last event and
 * returns, summed over the matvec chunks recorded since the previous call, ms[0] = gather,
 * ms[1] = phase 1, ms[2] = phase 2, ms[3] = their sum; *count = number of chunks (may be NULL).
 */
hh_status hh_matvec_profile(hh_handle H, int32_t enable);
hh_status hh_matvec_timing(hh_handle H, double *ms, int64_t *count);

/*
 * hh_switch_level_search — Alg. 5 (alg:algo_optimal_level): the switching
 * level ell* maximising S_1(ell) - S_2(ell) (Eqs. S1/S2), i.e. the H_h with the
 * least storage relative to the pure standard H (H_s).  Bottom-up as in the paper: ell = L
 * (Alg. 1's ell = L branch is H_s, so S_1(L) = S_2(L)), then ell - 1 while the gain
 * S_s - S_h(ell - 1) grows.  Storage comes from ledger-only builds (ranks, tags and bytes,
 * nothing stored), counted in each block's storage bits — the mixed-precision variant the
 * paper leaves open; with precision_set = HH_P_FP64 it is the uniform one.
 *   points, N, d, kernel, eps, eta, leaf_size, precision_set, cuda_stream: as hh_build.
 *   out_level  receives ell* in [0, L]; ell* = L means H_s (build it with HH_SWITCH_NONE).
 *   bytes      optional host int64 array of bytes_len >= L + 2 entries: bytes[l] = S_h(l) for the
 *              levels visited (-1 for the others), bytes[L + 1] = S_s.  NULL to skip;
 *              HH_EINVAL if bytes_len is too small (L is reported in out_L when non-NULL).
 */
hh_status hh_switch_level_search(const double *points, int64_t N, int32_t d, hh_kernel kernel, double eps,
                                 double eta, int32_t leaf_size, uint32_t precision_set, void *cuda_stream,
                                 int32_t *out_level, int32_t *out_L, int64_t *bytes, int32_t bytes_len);

/* Summary of a built handle (always available, host memory, filled by hh_info). */
typedef struct {
  int32_t d, L, switch_level, kernel_kind;
  int64_t N;
  double eta, eps, kernel_scale;
  uint32_t precision_set;
  int32_t ledger_only;
  int64_t n_cells;            /* 2^{dL} leaf cells (empty ones included) */
  int64_t nblocks;            /* all blocks, incl. leaf diagonals, canonical order */
  int64_t n_lowrank, n_dense;
  int64_t total_rank;         /* sum of ranks = length of the z workspace */
  double norm2;               /* ||H~||_F^2 (Alg. 4) */
  int64_t w_bytes[7];         /* W arena sizes per tag 0..6 (padded) */
  int64_t u_bytes[7];         /* U arena sizes per tag 0..6 (padded) */
  int64_t d_bytes;            /* dense fp64 arena size (padded) */
  int64_t stored_bytes;       /* algorithmic: sum p(|I|+|J|) bytes(tag) + sum |I||J| 8 */
  int64_t stored_bytes_tag[8];/* the same split by tag 0..6 and 7 = dense */
  int64_t padded_bytes;       /* bytes actually streamed by a matvec (arenas incl. padding) */
  int32_t c_far, c_nbr, c_sib;/* measured sparsity constants (max blocks per target) */
  int64_t n_fallback, n_promoted, n_coincident, n_retry;
  double build_seconds;
  int64_t n_inexact;          /* blocks whose rank decision could not be proved equal to the truncated-SVD
                                 rank within the 4096-column sketch limit (accepted; see hh_build) */
} hh_info_t;

hh_status hh_info(hh_handle H, hh_info_t *info);

/* Exported block record (canonical order: level, tgt, src). */
typedef struct {
  int64_t tgt, src;           /* Morton codes of target / source cluster at `level` */
  int64_t zoff;               /* offset in z (low-rank), -1 otherwise */
  int64_t w_off;              /* byte offset of the block's source panel in W[tag] (rank > 0), -1 otherwise */
  int64_t wcol;               /* first column of the block inside that panel, -1 otherwise */
  int64_t ucol;               /* first column inside the target's leaf streams, -1 otherwise */
  int64_t d_off;              /* byte offset in the dense arena (dense blocks), -1 otherwise */
  double nb2;                 /* ||H~_b||_F^2 = sum of kept sigma^2 (low-rank) */
  double tot;                 /* ||H_b||_F^2 (computed from the entries) */
  double maxabs;              /* max |entry| over the unrounded factors */
  int32_t rank;
  uint8_t level, kind, tag, storage;
} hh_block_t;

/*
 * hh_export — copy tables and arena bytes to host memory.
 * Two-call protocol: call with every pointer NULL to get sizes via hh_info (or read
 * out->info); then set the pointers you want and call again.  Each pointer may be NULL
 * (skipped).  Arena windows: `arena` selects 0..6 = W[tag], 7..13 = U[tag], 14 = dense,
 * bytes [arena_off, arena_off + arena_len) are copied to arena_dst.
 */
typedef struct {
  hh_info_t info;             /* always filled */
  int32_t *perm;              /* [N]   tree position -> original index */
  int64_t *leaf_start;        /* [n_cells + 1] */
  hh_block_t *blocks;         /* [nblocks] */
  int64_t *u_leaf_off;        /* [HH_NTAG * (n_cells + 1)] byte offsets of leaf streams per tag */
  int64_t *d_leaf_off;        /* [n_cells + 1] */
  int32_t arena;
  int64_t arena_off, arena_len;
  void *arena_dst;
} hh_export_t;

hh_status hh_export(hh_handle H, hh_export_t *out);

/* hh_free — release every device and host resource of the handle (NULL is a no-op). */
hh_status hh_free(hh_handle H);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char *hh_last_error(void);

/* Test hook: the device storage-rounding routine of `tag` (HH_TAG_FP32/FP16/BF16/Q43/BF24) applied to
 * n host doubles; host_bits receives the target bit patterns (RNE, single rounding, G16). */
hh_status hh_selftest_round(const double *host_in, int64_t n, int32_t tag, uint32_t *host_bits);

/*
 * Test hooks on the library's host-side C++ (no device needed; used by the CPU test suite):
 *   hh_selftest_partition — the block partition (partition.cpp: Eq. 3.1 expansion, canonical
 *     order) of a tree given by its leaf offsets leaf_start[2^{dL}+1].  Writes up to
 *     `capacity` blocks (level, kind, tgt, src) and the total count to *nblocks (HH_EINVAL if
 *     capacity is too small: call with capacity 0 to size).
 *   hh_selftest_layout — the packing function (layout.cpp) for given blocks,
 *     ranks, tags and storage kinds: every offset hh_export reports, u_leaf_off[HH_NTAG*(ncell+1)],
 *     d_leaf_off[ncell+1] and w_bytes[HH_NTAG].
 */
hh_status hh_selftest_partition(const int64_t *leaf_start, int32_t d, int32_t L, double eta, int32_t switch_level,
                                int64_t capacity, int64_t *nblocks, uint8_t *level, uint8_t *kind, int64_t *tgt,
                                int64_t *src);
hh_status hh_selftest_layout(const int64_t *leaf_start, int32_t d, int32_t L, int64_t nblocks, const uint8_t *level,
                             const int64_t *tgt, const int64_t *src, const int32_t *rank, const uint8_t *tag,
                             const uint8_t *storage, int64_t *zoff, int64_t *w_off, int64_t *wcol, int64_t *ucol,
                             int64_t *d_off, int64_t *u_leaf_off, int64_t *d_leaf_off, int64_t *w_bytes);

/*
 * hh_selftest_tags — the library's host-side Alg. 4 norm + Alg. 2 / Eq. 4.4 tagging (layout.cpp:
 * assign_tags: squared exact form, range guard, HH_TIE_FP16, PAPER.md:992 beneficial rule) on
 * given per-block ranks, ||H~_b||^2 (nb2), ||H_b||^2 (tot) and factor max |entry| (maxabs), with the
 * storage kinds hh_build starts from (diagonal dense; leaf neighbours dense in uniform precision).
 * Outputs tag[], storage[], rank[] (in/out: 0 for neighbours the beneficial rule keeps dense),
 * *norm2 = ||H~||^2 and counts[0] = n_fallback, counts[1] = n_promoted.  No device needed.
 */
hh_status hh_selftest_tags(const int64_t *leaf_start, int32_t d, int32_t L, int64_t nblocks, const uint8_t *level,
                          const uint8_t *kind, const int64_t *tgt, const int64_t *src, int32_t *rank,
                          const double *nb2, const double *tot, const double *maxabs, double eps,
                          uint32_t precision_set, uint8_t *tag, uint8_t *storage, double *norm2, int64_t *counts);

/* Number of kernels the library enqueued since load (launch accounting for bench.py). */
int64_t hh_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* HH_H */
