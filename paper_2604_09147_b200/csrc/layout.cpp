// layout.cpp — §8(a) rows a4–a6 (host side): global norm, precision tags, packing function,
// and the matvec work plan.
//
//   a4  ||H~||^2 = sum_b nb2_b over low-rank blocks + sum ||H_b||^2 over dense blocks; for
//       pure H_s the leaf neighbours enter with their direct norm (Alg. 4).
//   a5  Eq. 4.4 / Alg. 2 in squared exact form (G15):
//           u^2 2^{d l} nb2_b <= eps^2 ||H~||^2,  largest such u in the precision set;
//       none -> fp64 (fallback); range guard promotes when a factor entry would overflow;
//       pure H_s mixed: leaf neighbour low-rank iff p(|I|+|J|) bits < |I||J| 64.
//   a6  packing function — the C++ twin of the oracle's pack.py, written
//       independently; check (1c) compares them bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <vector>

#include "build.h"

namespace hh {

static const double kU[NTAG] = {0x1p-53, 0x1p-24, 0x1p-11, 0x1p-8, 0x1p-4, 0x1p-16, 0x1p-37};
static const uint32_t kBit[NTAG] = {HH_P_FP64, HH_P_FP32, HH_P_FP16, HH_P_BF16, HH_P_Q43, HH_P_BF24, HH_P_FP48};
// formats in decreasing unit roundoff (the order Eq. 4.4 tries them; the range guard steps right)
static const int kByU[NTAG] = {TAG_Q43, TAG_BF16, TAG_FP16, TAG_BF24, TAG_FP32, TAG_FP48, TAG_FP64};

void cluster_range(const hh_matrix *H, int l, int64_t m, int64_t &a, int64_t &n) {
  const int sh = H->d * (H->L - l);
  a = H->leaf_start[m << sh];
  n = H->leaf_start[(m + 1) << sh] - a;
}

// Range guard (G16): does the single RNE rounding of |x| to format `tag` overflow to inf?  Decided
// by the same rounding routine that stores the factors (common.cuh), not by a threshold table.
static bool overflows(int tag, double x) {
  switch (tag) {
    case TAG_FP32: return (to_fp32_bits(x) & 0x7FFFFFFFu) == 0x7F800000u;
    case TAG_FP16: return (to_fp16_bits(x) & 0x7FFFu) == 0x7C00u;
    case TAG_BF16: return (to_bf16_bits(x) & 0x7FFFu) == 0x7F80u;
    case TAG_Q43: return (to_q43_bits(x) & 0x7Fu) == 0x78u;
    case TAG_BF24: return (to_bf24_bits(x) & 0x7FFFFFu) == 0x7F8000u;
    case TAG_FP48: return (to_fp48_bits(x) & 0x7FFFFFFFFFFFull) == 0x7FF000000000ull;
    default: return false;
  }
}

void assign_tags(hh_matrix *H) {
  const size_t nb = H->level.size();
  const bool mixed = (H->pset & HH_P_ALL) != HH_P_FP64;
  // a4: global norm in canonical order
  double norm2 = 0.0;
  for (size_t b = 0; b < nb; ++b) {
    const int k = H->kind[b];
    norm2 += (k == KIND_DIAG || k == KIND_LNBR) ? H->tot[b] : H->nb2[b];
  }
  H->norm2 = norm2;
  const double rhs = (H->eps * H->eps) * norm2;
  int64_t fb = 0, pr = 0;
  for (size_t b = 0; b < nb; ++b) {
    if (H->storage[b] != STORE_LR) continue;
    const int l = H->level[b];
    int tag = TAG_FP64;
    bool found = false;
    for (int t : kByU) {
      if (!(H->pset & kBit[t])) continue;
      const double u = kU[t];
      if ((u * u) * std::ldexp(1.0, H->d * l) * H->nb2[b] <= rhs) {
        tag = t;
        found = true;
        break;
      }
    }
    fb += !found;
    // NEXT-3 tie rule: fp16 instead of bf16 (same bits, smaller u) unless fp16 would overflow
    if (H->tie16 && tag == TAG_BF16 && !overflows(TAG_FP16, H->maxabs[b])) tag = TAG_FP16;
    // range guard: promote while the largest factor entry would overflow the format (the
    // promoted counter counts blocks, however many steps they take)
    bool promoted = false;
    while (tag != TAG_FP64 && overflows(tag, H->maxabs[b])) {
      int i = 0;
      while (kByU[i] != tag) ++i;
      do ++i;
      while (kByU[i] != TAG_FP64 && !(H->pset & kBit[kByU[i]]));
      tag = kByU[i];
      promoted = true;
    }
    pr += promoted;
    H->tag[b] = (uint8_t)tag;
    if (H->kind[b] == KIND_LNBR && mixed) {
      int64_t i0, m, j0, n;
      cluster_range(H, l, H->tgt[b], i0, m);
      cluster_range(H, l, H->src[b], j0, n);
      const int bits = 8 * tag_bytes(tag);
      if (!((int64_t)H->rank[b] * (m + n) * bits < m * n * 64)) {
        H->storage[b] = STORE_DENSE;
        H->rank[b] = 0;
        H->tag[b] = TAG_FP64;
      }
    }
  }
  H->info.n_fallback = fb;
  H->info.n_promoted = pr;
}

// a6: packing function.  Fills zoff, w_off, ucol, u_leaf_off, d_off, d_leaf_off and sizes.
void compute_layout(hh_matrix *H) {
  const size_t nb = H->level.size();
  const int d = H->d, L = H->L;
  const int64_t ncell = H->ncell;
  H->zoff.assign(nb, -1);
  H->w_off.assign(nb, -1);
  H->ucol.assign(nb, -1);
  H->d_off.assign(nb, -1);
  std::vector<int64_t> I0(nb), M(nb), J0(nb), Nn(nb);
  for (size_t b = 0; b < nb; ++b) {
    cluster_range(H, H->level[b], H->tgt[b], I0[b], M[b]);
    cluster_range(H, H->level[b], H->src[b], J0[b], Nn[b]);
  }
  auto is_lr = [&](size_t b) { return H->storage[b] == STORE_LR; };
  // z: (level, tgt, tag, src); canonical order is (level, tgt, src): stable-sort by tag
  // inside each (level, tgt) run
  {
    int64_t z = 0;
    size_t b = 0;
    while (b < nb) {
      size_t e = b;
      while (e < nb && H->level[e] == H->level[b] && H->tgt[e] == H->tgt[b]) ++e;
      for (int t = 0; t < NTAG; ++t)
        for (size_t i = b; i < e; ++i)
          if (is_lr(i) && H->tag[i] == t) {
            H->zoff[i] = z;
            z += H->rank[i];
          }
      b = e;
    }
    H->ztotal = z;
  }
  // W[g]: panels.  Tag-g low-rank blocks with p > 0 in (level, src, tgt) order; a run of
  // equal (level, src) is one panel of |J| rows and P = sum p columns; block b occupies panel
  // columns [wcol, wcol + p).  Column tiles of W_CT columns (the last one narrower), each
  // stored row-major, start at multiples of ALIGN.  w_off[b] = byte offset of b's panel.
  H->wcol.assign(nb, -1);
  H->wpanel.assign(nb, -1);
  {
    std::vector<size_t> idx;
    for (size_t b = 0; b < nb; ++b)
      if (is_lr(b) && H->rank[b] > 0) idx.push_back(b);
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t c) {
      if (H->tag[a] != H->tag[c]) return H->tag[a] < H->tag[c];
      if (H->level[a] != H->level[c]) return H->level[a] < H->level[c];
      if (H->src[a] != H->src[c]) return H->src[a] < H->src[c];
      return H->tgt[a] < H->tgt[c];
    });
    int64_t off[NTAG] = {};
    size_t i = 0;
    while (i < idx.size()) {
      size_t e = i;
      const size_t b0 = idx[i];
      int64_t P = 0;
      while (e < idx.size() && H->tag[idx[e]] == H->tag[b0] && H->level[idx[e]] == H->level[b0] &&
             H->src[idx[e]] == H->src[b0]) {
        const size_t b = idx[e];
        H->wcol[b] = P;
        P += H->rank[b];
        ++e;
      }
      const int g = H->tag[b0];
      for (size_t k = i; k < e; ++k) {
        H->w_off[idx[k]] = off[g];
        H->wpanel[idx[k]] = P;
      }
      const int64_t n = Nn[b0];
      for (int64_t c0 = 0; c0 < P; c0 += W_CT) off[g] += align_up(n * std::min<int64_t>(W_CT, P - c0) * tag_bytes(g));
      i = e;
    }
    for (int g = 0; g < NTAG; ++g) H->w_bytes[g] = off[g];
  }
  // U[g]: per-leaf streams.  Column base of block b = columns of coarser levels of its
  // target's ancestors + prefix inside its (level, tgt, tag) group.
  {
    // group totals per (level, tgt, tag)
    std::vector<std::vector<int64_t>> gtot(L + 1);
    for (int l = 0; l <= L; ++l) gtot[l].assign((size_t)NTAG << (d * l), 0);
    for (size_t b = 0; b < nb; ++b)
      if (is_lr(b) && H->rank[b] > 0) gtot[H->level[b]][(size_t)H->tgt[b] * NTAG + H->tag[b]] += H->rank[b];
    // coarser-level column base per (level, tgt, tag): base[l][t] = sum_{l' < l} gtot[l'][anc(t)]
    std::vector<std::vector<int64_t>> base(L + 1);
    for (int l = 0; l <= L; ++l) {
      base[l].assign((size_t)NTAG << (d * l), 0);
      if (l > 0)
        for (int64_t t = 0; t < (1ll << (d * l)); ++t)
          for (int g = 0; g < NTAG; ++g)
            base[l][t * NTAG + g] = base[l - 1][(t >> d) * NTAG + g] + gtot[l - 1][(t >> d) * NTAG + g];
    }
    size_t b = 0;
    while (b < nb) {
      size_t e = b;
      while (e < nb && H->level[e] == H->level[b] && H->tgt[e] == H->tgt[b]) ++e;
      int64_t within[NTAG] = {};
      for (size_t i = b; i < e; ++i)
        if (is_lr(i) && H->rank[i] > 0) {
          const int g = H->tag[i];
          H->ucol[i] = base[H->level[i]][(size_t)H->tgt[i] * NTAG + g] + within[g];
          within[g] += H->rank[i];
        }
      b = e;
    }
    H->u_leaf_off.assign((size_t)NTAG * (ncell + 1), 0);
    for (int g = 0; g < NTAG; ++g) {
      int64_t off = 0;
      for (int64_t R = 0; R < ncell; ++R) {
        H->u_leaf_off[(size_t)g * (ncell + 1) + R] = off;
        const int64_t nr = H->leaf_start[R + 1] - H->leaf_start[R];
        const int64_t cols = base[L][(size_t)R * NTAG + g] + gtot[L][(size_t)R * NTAG + g];
        off += align_up(nr * cols * tag_bytes(g));
      }
      H->u_leaf_off[(size_t)g * (ncell + 1) + ncell] = off;
      H->u_bytes[g] = off;
    }
  }
  // dense arena: per target leaf, src order, 16-B aligned leaf groups
  {
    H->d_leaf_off.assign(ncell + 1, 0);
    std::vector<int64_t> per(ncell, 0);
    for (size_t b = 0; b < nb; ++b)
      if (H->storage[b] == STORE_DENSE) per[H->tgt[b]] += M[b] * Nn[b] * 8;
    int64_t off = 0;
    for (int64_t R = 0; R < ncell; ++R) {
      H->d_leaf_off[R] = off;
      off += align_up(per[R]);
    }
    H->d_leaf_off[ncell] = off;
    H->d_bytes = off;
    std::vector<int64_t> cur(H->d_leaf_off.begin(), H->d_leaf_off.end() - 1);
    for (size_t b = 0; b < nb; ++b)  // canonical order = (tgt, src) inside level L
      if (H->storage[b] == STORE_DENSE) {
        H->d_off[b] = cur[H->tgt[b]];
        cur[H->tgt[b]] += M[b] * Nn[b] * 8;
      }
  }
  // ledger
  int64_t tagged[NTAG + 1] = {};
  int64_t nlr = 0, nd = 0;
  for (size_t b = 0; b < nb; ++b) {
    if (H->storage[b] == STORE_DENSE) {
      tagged[NTAG] += M[b] * Nn[b] * 8;
      ++nd;
    } else {
      tagged[H->tag[b]] += (int64_t)H->rank[b] * (M[b] + Nn[b]) * tag_bytes(H->tag[b]);
      ++nlr;
    }
  }
  int64_t tot = 0, pad = H->d_bytes;
  for (int i = 0; i <= NTAG; ++i) {
    H->info.stored_bytes_tag[i] = tagged[i];
    tot += tagged[i];
  }
  for (int g = 0; g < NTAG; ++g) pad += H->w_bytes[g] + H->u_bytes[g];
  H->info.stored_bytes = tot;
  H->info.padded_bytes = pad;
  H->info.n_lowrank = nlr;
  H->info.n_dense = nd;
}

// ----------------------------------------------------------------- matvec work plan
// Phase 1: one item per W column tile, largest first (the kernels take items from a work
// counter, so big tiles start early).  zmap[zbase + c] = z index of tile column c.
// Phase 2: per leaf, dense segments then per tag the levels' U column groups; leaves with
// the most bytes first.
void build_plan(hh_matrix *H, std::vector<P1Tile> &tiles, std::vector<int32_t> &zmap, std::vector<P1Combine> &comb,
                int64_t &npartial, std::vector<P2Seg> &segs, std::vector<P2Leaf> &leaves,
                std::vector<P2Leaf> &leaves_morton) {
  const size_t nb = H->level.size();
  const int d = H->d, L = H->L;
  const int64_t N = H->N;
  tiles.clear();
  zmap.clear();
  comb.clear();
  npartial = 0;
  segs.clear();
  leaves.clear();
  HH_REQUIRE(H->ztotal < INT32_MAX, HH_EUNSUPPORTED, "total rank exceeds 2^31");
  // ---- phase 1
  std::vector<size_t> idx;
  for (size_t b = 0; b < nb; ++b)
    if (H->storage[b] == STORE_LR && H->rank[b] > 0) idx.push_back(b);
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t c) {
    if (H->tag[a] != H->tag[c]) return H->tag[a] < H->tag[c];
    if (H->w_off[a] != H->w_off[c]) return H->w_off[a] < H->w_off[c];
    return H->wcol[a] < H->wcol[c];
  });
  std::vector<int64_t> tbytes;
  // Row-split threshold.  A piece should stay below the average share of one resident CTA
  // (~444 on a B200), or the phase ends on a few CTAs still streaming a coarse-level panel:
  // at 2D N=65536 (0.35 GB of W, 4096-row level-2 panels) pieces of 4096 rows took 0.087 ms,
  // pieces of 512 rows 0.071 ms (profiles/r02f_2d_rowsplit_ab.txt).  Large problems keep
  // P1_ROWS.  HH_P1_ROWS overrides it (tests exercise the split on small inputs).
  int64_t split_rows = P1_ROWS;
  if (getenv("HH_P1_ROWS")) {
    split_rows = std::max(1ll, atoll(getenv("HH_P1_ROWS")));
  } else {
    int64_t wtotal = 0;
    for (const size_t b : idx) {
      int64_t j0, n;
      cluster_range(H, H->level[b], H->src[b], j0, n);
      wtotal += n * H->rank[b] * tag_bytes(H->tag[b]);
    }
    const int64_t share_rows = wtotal / 444 / (W_CT * 4);  // rows of a full fp32 tile in one CTA's share
    while (split_rows > 512 && split_rows > share_rows) split_rows >>= 1;
  }
  size_t i = 0;
  while (i < idx.size()) {
    size_t e = i;
    while (e < idx.size() && H->tag[idx[e]] == H->tag[idx[i]] && H->w_off[idx[e]] == H->w_off[idx[i]]) ++e;
    const size_t b0 = idx[i];
    const int g = H->tag[b0];
    int64_t j0, n;
    cluster_range(H, H->level[b0], H->src[b0], j0, n);
    const int64_t P = H->wpanel[b0];
    // panel column -> z index
    std::vector<int32_t> pz;
    pz.reserve(P);
    for (size_t k = i; k < e; ++k)
      for (int c = 0; c < H->rank[idx[k]]; ++c) pz.push_back((int32_t)(H->zoff[idx[k]] + c));
    int64_t off = H->w_off[b0];
    for (int64_t c0 = 0; c0 < P; c0 += W_CT) {
      const int64_t ct = std::min<int64_t>(W_CT, P - c0);
      const int64_t zb = (int64_t)zmap.size();
      if (n <= split_rows) {
        tiles.push_back(P1Tile{off, j0, zb, -1, (int32_t)n, 0, (int16_t)ct, (int16_t)g, 0});
        tbytes.push_back(n * ct * tag_bytes(g));
      } else {
        const int32_t np = (int32_t)((n + split_rows - 1) / split_rows);
        comb.push_back(P1Combine{zb, npartial, (int32_t)ct, np});
        for (int32_t q = 0; q < np; ++q) {
          const int64_t r0 = (int64_t)q * split_rows, rn = std::min<int64_t>(split_rows, n - r0);
          tiles.push_back(P1Tile{off, j0, zb, npartial + q * ct, (int32_t)rn, (int32_t)r0, (int16_t)ct, (int16_t)g, 0});
          tbytes.push_back(rn * ct * tag_bytes(g));
        }
        npartial += (int64_t)np * ct;
      }
      zmap.insert(zmap.end(), pz.begin() + c0, pz.begin() + c0 + ct);
      off += align_up(n * ct * tag_bytes(g));
    }
    i = e;
  }
  {
    std::vector<size_t> ord(tiles.size());
    for (size_t k = 0; k < ord.size(); ++k) ord[k] = k;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t c) { return tbytes[a] > tbytes[c]; });
    std::vector<P1Tile> t2(tiles.size());
    for (size_t k = 0; k < ord.size(); ++k) t2[k] = tiles[ord[k]];
    tiles.swap(t2);
  }
  // ---- phase 2: group (level, tgt, tag) -> (zbeg, P)
  std::vector<std::vector<int64_t>> gz(L + 1), gp(L + 1);
  for (int l = 0; l <= L; ++l) {
    gz[l].assign((size_t)NTAG << (d * l), -1);
    gp[l].assign((size_t)NTAG << (d * l), 0);
  }
  for (size_t b = 0; b < nb; ++b)
    if (H->storage[b] == STORE_LR && H->rank[b] > 0) {
      const size_t key = (size_t)H->tgt[b] * NTAG + H->tag[b];
      if (gz[H->level[b]][key] < 0) gz[H->level[b]][key] = H->zoff[b];
      gp[H->level[b]][key] += H->rank[b];
    }
  std::vector<std::vector<size_t>> dense(H->ncell);
  for (size_t b = 0; b < nb; ++b)
    if (H->storage[b] == STORE_DENSE) dense[H->tgt[b]].push_back(b);
  std::vector<int64_t> lbytes;
  for (int64_t R = 0; R < H->ncell; ++R) {
    const int64_t r0 = H->leaf_start[R], nr = H->leaf_start[R + 1] - r0;
    if (nr == 0) continue;
    P2Leaf lf{r0, (int32_t)nr, 0, (int64_t)segs.size(), 0};
    int64_t bytes = 0;
    for (const size_t b : dense[R]) {
      int64_t j0, n;
      cluster_range(H, H->level[b], H->src[b], j0, n);
      segs.push_back(P2Seg{H->d_off[b], j0, (int32_t)n, (int16_t)TAG_FP64, 1});
      bytes += nr * n * 8;
    }
    for (int g = 0; g < NTAG; ++g) {
      const int w = tag_bytes(g);
      int64_t col = 0;
      const int64_t base = H->u_leaf_off[(size_t)g * (H->ncell + 1) + R];
      for (int l = 0; l <= L; ++l) {
        const size_t key = (size_t)(R >> (d * (L - l))) * NTAG + g;
        const int64_t P = gp[l][key];
        if (P == 0) continue;
        segs.push_back(P2Seg{base + col * nr * w, N + gz[l][key], (int32_t)P, (int16_t)g, 0});
        bytes += nr * P * w;
        col += P;
      }
    }
    lf.s1 = (int64_t)segs.size();
    leaves.push_back(lf);
    lbytes.push_back(bytes);
  }
  // Morton order (the construction order) is kept for the multi-RHS products: there z is NR
  // times larger (5.8 GB at 3D N=2^20 and 16 RHS) and leaves processed at the same time must
  // share their ancestors' z slices in L2 (ncu r02: in LPT order phase 2 at 16 RHS read 1.8x
  // its U bytes from DRAM on the proxy).  At one RHS z (45 MB) stays in L2 in any order and
  // leaves with the most bytes first (LPT) were measured ~4% faster (profiles/r01_variants.txt).
  leaves_morton = leaves;
#ifndef HH_P2_MORTON
  {
    std::vector<size_t> ord(leaves.size());
    for (size_t k = 0; k < ord.size(); ++k) ord[k] = k;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t c) { return lbytes[a] > lbytes[c]; });
    std::vector<P2Leaf> l2(leaves.size());
    for (size_t k = 0; k < ord.size(); ++k) l2[k] = leaves[ord[k]];
    leaves.swap(l2);
  }
#else
  (void)lbytes;
#endif
}

// ----------------------------------------------------------------- single-RHS stage plan
// The windows are exactly those the on-the-fly producer of matvec.cu would form for NR = 1
// (rows per stage = min(vector entries, factor bytes / row bytes), at least 1), so the
// consumers see the same descriptors either way.
namespace {
void add_stage(std::vector<StageCopy> &copy, std::vector<StageMeta> &meta, uint64_t wsrc, int64_t wlen, uint64_t xsrc,
               int64_t xlen, StageMeta m) {
  auto win = [](uint64_t s, int64_t len, uint64_t &a, uint32_t &bytes) {
    a = s & ~(uint64_t)15;
    bytes = len > 0 ? (uint32_t)(((s + (uint64_t)len + 15) & ~(uint64_t)15) - a) : 0u;
  };
  StageCopy c{};
  win(wsrc, wlen, c.wsrc, c.wbytes);
  win(xsrc, xlen, c.xsrc, c.xbytes);
  m.kind = 0;
  m.wlead = (int32_t)(wsrc & 15);
  m.xlead = (int32_t)(xsrc & 15);
  copy.push_back(c);
  meta.push_back(m);
}
}  // namespace

void build_stage_plan(hh_matrix *H, const std::vector<P1Tile> &tiles, const std::vector<P2Seg> &segs,
                      const std::vector<P2Leaf> &leaves, std::vector<StageItem> (&item)[2],
                      std::vector<StageCopy> (&copy)[2], std::vector<StageMeta> (&meta)[2]) {
  const uint64_t vaddr = (uint64_t)(uintptr_t)H->v.p;
  // Stage geometry per phase: kStageGeo[0] everywhere.  The deeper ring of smaller stages
  // (kStageGeo[1]) was measured slower on every workload, small-leaf plans included
  // (profiles/r02h_ab_quart_geom.txt, r02k_ab_planned.txt): those are bound by per-stage
  // instruction overhead in the consumers, which more and smaller stages only multiply.
  // HH_MV_GEOM1 / HH_MV_GEOM2 = 1 select it per phase for A/B runs.
  H->geom[0] = getenv("HH_MV_GEOM1") ? atoi(getenv("HH_MV_GEOM1")) != 0 : 0;
  H->geom[1] = getenv("HH_MV_GEOM2") ? atoi(getenv("HH_MV_GEOM2")) != 0 : 0;
  for (int ph = 0; ph < 2; ++ph) {
    item[ph].clear();
    copy[ph].clear();
    meta[ph].clear();
  }
  auto close_item = [&](int ph, int64_t s0) {
    StageItem it{};
    it.s0 = s0;
    it.s1 = (int64_t)copy[ph].size();
    if (it.s1 > it.s0) it.first = copy[ph][s0];
    item[ph].push_back(it);
  };
  // ---- phase 1: tile windows of rs rows
  {
    const StageGeo g = kStageGeo[H->geom[0]];
    item[0].reserve(tiles.size());
    for (const P1Tile &T : tiles) {
      const int64_t first = (int64_t)copy[0].size();
      const int w = tag_bytes(T.tag);
      const int64_t rowb = (int64_t)T.ct * w;
      const int64_t rs = std::max<int64_t>(1, std::min<int64_t>(g.xelems, g.wdata / rowb));
      const uint64_t wbase = (uint64_t)(uintptr_t)H->W[T.tag].p + (uint64_t)T.src + (uint64_t)T.r0 * rowb;
      const uint64_t xbase = vaddr + (uint64_t)(T.x0 + T.r0) * 8;
      for (int64_t r0 = 0; r0 < T.n; r0 += rs) {
        const int64_t r1 = std::min<int64_t>(T.n, r0 + rs);
        StageMeta m{};
        m.r0 = (int32_t)r0;
        m.r1 = (int32_t)r1;
        m.a = T.ct;
        m.b = T.tag;
        m.p = T.zbase;
        m.q = T.n;
        m.pb = T.pbase;
        add_stage(copy[0], meta[0], wbase + (uint64_t)r0 * rowb, (r1 - r0) * rowb, xbase + (uint64_t)r0 * 8,
                  (r1 - r0) * 8, m);
      }
      close_item(0, first);
    }
  }
  // ---- phase 2: segment windows of cs columns, leaves in the order of `leaves`
  {
    const StageGeo g = kStageGeo[H->geom[1]];
    item[1].reserve(leaves.size());
    for (const P2Leaf &lf : leaves) {
      const int64_t first = (int64_t)copy[1].size();
      for (int64_t si = lf.s0; si < lf.s1; ++si) {
        const P2Seg &S = segs[si];
        const int w = tag_bytes(S.tag);
        const int64_t colb = (int64_t)lf.nr * w;
        const int64_t cs = std::max<int64_t>(1, std::min<int64_t>(g.xelems, g.wdata / colb));
        const uint64_t ubase = (uint64_t)(uintptr_t)(S.dense ? H->D.p : H->U[S.tag].p) + (uint64_t)S.src;
        const uint64_t zbase = vaddr + (uint64_t)S.vbeg * 8;
        for (int64_t c0 = 0; c0 < S.ncols; c0 += cs) {
          const int64_t c1 = std::min<int64_t>(S.ncols, c0 + cs);
          StageMeta m{};
          m.r0 = (int32_t)c0;
          m.r1 = (int32_t)c1;
          m.flags = (si + 1 == lf.s1 && c1 == S.ncols) ? 1 : 0;
          m.a = lf.nr;
          m.b = S.tag | (S.dense << 8);
          m.p = lf.r0;
          add_stage(copy[1], meta[1], ubase + (uint64_t)c0 * colb, (c1 - c0) * colb, zbase + (uint64_t)c0 * 8,
                    (c1 - c0) * 8, m);
        }
      }
      close_item(1, first);
    }
  }
}

}  // namespace hh
