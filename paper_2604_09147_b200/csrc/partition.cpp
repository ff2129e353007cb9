// partition.cpp — §8(a) row a2: block partition under hybrid admissibility (host C++).
//
// Standard admissibility Eq. 2.1 on grid boxes (reading G5): two level-l
// boxes with integer offset a are admissible iff d <= eta^2 * sum_k max(0,|a_k|-1)^2, with
// eta^2 snapped to an integer when within 1e-12 (G6).  Hybrid admissibility Eq. 3.1
// enumerated as PAPER.md:552-557 / Alg. 1, read as G7:
//   level l <  s : admissible pair -> FAR block, else inadmissible (descend)
//   level l == s : non-self pair   -> FAR (admissible) or NBR ("finer neighbour") block
//   level l >  s : non-self pair   -> SIB (weak admissibility)
//   s == NONE    : standard at every level; inadmissible leaf pairs -> DIAG / LNBR (pure H_s)
// Children pairs of inadmissible parents only; a pair with an empty side is skipped (G20).
// Output: blocks in canonical order (level, target Morton code, source Morton code).
#include <algorithm>
#include <cmath>
#include <vector>

#include "build.h"

namespace hh {

namespace {
struct Blk {
  int64_t t, s;
  uint8_t kind;
};

inline void decode(int64_t code, int d, int l, int64_t *c) {
  for (int k = 0; k < d; ++k) c[k] = 0;
  for (int b = 0; b < l; ++b)
    for (int k = 0; k < d; ++k) c[k] |= ((code >> (b * d + k)) & 1) << b;
}
}  // namespace

double snap_eta2(double eta) {
  double e2 = eta * eta;
  double r = std::nearbyint(e2);
  return std::fabs(e2 - r) <= 1e-12 * e2 ? r : e2;
}

void build_partition(hh_matrix *H) {
  const int d = H->d, L = H->L, s = H->s;
  const double eta2 = snap_eta2(H->eta);
  const int nch = 1 << d;
  auto size_at = [&](int l, int64_t m) {
    const int sh = d * (L - l);
    return H->leaf_start[(m + 1) << sh] - H->leaf_start[m << sh];
  };
  std::vector<std::pair<int64_t, int64_t>> parents{{0, 0}}, next;
  auto push = [&](int l, const std::vector<Blk> &v) {
    for (const Blk &b : v) {
      H->level.push_back((uint8_t)l);
      H->kind.push_back(b.kind);
      H->tgt.push_back(b.t);
      H->src.push_back(b.s);
    }
  };
  if (L == 0) {
    push(0, {Blk{0, 0, (uint8_t)KIND_DIAG}});
  }
  int64_t ci_c[3], cj_c[3];
  for (int l = 1; l <= L; ++l) {
    std::vector<Blk> blocks;
    next.clear();
    for (const auto &pp : parents) {
      for (int a = 0; a < nch; ++a) {
        const int64_t ci = pp.first * nch + a;
        if (size_at(l, ci) == 0) continue;
        decode(ci, d, l, ci_c);
        for (int b = 0; b < nch; ++b) {
          const int64_t cj = pp.second * nch + b;
          if (size_at(l, cj) == 0) continue;
          decode(cj, d, l, cj_c);
          int64_t G = 0;
          for (int k = 0; k < d; ++k) {
            int64_t g = std::llabs(cj_c[k] - ci_c[k]) - 1;
            if (g > 0) G += g * g;
          }
          const bool adm = (double)d <= eta2 * (double)G;
          const bool same = ci == cj;
          bool blk;
          uint8_t kind;
          if (s == HH_SWITCH_NONE || l < s) {
            blk = adm;
            kind = KIND_FAR;
          } else if (l == s) {
            blk = !same;
            kind = adm ? KIND_FAR : KIND_NBR;
          } else {
            blk = !same;
            kind = KIND_SIB;
          }
          if (blk) {
            blocks.push_back(Blk{ci, cj, kind});
          } else if (l == L) {
            blocks.push_back(Blk{ci, cj, (uint8_t)(same ? KIND_DIAG : KIND_LNBR)});
          } else {
            next.emplace_back(ci, cj);
          }
        }
      }
    }
    std::sort(blocks.begin(), blocks.end(), [](const Blk &x, const Blk &y) {
      return x.t != y.t ? x.t < y.t : x.s < y.s;
    });
    push(l, blocks);
    parents.swap(next);
  }
  // measured sparsity constants (max blocks of a kind per (level, target))
  const size_t nb = H->level.size();
  int cf = 0, cn = 0, cs = 0;
  size_t b = 0;
  while (b < nb) {
    size_t e = b;
    int f = 0, n = 0, sb = 0;
    while (e < nb && H->level[e] == H->level[b] && H->tgt[e] == H->tgt[b]) {
      f += H->kind[e] == KIND_FAR;
      n += H->kind[e] == KIND_NBR || H->kind[e] == KIND_LNBR;
      sb += H->kind[e] == KIND_SIB;
      ++e;
    }
    cf = std::max(cf, f);
    cn = std::max(cn, n);
    cs = std::max(cs, sb);
    b = e;
  }
  H->info.c_far = cf;
  H->info.c_nbr = cn;
  H->info.c_sib = cs;
}

}  // namespace hh
