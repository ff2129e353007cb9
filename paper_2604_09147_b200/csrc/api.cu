// api.cpp — the C-ABI (include/hh.h): argument validation, build orchestration, export.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "build.h"

namespace hh {
static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches += n; }

namespace {
thread_local std::string g_err;

hh_status fail(hh_status s, const std::string &m) {
  g_err = m;
  return s;
}


__global__ void k_round(const double *in, int64_t n, int tag, uint32_t *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = tag == TAG_FP32   ? to_fp32_bits(in[i])
           : tag == TAG_FP16 ? to_fp16_bits(in[i])
           : tag == TAG_BF16 ? to_bf16_bits(in[i])
           : tag == TAG_BF24 ? to_bf24_bits(in[i])
                             : to_q43_bits(in[i]);
}

__global__ void k_leaf_of(const int64_t *leaf_start, int64_t ncell, int32_t *leaf_of) {
  for (int64_t R = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; R < ncell; R += (int64_t)gridDim.x * blockDim.x)
    for (int64_t t = leaf_start[R]; t < leaf_start[R + 1]; ++t) leaf_of[t] = (int32_t)R;
}

size_t workspace_budget() {
  size_t fr = 0, tot = 0;
  HH_CUDA(cudaMemGetInfo(&fr, &tot));
  size_t b = fr / 3;
  return std::max<size_t>(std::min<size_t>(b, (size_t)24 << 30), (size_t)256 << 20);
}

// Runs jobs through the batched path (compress.cu) or, one by one, the whole-GPU path for
// large wide-sketch blocks (compress_big.cu); results in job order.
void compress_jobs(hh_matrix *H, const double *pts, const std::vector<CompressJob> &jobs, bool write, const Arenas *ar,
                   std::vector<CompressResult> &res, cudaStream_t st, BigCtx &big) {
  res.assign(jobs.size(), CompressResult{});
  std::vector<CompressJob> small;
  std::vector<size_t> small_idx;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const int64_t b = jobs[i].block;
    int64_t i0, m, j0, n;
    cluster_range(H, H->level[b], H->tgt[b], i0, m);
    cluster_range(H, H->level[b], H->src[b], j0, n);
    if (use_big_path(m, n, jobs[i].k)) {
      run_compress_big(H, pts, jobs[i], write, ar, res[i], st, big);
    } else {
      small.push_back(jobs[i]);
      small_idx.push_back(i);
    }
  }
  if (!small.empty()) {
    std::vector<CompressResult> rs;
    run_compress(H, pts, small, write, ar, rs, st, workspace_budget());
    for (size_t i = 0; i < small.size(); ++i) res[small_idx[i]] = rs[i];
  }
}

void compress_all(hh_matrix *H, const double *pts, const std::vector<int64_t> &lr, cudaStream_t st, BigCtx &big) {
  // pass 1 with adaptive sketch width: k0 per (level, kind) class from the ranks seen so far
  const size_t nb = H->level.size();
  H->rank.assign(nb, 0);
  H->kfinal.assign(nb, 0);
  H->nb2.assign(nb, 0.0);
  H->maxabs.assign(nb, 0.0);
  std::vector<int> kest(64 * 8, 32);
  std::vector<CompressJob> jobs;
  size_t pos = 0;
  const size_t batch = 16384;
  int64_t retries = 0, inexact = 0;
  std::vector<CompressJob> retry;
  std::vector<CompressResult> res;
  std::vector<std::vector<int>> cls_p(64 * 8);
  while (pos < lr.size() || !retry.empty()) {
    jobs.clear();
    if (!retry.empty()) {
      jobs.swap(retry);
    } else {
      const size_t end = std::min(lr.size(), pos + batch);
      for (size_t i = pos; i < end; ++i) {
        const int64_t b = lr[i];
        jobs.push_back(CompressJob{b, kest[H->level[b] * 8 + H->kind[b]]});
      }
      pos = end;
    }
    compress_jobs(H, pts, jobs, false, nullptr, res, st, big);
    for (size_t i = 0; i < jobs.size(); ++i) {
      const int64_t b = jobs[i].block;
      const CompressResult &r = res[i];
      int64_t i0, m, j0, n;
      cluster_range(H, H->level[b], H->tgt[b], i0, m);
      cluster_range(H, H->level[b], H->src[b], j0, n);
      const int kfull = (int)std::min<int64_t>(std::min(m, n), KMAX);
      if (!r.ok && r.k < kfull) {
        // widen the sketch: x2 while small or on the whole-GPU path, then x1.5
        const int kn = (r.k < 64 || use_big_path(m, n, r.k)) ? 2 * r.k : ((r.k + r.k / 2 + 7) / 8) * 8;
        retry.push_back(CompressJob{b, std::min(kfull, kn)});
        ++retries;
        continue;
      }
      HH_REQUIRE(r.p >= 0, HH_EUNSUPPORTED, "block rank exceeds the sketch limit (4096)");
      inexact += !r.ok;  // at the sketch limit: valid (residual <= eps) but not proved minimal
      HH_REQUIRE(std::isfinite(r.tot) && std::isfinite(r.nb2), HH_ENUMERIC, "non-finite kernel entry");
      H->rank[b] = r.p;
      H->kfinal[b] = r.k;
      H->nb2[b] = r.nb2;
      H->tot[b] = r.tot;
      H->maxabs[b] = r.maxabs;
      cls_p[H->level[b] * 8 + H->kind[b]].push_back(r.p);
    }
    // next sketch width per (level, kind): 90th percentile of the ranks just accepted + 12
    for (size_t c = 0; c < cls_p.size(); ++c) {
      std::vector<int> &v = cls_p[c];
      if (v.empty()) continue;
      std::nth_element(v.begin(), v.begin() + (v.size() * 9) / 10, v.end());
      kest[c] = std::min(KMAX, std::max(16, ((v[(v.size() * 9) / 10] + 12 + 7) / 8) * 8));
      v.clear();
    }
  }
  H->info.n_retry = retries;
  H->info.n_inexact = inexact;
}

}  // namespace
}  // namespace hh

using namespace hh;

extern "C" {

const char *hh_last_error(void) { return g_err.c_str(); }
int64_t hh_kernel_launches(void) { return g_launches.load(); }

hh_status hh_build(const double *points, int64_t N, int32_t d, hh_kernel kernel, double eps, double eta,
                   int32_t leaf_size, int32_t switch_level, uint32_t precision_set, void *cuda_stream,
                   hh_handle *out) {
  g_err.clear();
  if (!points || !out) return fail(HH_EINVAL, "NULL pointer");
  if (N < 1 || N > (int64_t)INT32_MAX) return fail(HH_EINVAL, "N must be in [1, 2^31)");
  if (d < 1) return fail(HH_EINVAL, "d must be >= 1");
  if (d > 3) return fail(HH_EUNSUPPORTED, "this build supports d <= 3");
  if (!(eps > 0x1p-53 && eps < 1.0)) return fail(HH_EINVAL, "eps must be in (2^-53, 1)");
  if (!(eta > 0.0) || !std::isfinite(eta)) return fail(HH_EINVAL, "eta must be > 0");
  if (leaf_size < 1) return fail(HH_EINVAL, "leaf_size must be >= 1");
  if (leaf_size > 256) return fail(HH_EUNSUPPORTED, "leaf_size > 256 not supported by this build");
  if (!(precision_set & HH_P_FP64)) return fail(HH_EINVAL, "precision_set must contain HH_P_FP64");
  if (precision_set & ~(HH_P_ALL | HH_LEDGER_ONLY | HH_TIE_FP16)) return fail(HH_EINVAL, "unknown precision_set bits");
  if (kernel.kind < 0 || kernel.kind > 4) return fail(HH_EINVAL, "unknown kernel kind");
  if ((kernel.kind == HH_K_GAUSS || kernel.kind == HH_K_EXP) && !(kernel.scale > 0.0))
    return fail(HH_EINVAL, "kernel scale must be > 0");
  if (switch_level < HH_SWITCH_NONE) return fail(HH_EINVAL, "switch_level must be >= 0 or HH_SWITCH_NONE");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(HH_ECUDA, "no CUDA device");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  hh_matrix *H = nullptr;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    H = new hh_matrix();
    H->N = N;
    H->d = d;
    H->kernel = kernel;
    H->eps = eps;
    H->eta = eta;
    H->leaf_size = leaf_size;
    H->s = switch_level;
    H->pset = precision_set & HH_P_ALL;
    H->ledger = (precision_set & HH_LEDGER_ONLY) != 0;
    H->tie16 = (precision_set & HH_TIE_FP16) && (precision_set & HH_P_FP16) && (precision_set & HH_P_BF16);
    DBuf pts;
    build_tree(H, points, st, pts);                                   // a1
    HH_REQUIRE(switch_level == HH_SWITCH_NONE || switch_level <= H->L, HH_EINVAL, "switch_level > L");
    build_partition(H);                                               // a2
    const size_t nb = H->level.size();
    const bool mixed = H->pset != HH_P_FP64;
    H->storage.assign(nb, STORE_LR);
    H->tag.assign(nb, TAG_FP64);
    H->tot.assign(nb, 0.0);
    std::vector<int64_t> lr, dn;
    for (size_t b = 0; b < nb; ++b) {
      const int k = H->kind[b];
      if (k == KIND_DIAG || (k == KIND_LNBR && !mixed)) {
        H->storage[b] = STORE_DENSE;
        dn.push_back((int64_t)b);
      } else {
        lr.push_back((int64_t)b);
      }
    }
    BigCtx big;
    compress_all(H, pts.as<double>(), lr, st, big);                    // a3 (pass 1)
    run_dense(H, pts.as<double>(), dn, false, st);                    // dense norms
    for (size_t b = 0; b < nb; ++b)
      HH_REQUIRE(std::isfinite(H->tot[b]), HH_ENUMERIC, "non-finite kernel entry");
    assign_tags(H);                                                   // a4 + a5
    compute_layout(H);                                                // a6 (offsets)
    if (!H->ledger) {
      for (int g = 0; g < NTAG; ++g) {
        H->W[g].alloc(H->w_bytes[g]);
        H->U[g].alloc(H->u_bytes[g]);
        HH_CUDA(cudaMemsetAsync(H->U[g].p, 0, H->U[g].bytes, st));
        HH_CUDA(cudaMemsetAsync(H->W[g].p, 0, H->W[g].bytes, st));
      }
      H->D.alloc(H->d_bytes);
      HH_CUDA(cudaMemsetAsync(H->D.p, 0, H->D.bytes, st));
      // pass 2: recompute (bitwise identical) and store rounded factors
      DBuf d_uoff, d_ls, d_leaf_of;
      h2d(d_uoff, H->u_leaf_off, st);
      h2d(d_ls, H->leaf_start, st);
      d_leaf_of.alloc(sizeof(int32_t) * N);
      k_leaf_of<<<1184, 256, 0, st>>>(d_ls.as<int64_t>(), H->ncell, d_leaf_of.as<int32_t>());
      HH_LAUNCHED();
      Arenas ar{};
      for (int g = 0; g < NTAG; ++g) {
        ar.W[g] = H->W[g].as<uint8_t>();
        ar.U[g] = H->U[g].as<uint8_t>();
      }
      ar.u_leaf_off = d_uoff.as<int64_t>();
      ar.leaf_start = d_ls.as<int64_t>();
      ar.leaf_of = d_leaf_of.as<int32_t>();
      ar.ncell = H->ncell;
      std::vector<CompressJob> jobs;
      for (size_t b = 0; b < nb; ++b)
        if (H->storage[b] == STORE_LR && H->rank[b] > 0) jobs.push_back(CompressJob{(int64_t)b, H->kfinal[b]});
      std::vector<CompressResult> res;
      compress_jobs(H, pts.as<double>(), jobs, true, &ar, res, st, big);
      // pass 2 writes the factors of the pass-1 rank; its maxabs must reproduce pass 1's
      // (the range guard decided the tags from it): a cheap determinism check
      int64_t mism = 0;
      for (size_t i = 0; i < jobs.size(); ++i) mism += res[i].maxabs != H->maxabs[jobs[i].block];
      HH_REQUIRE(mism == 0, HH_ECUDA, "pass-2 recompression disagreed with pass 1 (non-deterministic kernel)");
      // dense blocks (diagonal + dense neighbours) after tagging
      std::vector<int64_t> dn2;
      for (size_t b = 0; b < nb; ++b)
        if (H->storage[b] == STORE_DENSE) dn2.push_back((int64_t)b);
      run_dense(H, pts.as<double>(), dn2, true, st);
      // matvec plan + workspace
      std::vector<P1Tile> tiles;
      std::vector<int32_t> zmap;
      std::vector<P1Combine> comb;
      std::vector<P2Seg> segs;
      std::vector<P2Leaf> leaves, leaves_mo;
      int64_t npartial = 0;
      build_plan(H, tiles, zmap, comb, npartial, segs, leaves, leaves_mo);
      h2d(H->p1_tiles, tiles, st);
      h2d(H->zmap, zmap, st);
      h2d(H->p1_comb, comb, st);
      H->n_p1_comb = (int64_t)comb.size();
      H->n_partial = npartial;
      H->partial.alloc(sizeof(double) * 16 * (size_t)std::max<int64_t>(1, npartial));
      h2d(H->p2_segs, segs, st);
      h2d(H->p2_leaves, leaves, st);
      h2d(H->p2_leaves_mo, leaves_mo, st);
      H->n_p1_tiles = (int64_t)tiles.size();
      H->n_p2_leaves = (int64_t)leaves.size();
      H->v.alloc(sizeof(double) * 16 * (size_t)(N + H->ztotal) + 64);
      {  // stage plan of the single-RHS product (absolute addresses: arenas and v exist now)
        std::vector<StageItem> sitem[2];
        std::vector<StageCopy> scopy[2];
        std::vector<StageMeta> smeta[2];
        build_stage_plan(H, tiles, segs, leaves, sitem, scopy, smeta);
        for (int ph = 0; ph < 2; ++ph) {
          h2d(H->st_item[ph], sitem[ph], st);
          h2d(H->st_copy[ph], scopy[ph], st);
          h2d(H->st_meta[ph], smeta[ph], st);
        }
        HH_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
      }
      H->ctr.alloc(64);
      HH_CUDA(cudaMemsetAsync(H->ctr.p, 0, 64, st));
      HH_CUDA(cudaStreamSynchronize(st));
    }
    // info
    hh_info_t &I = H->info;
    I.d = d;
    I.L = H->L;
    I.switch_level = switch_level;
    I.kernel_kind = kernel.kind;
    I.N = N;
    I.eta = eta;
    I.eps = eps;
    I.kernel_scale = kernel.scale;
    I.precision_set = H->pset;
    I.ledger_only = H->ledger;
    I.n_cells = H->ncell;
    I.nblocks = (int64_t)nb;
    I.total_rank = H->ztotal;
    I.norm2 = H->norm2;
    for (int g = 0; g < NTAG; ++g) {
      I.w_bytes[g] = H->w_bytes[g];
      I.u_bytes[g] = H->u_bytes[g];
    }
    I.d_bytes = H->d_bytes;
    I.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (getenv("HH_PROFILE_BUILD")) {
      print_build_profile();
      fprintf(stderr, "[hh build profile] total %.2fs retries=%lld\n", I.build_seconds, (long long)I.n_retry);
    }
    *out = H;
    return HH_OK;
  } catch (const Error &e) {
    delete H;
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    delete H;
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    delete H;
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    delete H;
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_matvec(hh_handle H, const double *x, double *y, int32_t nrhs, void *cuda_stream) {
  g_err.clear();
  if (!H || !x || !y) return fail(HH_EINVAL, "NULL pointer");
  if (nrhs < 1) return fail(HH_EINVAL, "nrhs must be >= 1");
  if (H->ledger) return fail(HH_EINVAL, "ledger-only handle has no factors");
  const char *xb = (const char *)x, *yb = (const char *)y;
  const size_t bytes = sizeof(double) * (size_t)H->N * nrhs;
  if (!(xb + bytes <= yb || yb + bytes <= xb)) return fail(HH_EINVAL, "x and y overlap");
  try {
    run_matvec(H, x, y, nrhs, (cudaStream_t)cuda_stream);
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_matvec_wp(hh_handle H, const double *x, double *y, int32_t nrhs, int32_t working_precision,
                       void *cuda_stream) {
  g_err.clear();
  if (working_precision < HH_WP_FP64 || working_precision > HH_WP_FP16)
    return fail(HH_EINVAL, "working_precision must be HH_WP_FP64, HH_WP_FP32 or HH_WP_FP16");
  if (!H || !x || !y) return fail(HH_EINVAL, "NULL pointer");
  if (nrhs < 1) return fail(HH_EINVAL, "nrhs must be >= 1");
  if (H->ledger) return fail(HH_EINVAL, "ledger-only handle has no factors");
  const char *xb = (const char *)x, *yb = (const char *)y;
  const size_t bytes = sizeof(double) * (size_t)H->N * nrhs;
  if (!(xb + bytes <= yb || yb + bytes <= xb)) return fail(HH_EINVAL, "x and y overlap");
  try {
    run_matvec(H, x, y, nrhs, (cudaStream_t)cuda_stream, working_precision);
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_matvec_host(hh_handle H, const double *x_host, double *y_host, int32_t nrhs, void *cuda_stream) {
  g_err.clear();
  if (!H || !x_host || !y_host) return fail(HH_EINVAL, "NULL pointer");
  if (nrhs < 1) return fail(HH_EINVAL, "nrhs must be >= 1");
  if (H->ledger) return fail(HH_EINVAL, "ledger-only handle has no factors");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  try {
    const size_t bytes = sizeof(double) * (size_t)H->N * nrhs;
    if (H->hx.bytes < bytes) {  // handle-owned staging, grown on demand
      H->hx.alloc(bytes);
      H->hy.alloc(bytes);
    }
    HH_CUDA(cudaMemcpyAsync(H->hx.p, x_host, bytes, cudaMemcpyHostToDevice, st));
    run_matvec(H, H->hx.as<double>(), H->hy.as<double>(), nrhs, st);
    HH_CUDA(cudaMemcpyAsync(y_host, H->hy.p, bytes, cudaMemcpyDeviceToHost, st));
    HH_CUDA(cudaStreamSynchronize(st));
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_matvec_profile(hh_handle H, int32_t enable) {
  if (!H) return fail(HH_EINVAL, "NULL handle");
  H->prof = enable != 0;
  return HH_OK;
}

hh_status hh_matvec_timing(hh_handle H, double *ms, int64_t *count) {
  g_err.clear();
  if (!H || !ms) return fail(HH_EINVAL, "NULL pointer");
  try {
    for (int i = 0; i < 4; ++i) ms[i] = 0.0;
    const size_t n = H->prof_ev.size() / 4;
    if (n) HH_CUDA(cudaEventSynchronize(H->prof_ev.back()));
    for (size_t c = 0; c < n; ++c) {
      float t[3];
      for (int i = 0; i < 3; ++i) HH_CUDA(cudaEventElapsedTime(&t[i], H->prof_ev[4 * c + i], H->prof_ev[4 * c + i + 1]));
      for (int i = 0; i < 3; ++i) {
        ms[i] += t[i];
        ms[3] += t[i];
      }
    }
    for (auto e : H->prof_ev) cudaEventDestroy(e);
    H->prof_ev.clear();
    if (count) *count = (int64_t)n;
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_info(hh_handle H, hh_info_t *info) {
  if (!H || !info) return fail(HH_EINVAL, "NULL pointer");
  *info = H->info;
  return HH_OK;
}

hh_status hh_export(hh_handle H, hh_export_t *out) {
  g_err.clear();
  if (!H || !out) return fail(HH_EINVAL, "NULL pointer");
  try {
    out->info = H->info;
    if (out->perm) HH_CUDA(cudaMemcpy(out->perm, H->d_perm.p, sizeof(int32_t) * H->N, cudaMemcpyDeviceToHost));
    if (out->leaf_start) memcpy(out->leaf_start, H->leaf_start.data(), sizeof(int64_t) * H->leaf_start.size());
    if (out->u_leaf_off && !H->u_leaf_off.empty())
      memcpy(out->u_leaf_off, H->u_leaf_off.data(), sizeof(int64_t) * H->u_leaf_off.size());
    if (out->d_leaf_off && !H->d_leaf_off.empty())
      memcpy(out->d_leaf_off, H->d_leaf_off.data(), sizeof(int64_t) * H->d_leaf_off.size());
    if (out->blocks) {
      const size_t nb = H->level.size();
      for (size_t b = 0; b < nb; ++b) {
        hh_block_t &r = out->blocks[b];
        r.tgt = H->tgt[b];
        r.src = H->src[b];
        r.zoff = H->zoff.empty() ? -1 : H->zoff[b];
        r.w_off = H->w_off.empty() ? -1 : H->w_off[b];
        r.wcol = H->wcol.empty() ? -1 : H->wcol[b];
        r.ucol = H->ucol.empty() ? -1 : H->ucol[b];
        r.d_off = H->d_off.empty() ? -1 : H->d_off[b];
        r.nb2 = H->nb2.empty() ? 0 : H->nb2[b];
        r.tot = H->tot[b];
        r.maxabs = H->maxabs.empty() ? 0 : H->maxabs[b];
        r.rank = H->rank[b];
        r.level = H->level[b];
        r.kind = H->kind[b];
        r.tag = H->tag[b];
        r.storage = H->storage[b];
      }
    }
    if (out->arena_dst && out->arena_len > 0) {
      if (H->ledger) return fail(HH_EINVAL, "ledger-only handle has no arenas");
      const DBuf *src = nullptr;
      if (out->arena >= 0 && out->arena < NTAG) src = &H->W[out->arena];
      else if (out->arena >= NTAG && out->arena < 2 * NTAG) src = &H->U[out->arena - NTAG];
      else if (out->arena == 2 * NTAG) src = &H->D;
      if (!src) return fail(HH_EINVAL, "arena must be 0 .. 2 * HH_NTAG");
      const int64_t size = out->arena < NTAG       ? H->w_bytes[out->arena]
                           : out->arena < 2 * NTAG ? H->u_bytes[out->arena - NTAG]
                                                   : H->d_bytes;
      if (out->arena_off < 0 || out->arena_off + out->arena_len > size) return fail(HH_EINVAL, "arena window out of range");
      HH_CUDA(cudaMemcpy(out->arena_dst, (const char *)src->p + out->arena_off, out->arena_len, cudaMemcpyDeviceToHost));
    }
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

hh_status hh_switch_level_search(const double *points, int64_t N, int32_t d, hh_kernel kernel, double eps,
                                 double eta, int32_t leaf_size, uint32_t precision_set, void *cuda_stream,
                                 int32_t *out_level, int32_t *out_L, int64_t *bytes, int32_t bytes_len) {
  g_err.clear();
  if (!out_level) return fail(HH_EINVAL, "NULL pointer");
  const uint32_t pset = (precision_set & (HH_P_ALL | HH_TIE_FP16)) | HH_LEDGER_ONLY;
  auto ledger_bytes = [&](int32_t s, int64_t &out, int32_t *L) -> hh_status {
    hh_handle h = nullptr;
    const hh_status st = hh_build(points, N, d, kernel, eps, eta, leaf_size, s, pset, cuda_stream, &h);
    if (st != HH_OK) return st;
    out = h->info.stored_bytes;
    if (L) *L = h->L;
    hh_free(h);
    return HH_OK;
  };
  int64_t Ss = 0;
  int32_t L = 0;
  hh_status st = ledger_bytes(HH_SWITCH_NONE, Ss, &L);  // S_s: pure H_s (the paper's ell = L)
  if (st != HH_OK) return st;
  if (out_L) *out_L = L;
  if (bytes && bytes_len < L + 2) return fail(HH_EINVAL, "bytes_len must be >= L + 2");
  if (bytes) {
    for (int i = 0; i < L + 2; ++i) bytes[i] = -1;
    bytes[L] = Ss;
    bytes[L + 1] = Ss;
  }
  int32_t ell = L;
  int64_t gain = 0;  // S_1(L) - S_2(L) = 0
  while (ell > 0) {
    int64_t Sh = 0;
    st = ledger_bytes(ell - 1, Sh, nullptr);
    if (st != HH_OK) return st;
    if (bytes) bytes[ell - 1] = Sh;
    const int64_t gnew = Ss - Sh;  // S_1(ell-1) - S_2(ell-1): the common terms cancel
    if (gnew <= gain) break;
    gain = gnew;
    --ell;
  }
  *out_level = ell;
  return HH_OK;
}

hh_status hh_free(hh_handle H) {
  delete H;
  return HH_OK;
}

hh_status hh_selftest_partition(const int64_t *leaf_start, int32_t d, int32_t L, double eta, int32_t switch_level,
                                int64_t capacity, int64_t *nblocks, uint8_t *level, uint8_t *kind, int64_t *tgt,
                                int64_t *src) {
  g_err.clear();
  if (!leaf_start || !nblocks || d < 1 || d > 3 || L < 0 || d * L > 26 || !(eta > 0))
    return fail(HH_EINVAL, "bad argument");
  try {
    hh_matrix H;
    H.d = d;
    H.L = L;
    H.s = switch_level;
    H.eta = eta;
    H.ncell = 1ll << (d * L);
    H.leaf_start.assign(leaf_start, leaf_start + H.ncell + 1);
    build_partition(&H);
    const int64_t nb = (int64_t)H.level.size();
    *nblocks = nb;
    if (capacity < nb) return capacity == 0 ? HH_OK : fail(HH_EINVAL, "capacity too small");
    for (int64_t b = 0; b < nb; ++b) {
      if (level) level[b] = H.level[b];
      if (kind) kind[b] = H.kind[b];
      if (tgt) tgt[b] = H.tgt[b];
      if (src) src[b] = H.src[b];
    }
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (...) {
    return fail(HH_EINVAL, "partition failed");
  }
}

hh_status hh_selftest_layout(const int64_t *leaf_start, int32_t d, int32_t L, int64_t nblocks, const uint8_t *level,
                             const int64_t *tgt, const int64_t *src, const int32_t *rank, const uint8_t *tag,
                             const uint8_t *storage, int64_t *zoff, int64_t *w_off, int64_t *wcol, int64_t *ucol,
                             int64_t *d_off, int64_t *u_leaf_off, int64_t *d_leaf_off, int64_t *w_bytes) {
  g_err.clear();
  if (!leaf_start || !level || !tgt || !src || !rank || !tag || !storage || nblocks < 0 || d < 1 || d > 3 || L < 0 ||
      d * L > 26)
    return fail(HH_EINVAL, "bad argument");
  try {
    hh_matrix H;
    H.d = d;
    H.L = L;
    H.ncell = 1ll << (d * L);
    H.leaf_start.assign(leaf_start, leaf_start + H.ncell + 1);
    H.level.assign(level, level + nblocks);
    H.tgt.assign(tgt, tgt + nblocks);
    H.src.assign(src, src + nblocks);
    H.rank.assign(rank, rank + nblocks);
    H.tag.assign(tag, tag + nblocks);
    H.storage.assign(storage, storage + nblocks);
    compute_layout(&H);
    for (int64_t b = 0; b < nblocks; ++b) {
      if (zoff) zoff[b] = H.zoff[b];
      if (w_off) w_off[b] = H.w_off[b];
      if (wcol) wcol[b] = H.wcol[b];
      if (ucol) ucol[b] = H.ucol[b];
      if (d_off) d_off[b] = H.d_off[b];
    }
    if (u_leaf_off) std::copy(H.u_leaf_off.begin(), H.u_leaf_off.end(), u_leaf_off);
    if (d_leaf_off) std::copy(H.d_leaf_off.begin(), H.d_leaf_off.end(), d_leaf_off);
    if (w_bytes)
      for (int g = 0; g < NTAG; ++g) w_bytes[g] = H.w_bytes[g];
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (...) {
    return fail(HH_EINVAL, "layout failed");
  }
}

hh_status hh_selftest_tags(const int64_t *leaf_start, int32_t d, int32_t L, int64_t nblocks, const uint8_t *level,
                          const uint8_t *kind, const int64_t *tgt, const int64_t *src, int32_t *rank,
                          const double *nb2, const double *tot, const double *maxabs, double eps,
                          uint32_t precision_set, uint8_t *tag, uint8_t *storage, double *norm2, int64_t *counts) {
  g_err.clear();
  if (!leaf_start || !level || !kind || !tgt || !src || !rank || !nb2 || !tot || !maxabs || !tag || !storage ||
      !norm2 || !counts || nblocks < 0 || d < 1 || d > 3 || L < 0 || d * L > 26 || !(precision_set & HH_P_FP64))
    return fail(HH_EINVAL, "bad argument");
  try {
    hh_matrix H;
    H.d = d;
    H.L = L;
    H.eps = eps;
    H.ncell = 1ll << (d * L);
    H.leaf_start.assign(leaf_start, leaf_start + H.ncell + 1);
    H.pset = precision_set & HH_P_ALL;
    H.tie16 = (precision_set & HH_TIE_FP16) && (precision_set & HH_P_FP16) && (precision_set & HH_P_BF16);
    H.level.assign(level, level + nblocks);
    H.kind.assign(kind, kind + nblocks);
    H.tgt.assign(tgt, tgt + nblocks);
    H.src.assign(src, src + nblocks);
    H.rank.assign(rank, rank + nblocks);
    H.nb2.assign(nb2, nb2 + nblocks);
    H.tot.assign(tot, tot + nblocks);
    H.maxabs.assign(maxabs, maxabs + nblocks);
    const bool mixed = H.pset != HH_P_FP64;  // as hh_build: dense = diagonal (+ leaf neighbours when uniform)
    H.storage.assign(nblocks, STORE_LR);
    H.tag.assign(nblocks, TAG_FP64);
    for (int64_t b = 0; b < nblocks; ++b)
      if (H.kind[b] == KIND_DIAG || (H.kind[b] == KIND_LNBR && !mixed)) H.storage[b] = STORE_DENSE;
    assign_tags(&H);
    for (int64_t b = 0; b < nblocks; ++b) {
      tag[b] = H.tag[b];
      storage[b] = H.storage[b];
      rank[b] = H.rank[b];
    }
    *norm2 = H.norm2;
    counts[0] = H.info.n_fallback;
    counts[1] = H.info.n_promoted;
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (...) {
    return fail(HH_EINVAL, "tagging failed");
  }
}

/* Test hook: apply the device storage-rounding routine of `tag` (1..3) to host values and
 * return the bit patterns (checked against the oracle's definition-based rounding). */
hh_status hh_selftest_round(const double *host_in, int64_t n, int32_t tag, uint32_t *host_bits) {
  g_err.clear();
  if (!host_in || !host_bits || n < 0 || tag < 1 || tag > 5) return fail(HH_EINVAL, "bad argument");
  try {
    DBuf a, b;
    a.alloc(sizeof(double) * n);
    b.alloc(sizeof(uint32_t) * n);
    HH_CUDA(cudaMemcpy(a.p, host_in, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_round<<<(unsigned)std::max<int64_t>(1, (n + 255) / 256), 256>>>(a.as<double>(), n, tag, b.as<uint32_t>());
    HH_LAUNCHED();
    HH_CUDA(cudaMemcpy(host_bits, b.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    return HH_OK;
  } catch (const Error &e) {
    return fail(e.st, e.what());
  } catch (const std::bad_alloc &) {
    return fail(HH_ENOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(HH_ECUDA, e.what());
  } catch (...) {
    return fail(HH_ECUDA, "unexpected error");
  }
}

}  // extern "C"
