// ref_capi.cpp -- extern "C" wrapper over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles the reference's own
// sources in place (/root/reference/proj/src/*.cpp minus commands.cpp, which
// needs the absent CLI11) plus this file into oracle/_ref/libdvsref.so.
// Nothing here re-implements the algorithm; every entry point forwards to the
// reference function named in its comment.  Used to (a) pin the C
// restatement in dvs_oracle.c, (b) generate tests/golden/ fixtures, and
// (c) serve as the "reference" CPU baseline in bench.py.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dvs/dataset.hpp"
#include "dvs/errors.hpp"
#include "dvs/graph_index.hpp"
#include "dvs/index.hpp"
#include "dvs/index_file.hpp"
#include "dvs/kmeans.hpp"
#include "dvs/router.hpp"
#include "dvs/simulator.hpp"
#include "dvs/topk.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const dvs::format_error& e) {
    g_err = e.what();
    return 3;
  } catch (const dvs::internal_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

dvs::Dataset make_ds(const float* data, std::uint64_t n, int dim) {
  dvs::Dataset ds;
  ds.dim = dim;
  ds.data.assign(data, data + n * static_cast<std::uint64_t>(dim));
  return ds;
}

// Order-preserving std::thread parallel-for (SPEC.md:95 allows per-query
// parallelism with order-preserving output).
template <class F>
void parallel_for(std::uint64_t n, int nthreads, F&& body) {
  if (nthreads <= 1 || n < 2) {
    body(0, n);
    return;
  }
  if (static_cast<std::uint64_t>(nthreads) > n) nthreads = static_cast<int>(n);
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nthreads));
  for (int t = 0; t < nthreads; ++t) {
    const std::uint64_t b = n * t / nthreads, e = n * (t + 1) / nthreads;
    th.emplace_back([&, t, b, e] {
      try {
        body(b, e);
      } catch (...) {
        errs[static_cast<std::size_t>(t)] = std::current_exception();
      }
    });
  }
  for (auto& x : th) x.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}
}  // namespace

extern "C" {

const char* dvsref_last_error() { return g_err.c_str(); }

// build_graph, graph_index.cpp:46-97 (gids nullable -> iota)
void* dvsref_build_graph(const float* data, std::uint64_t n, int dim, const std::uint32_t* gids,
                         int out_degree) {
  dvs::GraphIndex* out = nullptr;
  int rc = guarded([&] {
    dvs::Dataset ds = make_ds(data, n, dim);
    if (gids) {
      out = new dvs::GraphIndex(
          dvs::build_graph(ds, std::vector<std::uint32_t>(gids, gids + n), out_degree));
    } else {
      out = new dvs::GraphIndex(dvs::build_graph(ds, out_degree));
    }
  });
  return rc ? nullptr : out;
}

// GraphIndex assembled from caller arrays; entry order from compute_entry_order
// (graph_index.cpp:21-44) exactly as load_index does (index_file.cpp:290).
void* dvsref_graph_from_arrays(const float* data, std::uint64_t n, int dim,
                               const std::uint32_t* gids, int out_degree,
                               const std::uint32_t* adjacency) {
  dvs::GraphIndex* out = nullptr;
  int rc = guarded([&] {
    auto* g = new dvs::GraphIndex();
    g->vectors = make_ds(data, n, dim);
    g->global_ids.assign(gids, gids + n);
    g->out_degree = out_degree;
    g->adjacency.assign(adjacency, adjacency + n * static_cast<std::uint64_t>(out_degree));
    g->entry_order = dvs::compute_entry_order(g->vectors);
    out = g;
  });
  return rc ? nullptr : out;
}

void dvsref_graph_free(void* g) { delete static_cast<dvs::GraphIndex*>(g); }

std::uint64_t dvsref_graph_size(void* g) { return static_cast<dvs::GraphIndex*>(g)->size(); }

void dvsref_graph_arrays(void* gv, std::uint32_t* adjacency, std::uint32_t* entry_order,
                         std::uint32_t* gids) {
  auto* g = static_cast<dvs::GraphIndex*>(gv);
  if (adjacency) std::memcpy(adjacency, g->adjacency.data(), g->adjacency.size() * 4);
  if (entry_order) std::memcpy(entry_order, g->entry_order.data(), g->entry_order.size() * 4);
  if (gids) std::memcpy(gids, g->global_ids.data(), g->global_ids.size() * 4);
}

int dvsref_compute_entry_order(const float* data, std::uint64_t n, int dim, std::uint32_t* out) {
  return guarded([&] {
    auto ids = dvs::compute_entry_order(make_ds(data, n, dim));
    std::memcpy(out, ids.data(), ids.size() * 4);
  });
}

// beam_search_stats, graph_index.cpp:105-187, over a query batch
int dvsref_beam_search(void* gv, const float* queries, std::uint64_t nq, int iterations,
                       int beam_width, int k, int entry_count, int nthreads,
                       std::uint32_t* out_ids, float* out_dists, std::uint32_t* out_count,
                       std::uint64_t* out_visited) {
  return guarded([&] {
    const auto* g = static_cast<dvs::GraphIndex*>(gv);
    dvs::SearchParams p;
    p.iterations = iterations;
    p.beam_width = beam_width;
    p.k = k;
    p.entry_count = entry_count;
    const std::uint64_t dim = static_cast<std::uint64_t>(g->vectors.dim);
    parallel_for(nq, nthreads, [&](std::uint64_t b, std::uint64_t e) {
      for (std::uint64_t q = b; q < e; ++q) {
        const dvs::SearchResult r =
            dvs::beam_search_stats(*g, std::span<const float>(queries + q * dim, dim), p);
        for (std::size_t i = 0; i < r.hits.size(); ++i) {
          out_ids[q * k + i] = r.hits[i].id;
          out_dists[q * k + i] = r.hits[i].dist;
        }
        out_count[q] = static_cast<std::uint32_t>(r.hits.size());
        out_visited[q] = r.visited;
      }
    });
  });
}

// combine_results, simulator.cpp:219-243
int dvsref_combine_results(int nparts, const std::uint32_t* ids, const float* dists,
                           const std::uint32_t* counts, int stride, int k,
                           std::uint32_t* out_ids, float* out_dists, std::uint32_t* out_count) {
  return guarded([&] {
    std::vector<std::vector<dvs::ScoredId>> parts(static_cast<std::size_t>(nparts));
    for (int j = 0; j < nparts; ++j)
      for (std::uint32_t i = 0; i < counts[j]; ++i)
        parts[static_cast<std::size_t>(j)].push_back(
            {ids[static_cast<std::size_t>(j) * stride + i], dists[static_cast<std::size_t>(j) * stride + i]});
    const auto out = dvs::combine_results(parts, k);
    for (std::size_t i = 0; i < out.size(); ++i) {
      out_ids[i] = out[i].id;
      out_dists[i] = out[i].dist;
    }
    *out_count = static_cast<std::uint32_t>(out.size());
  });
}

// check_timeline, simulator.cpp:170-217.  Returns 0 when valid, 1 with the
// reference's message in msg (truncated to cap) otherwise.
int dvsref_check_timeline(int n, const int* rank, const int* lane, const int* stage, const int* mb,
                          const double* start, const double* end, char* msg, int cap) {
  dvs::Timeline tl;
  for (int i = 0; i < n; ++i)
    tl.intervals.push_back({rank[i], static_cast<dvs::Lane>(lane[i]), static_cast<dvs::Stage>(stage[i]),
                            mb[i], start[i], end[i]});
  const auto r = dvs::check_timeline(tl);
  if (!r) return 0;
  std::snprintf(msg, static_cast<std::size_t>(cap), "%s", r->c_str());
  return 1;
}

// assign_top_c, kmeans.cpp:243-280
int dvsref_assign_top_c(const float* cents, int clusters, int dim, const float* queries,
                        std::uint64_t nq, int c, std::uint32_t* out) {
  return guarded([&] {
    dvs::Centroids ct;
    ct.dim = dim;
    ct.centers.assign(cents, cents + static_cast<std::size_t>(clusters) * dim);
    const auto a = dvs::assign_top_c(ct, make_ds(queries, nq, dim), c);
    for (std::uint64_t q = 0; q < nq; ++q)
      for (int j = 0; j < c; ++j) out[q * c + j] = a[q][static_cast<std::size_t>(j)];
  });
}

// brute_force_topk, topk.cpp:12-30
int dvsref_brute_force_topk(const float* db, std::uint64_t n, int dim, const float* qs,
                            std::uint64_t nq, int k, int nthreads, std::uint32_t* out_ids,
                            float* out_dists) {
  return guarded([&] {
    const dvs::Dataset ds = make_ds(db, n, dim);
    parallel_for(nq, nthreads, [&](std::uint64_t b, std::uint64_t e) {
      for (std::uint64_t q = b; q < e; ++q) {
        const auto r = dvs::brute_force_topk(
            ds, std::span<const float>(qs + q * dim, static_cast<std::size_t>(dim)), k);
        for (int i = 0; i < k; ++i) {
          out_ids[q * k + i] = r[static_cast<std::size_t>(i)].id;
          out_dists[q * k + i] = r[static_cast<std::size_t>(i)].dist;
        }
      }
    });
  });
}

// kmeans_train (kmeans.cpp:189-241) -- offline build, used only to make fixtures
int dvsref_kmeans_train(const float* db, std::uint64_t n, int dim, int clusters, int max_iters,
                        std::uint64_t seed, float* out_centers) {
  return guarded([&] {
    const auto c = dvs::kmeans_train(make_ds(db, n, dim), clusters, max_iters, seed);
    std::memcpy(out_centers, c.centers.data(), c.centers.size() * 4);
  });
}

int dvsref_kmeans_train_stats(const float* db, std::uint64_t n, int dim, int clusters, int max_iters,
                              std::uint64_t seed, float* out_centers, int* iterations, double* wcss) {
  return guarded([&] {
    dvs::KmeansStats st;
    const auto c = dvs::kmeans_train(make_ds(db, n, dim), clusters, max_iters, seed, &st);
    std::memcpy(out_centers, c.centers.data(), c.centers.size() * 4);
    *iterations = st.iterations;
    for (std::size_t i = 0; i < st.wcss.size(); ++i) wcss[i] = st.wcss[i];
  });
}

int dvsref_partition_database(const float* db, std::uint64_t n, int dim, const float* cents, int clusters,
                              std::uint32_t* labels) {
  return guarded([&] {
    dvs::Centroids ce;
    ce.dim = dim;
    ce.centers.assign(cents, cents + static_cast<std::size_t>(clusters) * dim);
    const auto parts = dvs::partition_database(make_ds(db, n, dim), ce);
    for (std::size_t c = 0; c < parts.size(); ++c)
      for (const std::uint32_t id : parts[c]) labels[id] = static_cast<std::uint32_t>(c);
  });
}

// build_index, index.cpp:43-72
void* dvsref_build_index(const float* db, std::uint64_t n, int dim, int clusters, int out_degree,
                         int ranks, int ranks_per_node, int kmeans_iters, std::uint64_t seed) {
  dvs::BuiltIndex* out = nullptr;
  int rc = guarded([&] {
    dvs::ClusterTopology topo;
    topo.ranks = ranks;
    topo.ranks_per_node = ranks_per_node;
    out = new dvs::BuiltIndex(
        dvs::build_index(make_ds(db, n, dim), clusters, out_degree, topo, kmeans_iters, seed));
  });
  return rc ? nullptr : out;
}

// BuiltIndex from caller arrays (GPU-built graphs handed to the reference,
// SURVEY 8d).  cluster c owns rows [offsets[c], offsets[c+1]) of vectors,
// adjacency (local ids) and gids.  Entry orders via compute_entry_order.
void* dvsref_index_from_arrays(int clusters, int dim, int out_degree, const float* centroids,
                               const std::uint32_t* cluster_to_rank, int ranks,
                               const std::uint64_t* offsets, const float* vectors,
                               const std::uint32_t* adjacency, const std::uint32_t* gids) {
  dvs::BuiltIndex* out = nullptr;
  int rc = guarded([&] {
    auto* idx = new dvs::BuiltIndex();
    idx->centroids.dim = dim;
    idx->centroids.centers.assign(centroids, centroids + static_cast<std::size_t>(clusters) * dim);
    idx->placement.ranks = ranks;
    idx->placement.cluster_to_rank.assign(cluster_to_rank, cluster_to_rank + clusters);
    idx->out_degree = out_degree;
    idx->graphs.resize(static_cast<std::size_t>(clusters));
    for (int c = 0; c < clusters; ++c) {
      const std::uint64_t b = offsets[c], e = offsets[c + 1];
      dvs::GraphIndex& g = idx->graphs[static_cast<std::size_t>(c)];
      g.vectors = make_ds(vectors + b * dim, e - b, dim);
      g.global_ids.assign(gids + b, gids + e);
      g.out_degree = out_degree;
      g.adjacency.assign(adjacency + b * out_degree, adjacency + e * out_degree);
      g.entry_order = dvs::compute_entry_order(g.vectors);
    }
    dvs::validate(*idx);
    out = idx;
  });
  return rc ? nullptr : out;
}

void dvsref_index_free(void* idx) { delete static_cast<dvs::BuiltIndex*>(idx); }

int dvsref_index_save(void* idx, const char* path) {
  return guarded([&] { dvs::save_index(*static_cast<dvs::BuiltIndex*>(idx), path); });
}

void* dvsref_index_load(const char* path) {
  dvs::BuiltIndex* out = nullptr;
  int rc = guarded([&] { out = new dvs::BuiltIndex(dvs::load_index(path)); });
  return rc ? nullptr : out;
}

// shape query: clusters, dim, out_degree, ranks; sizes per cluster into `sizes`
void dvsref_index_info(void* iv, int* clusters, int* dim, int* out_degree, int* ranks,
                       std::uint64_t* sizes) {
  auto* idx = static_cast<dvs::BuiltIndex*>(iv);
  *clusters = idx->clusters();
  *dim = idx->dim();
  *out_degree = idx->out_degree;
  *ranks = idx->placement.ranks;
  if (sizes)
    for (int c = 0; c < idx->clusters(); ++c) sizes[c] = idx->graphs[static_cast<std::size_t>(c)].size();
}

// dump: centroids (C x dim), placement (C), then per cluster concatenated
// vectors / adjacency / gids / entry_order in cluster order.
void dvsref_index_dump(void* iv, float* centroids, std::uint32_t* placement, float* vectors,
                       std::uint32_t* adjacency, std::uint32_t* gids, std::uint32_t* entry) {
  auto* idx = static_cast<dvs::BuiltIndex*>(iv);
  std::memcpy(centroids, idx->centroids.centers.data(), idx->centroids.centers.size() * 4);
  std::memcpy(placement, idx->placement.cluster_to_rank.data(), idx->placement.cluster_to_rank.size() * 4);
  for (const auto& g : idx->graphs) {
    std::memcpy(vectors, g.vectors.data.data(), g.vectors.data.size() * 4);
    vectors += g.vectors.data.size();
    std::memcpy(adjacency, g.adjacency.data(), g.adjacency.size() * 4);
    adjacency += g.adjacency.size();
    std::memcpy(gids, g.global_ids.data(), g.global_ids.size() * 4);
    gids += g.global_ids.size();
    std::memcpy(entry, g.entry_order.data(), g.entry_order.size() * 4);
    entry += g.entry_order.size();
  }
}

// run_pipeline, simulator.cpp:245-366.  With nthreads > 1 the batch is cut
// into contiguous chunks, each run through the unmodified run_pipeline; the
// functional output is per-query so the concatenation is identical
// (simulator.hpp:95-97 "Functional output is independent of mode...").
int dvsref_run_pipeline(void* iv, const float* queries, std::uint64_t nq, int iterations,
                        int beam_width, int k, int entry_count, int fanout, int ranks,
                        int ranks_per_node, int batch_index, int nthreads,
                        std::uint32_t* out_ids, float* out_dists, std::uint32_t* out_count,
                        float* out_vectors, std::uint64_t* visited_total) {
  return guarded([&] {
    const auto* idx = static_cast<dvs::BuiltIndex*>(iv);
    dvs::SearchParams p;
    p.iterations = iterations;
    p.beam_width = beam_width;
    p.k = k;
    p.entry_count = entry_count;
    dvs::ClusterTopology topo;
    topo.ranks = ranks;
    topo.ranks_per_node = ranks_per_node;
    const dvs::GpuSpec gpu = dvs::a100_spec();
    dvs::PipelineOptions opts;
    opts.batch_index = batch_index;
    opts.pricing = dvs::SearchPricing::measured;
    const int dim = idx->dim();
    // chunks of >= 2 queries (two_microbatch needs >= 2)
    int chunks = nthreads;
    if (static_cast<std::uint64_t>(chunks) > nq / 2) chunks = static_cast<int>(nq / 2);
    if (chunks < 1) chunks = 1;
    std::vector<std::uint64_t> vis(static_cast<std::size_t>(chunks), 0);
    parallel_for(static_cast<std::uint64_t>(chunks), chunks, [&](std::uint64_t b, std::uint64_t e) {
      for (std::uint64_t ch = b; ch < e; ++ch) {
        const std::uint64_t qb = nq * ch / chunks, qe = nq * (ch + 1) / chunks;
        const dvs::Dataset qs = make_ds(queries + qb * dim, qe - qb, dim);
        const dvs::PipelineResult r = dvs::run_pipeline(*idx, qs, p, fanout, topo, gpu,
                                                        dvs::ElementFormat::fp32(), opts);
        for (std::uint64_t q = 0; q < qe - qb; ++q) {
          const auto& h = r.hits[q];
          for (std::size_t i = 0; i < h.size(); ++i) {
            out_ids[(qb + q) * k + i] = h[i].id;
            out_dists[(qb + q) * k + i] = h[i].dist;
          }
          out_count[qb + q] = static_cast<std::uint32_t>(h.size());
          if (out_vectors)
            std::memcpy(out_vectors + (qb + q) * k * dim, r.hit_vectors[q].data(),
                        r.hit_vectors[q].size() * 4);
        }
        vis[ch] = r.visited_total;
      }
    });
    std::uint64_t total = 0;
    for (auto v : vis) total += v;
    *visited_total = total;
  });
}

}  // extern "C"
