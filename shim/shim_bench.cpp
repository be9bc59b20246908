// shim_bench.cpp -- throughput of the link-level drop-in (shim/dvs_gpu.cpp):
// the reference's own beam_search_stats API, one query per call, served by
// the GPU behind the C-ABI, next to the batched C-ABI call on the same graph.
//   shim_bench [n=100000] [dim=128] [nq=4000]
// Data: integer-valued SIFT-like rows (so the shim builds the graph with K6).
// Prints one JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "dvs/graph_index.hpp"
#include "dvsg.h"

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000;
  const int dim = argc > 2 ? std::atoi(argv[2]) : 128;
  const std::size_t nq = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 4000;
  std::mt19937_64 rng(1);
  std::normal_distribution<float> nd(0.f, 1.f);
  const int rank = 16;
  std::vector<float> a((std::size_t)rank * dim);
  for (auto& x : a) x = nd(rng) / 4.0f;
  auto gen = [&](std::size_t m) {
    dvs::Dataset d;
    d.dim = dim;
    d.data.resize(m * (std::size_t)dim);
    std::vector<float> z(rank);
    for (std::size_t i = 0; i < m; ++i) {
      for (auto& x : z) x = nd(rng);
      for (int j = 0; j < dim; ++j) {
        float s = 0.1f * nd(rng);
        for (int r = 0; r < rank; ++r) s += z[(std::size_t)r] * a[(std::size_t)r * dim + j];
        d.data[i * (std::size_t)dim + j] = std::fmin(255.f, std::fmax(0.f, std::nearbyint(s * 40.f + 128.f)));
      }
    }
    return d;
  };
  const dvs::Dataset db = gen(n), qs = gen(nq);
  const dvs::GraphIndex g = dvs::build_graph(db, 32);
  dvs::SearchParams p;
  p.iterations = 6;
  p.beam_width = 64;
  p.k = 10;
  p.entry_count = 64;
  (void)dvs::beam_search_stats(g, qs[0], p);  // upload + warm
  auto t0 = std::chrono::steady_clock::now();
  std::uint64_t vis = 0;
  for (std::size_t i = 0; i < nq; ++i) vis += dvs::beam_search_stats(g, qs[i], p).visited;
  const double shim_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // the same queries as one batched C-ABI call on the same graph
  dvsg_ctx* ctx = nullptr;
  dvsg_create(0, &ctx);
  dvsg_load_partition(ctx, 0, n, dim, 32, db.data.data(), g.adjacency.data(), g.global_ids.data(),
                      g.entry_order.data());
  dvsg_search_params sp{p.iterations, p.beam_width, p.k, p.entry_count, DVSG_METRIC_L2, DVSG_ACCUM_F64};
  std::vector<std::uint32_t> ids(nq * 10), cnt(nq);
  std::vector<float> dists(nq * 10);
  std::vector<std::uint64_t> v(nq);
  dvsg_beam_search(ctx, 0, qs.data.data(), nq, dim, &sp, ids.data(), dists.data(), cnt.data(), v.data());
  t0 = std::chrono::steady_clock::now();
  dvsg_beam_search(ctx, 0, qs.data.data(), nq, dim, &sp, ids.data(), dists.data(), cnt.data(), v.data());
  const double batch_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::uint64_t vis2 = 0;
  for (auto x : v) vis2 += x;
  std::printf("{\"n\": %zu, \"dim\": %d, \"queries\": %zu, \"shim_one_query_per_call_qps\": %.1f, "
              "\"batched_c_abi_qps\": %.1f, \"visited_equal\": %s, \"params\": \"I=6 w=64 k=10 E=64 f64\"}\n",
              n, dim, nq, nq / shim_s, nq / batch_s, vis == vis2 ? "true" : "false");
  dvsg_destroy(ctx);
  return 0;
}
