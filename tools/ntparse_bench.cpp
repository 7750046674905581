// Host N-Triples parser throughput (diagnostic): split + parallel parse_range
// of gsm_ntparse.cpp over a file, as gsm_build_store's parse phase runs it.
//   g++ -O3 -std=c++17 -pthread -I paper_1807_07691_b200/csrc tools/ntparse_bench.cpp \
//       paper_1807_07691_b200/csrc/gsm_ntparse.cpp -o /tmp/ntparse_bench
//   /tmp/ntparse_bench file.nt [threads...]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <thread>
#include <vector>

#include "gsm_ntparse.h"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::ifstream f(argv[1], std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string buf = ss.str();
  std::vector<int> ths;
  for (int a = 2; a < argc; a++) ths.push_back(atoi(argv[a]));
  if (ths.empty()) ths = {1, (int)std::thread::hardware_concurrency()};
  for (int t : ths) {
    double best = 1e9;
    size_t triples = 0;
    for (int rep = 0; rep < 3; rep++) {
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<size_t> bounds;
      std::vector<int64_t> first;
      gsm::nt::split_lines(buf.data(), buf.size(), t, bounds, first);
      std::vector<gsm::nt::Chunk> chunks(bounds.size() - 1);
      std::vector<std::thread> th;
      for (size_t r = 0; r + 1 < bounds.size(); r++)
        th.emplace_back([&, r] { gsm::nt::parse_range(buf.data(), bounds[r], bounds[r + 1], first[r], chunks[r]); });
      for (auto& x : th) x.join();
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      triples = 0;
      for (auto& c : chunks) triples += c.s.size();
      if (s < best) best = s;
    }
    printf("%d threads: %.3f s, %.2f M triples/s, %.0f MB/s (%zu triples)\n", t, best, triples / best / 1e6,
           buf.size() / best / 1e6, triples);
  }
  return 0;
}
