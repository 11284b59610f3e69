// ref_bench.cpp — runs the REFERENCE's own mrsp::bench (engine.cpp:227-283)
// on this host and prints one JSON line per grid cell (engine.cpp:285-296).
// Test/baseline infrastructure: it is the literal reference CPU MR-SP path
// (toy model, 1 token/frame) reported beside the B200 numbers.
//
// usage: ref_bench FRAMES SP CACHE(0|1) REPS WARMUP [G]
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <thread>

#include "lvrl/engine.hpp"

int main(int argc, char** argv) {
  lvrl::mrsp::BenchOptions o;
  o.frames_grid = {argc > 1 ? std::atoi(argv[1]) : 512};
  o.sp_grid = {argc > 2 ? std::atoi(argv[2]) : 8};
  o.cache_grid = {argc > 3 ? std::atoi(argv[3]) != 0 : true};
  o.reps = argc > 4 ? std::atoi(argv[4]) : 5;
  o.warmup = argc > 5 ? std::atoi(argv[5]) : 2;
  if (argc > 6) o.group_size = std::atoi(argv[6]);
  for (const auto& c : lvrl::mrsp::bench(o)) std::cout << lvrl::mrsp::bench_cell_to_json(c) << "\n";
  return 0;
}
