// TEST INFRASTRUCTURE ONLY.  A reference-API caller of track_all<R> with a ProgressSink, linked
// with the drop-in shim (paper_1505_00383_b200/shim/tracker_b200.cpp), so the sink is fed by the
// device's event ring through the shim's adapter.  Prints one line per StepEvent:
//   path_id t_hex h_hex newton_iters status accepted
// (t and h as the bit patterns of the doubles); tests/test_gpu_dropin.py compares the lines of
// each path with the reference sink's events (tests/golden/events_cyclic5_*.npz).
//
//   shim_events SYSTEM_FILE PREC [max_newton h_init max_steps]
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "polypath/tracker.hpp"

using namespace polypath;

template <class R>
int run(const std::string& text, int argc, char** argv) {
  PolySystem f = parse_system(text);
  auto [g, sd] = total_degree_start<R>(f);
  auto h = make_homotopy<R>(f, g, convert_cplx<R>(random_gamma(1)));
  TrackConfig cfg = TrackConfig::defaults(precision_traits<R>::level);
  if (argc > 5) {
    cfg.max_newton = std::atoi(argv[3]);
    cfg.h_init = std::atof(argv[4]);
    cfg.max_steps = static_cast<uint32_t>(std::atoi(argv[5]));
  }
  uint64_t n = 0;
  ProgressSink sink = [&](const StepEvent& e) {
    uint64_t tb, hb;
    std::memcpy(&tb, &e.t, 8);
    std::memcpy(&hb, &e.h, 8);
    std::printf("%" PRIu64 " %016" PRIx64 " %016" PRIx64 " %u %d %d\n", e.path_id, tb, hb, e.newton_iters,
                static_cast<int>(e.status), e.accepted ? 1 : 0);
    ++n;
  };
  SolutionSet<R> sol = track_all<R>(h, sd, cfg, &sink);
  std::fprintf(stderr, "%zu paths, %" PRIu64 " events\n", sol.paths.size(), n);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string p = argv[2];
  if (p == "d") return run<double>(ss.str(), argc, argv);
  if (p == "dd") return run<DD>(ss.str(), argc, argv);
  return run<QD>(ss.str(), argc, argv);
}
