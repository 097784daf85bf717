// Golden lines for the result-table wire format (tests/test_wire.py), produced with the same
// library and calls the reference CLI uses: nlohmann::json::dump() for the echo line
// (proj/tools/spinners_cli.cpp:48-51) and snprintf("%.17g") for numbers (:26-30).
// Build + run:  g++ -std=c++17 -I <nlohmann include dir> make_wire_golden.cpp -o /tmp/wg && /tmp/wg > wire_golden.txt
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <limits>
#include <string>
#include <vector>

#include <json.hpp>

using nlohmann::json;

static std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

static void echo(const std::string& command, const json& config) {
  json e = {{"command", command}, {"config", config}, {"library", "spinners 1.0"}};
  std::cout << "# " << e.dump() << "\n";
}

int main() {
  // fmt17 of assorted values (one per line, prefixed "f ")
  const double vals[] = {0.0, -0.0, 1.0, 0.1, 2.0 / 3.0, 1e-300, 6.02214076e23, -1.5, 0.08,
                         std::nan(""), std::numeric_limits<double>::infinity(), 0.5, 1e21, 123456789.125};
  for (double v : vals) std::cout << "f " << fmt17(v) << "\n";
  // echo lines of the CLI commands' configs (spinners_cli.cpp:121-124,183-186,198-201,220-225)
  std::uint64_t seed = 42;
  echo("lsh-collision", {{"variant", "HD3HD2HD1"}, {"n", 256}, {"rows", 64}, {"pairs", 20000}, {"trials", 100},
                         {"seed", seed}});
  echo("lsh-compare", {{"a", "HD3HD2HD1"}, {"b", "GaussianDense"}, {"n", 64}, {"rows", 64}, {"pairs", 500},
                       {"trials", 50}, {"seed", seed}});
  echo("newton-sketch", {{"sketch", "HD3HD2HD1"}, {"rows", 1024}, {"n", 8192}, {"d", 64}, {"iters", 30},
                         {"gap_tolerance", 1e-10}, {"line_search", true}, {"seed", seed}});
  std::vector<std::size_t> feats = {64, 128, 256};
  echo("kernel-approx", {{"variant", "HD3HD2HD1"}, {"kernel", "gaussian"}, {"sigma", 2.5}, {"features", feats},
                         {"seeds", 3}, {"seed", seed},
                         {"dataset", {{"data", ""}, {"label_column", -1}, {"pad", false}, {"synth_dim", 64},
                                      {"synth_count", 200}}}});
  return 0;
}
