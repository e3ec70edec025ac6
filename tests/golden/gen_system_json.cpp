// Golden-vector generator (test infrastructure): writes the reference's own
// `bench gen` system dump (mdvec::dump_system_json, proj/src/bench.cpp) for
// two small systems, compiled from the reference sources where they lie
// (oracle/Makefile target `golden_json`; outputs tests/golden/ref_system_*.json).
#include <cstdio>
#include <fstream>
#include <string>

#include "mdvec/bench.hpp"

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  {
    mdvec::BenchConfig c;
    c.kind = mdvec::SystemKind::kUniformRandom;
    c.n_sites = 40;
    c.box = mdvec::OrthorhombicBox{9.0, 10.0, 11.0};
    c.seed = 7;
    std::ofstream(dir + "/ref_system_uniform.json") << mdvec::dump_system_json(c);
  }
  {
    mdvec::BenchConfig c;
    c.kind = mdvec::SystemKind::kLatticeWaterLike;
    c.n_sites = 27;
    c.box = mdvec::OrthorhombicBox{12.0, 12.0, 12.0};
    c.seed = 3;
    std::ofstream(dir + "/ref_system_lattice.json") << mdvec::dump_system_json(c);
  }
  std::puts("ok");
  return 0;
}
