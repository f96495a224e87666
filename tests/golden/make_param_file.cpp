// Writes a reference-format parameter file with the UNMODIFIED reference code
// (rnnwave::init_params + rnnwave::io::save_params, proj/include/rnnwave/param_io.hpp) -- test
// fixture generator only. Build and run (this container; /root/reference is read-only):
//   g++ -std=c++20 -O2 -I/root/reference/proj/include tests/golden/make_param_file.cpp -o /tmp/mkp
//   /tmp/mkp tests/golden/params_lstm_L2H5I7.bin
// The bias is set to 0.01 * (index + 1) so the fixture also pins the bias block.
#include <cstdio>
#include <string>

#include "rnnwave/param_io.hpp"
#include "rnnwave/params.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  rnnwave::LadderConfig cfg;
  cfg.layers = 2;
  cfg.hidden = 5;
  cfg.input = 7;
  cfg.batch = 3;
  cfg.steps = 4;
  cfg.seed = 11;
  auto params = rnnwave::init_params(cfg);
  for (auto& p : params)
    for (std::size_t i = 0; i < p.bias.size(); ++i) p.bias[i] = 0.01f * static_cast<float>(i + 1);
  rnnwave::io::ParamFileHeader h;
  h.kind = rnnwave::CellKind::Lstm;
  h.layers = cfg.layers;
  h.hidden = cfg.hidden;
  h.input = cfg.input;
  h.batch_hint = cfg.batch;
  rnnwave::io::save_params(argv[1], h, params);
  std::printf("wrote %s (%llu bytes)\n", argv[1], (unsigned long long)rnnwave::io::param_file_size(h));
  return 0;
}
