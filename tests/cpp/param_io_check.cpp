// CPU check of the facade's rnnwave/param_io.hpp against a file written by the unmodified
// reference (tests/golden/params_lstm_L2H5I7.bin): bit-exact load, equality with init_params,
// byte-identical save, and the reference's error messages. Exit code 0 = pass.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#include "rnnwave/param_io.hpp"

static int fails = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

static std::string slurp(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(in), {});
}

int main(int argc, char** argv) {
  const std::string fix = argv[1], tmp = argv[2];
  auto L = rnnwave::io::load_params(fix);
  CHECK(L.header.layers == 2 && L.header.hidden == 5 && L.header.input == 7 && L.header.batch_hint == 3);
  rnnwave::LadderConfig cfg;
  cfg.layers = 2; cfg.hidden = 5; cfg.input = 7; cfg.batch = 3; cfg.steps = 4; cfg.seed = 11;
  auto ref = rnnwave::init_params(cfg);
  for (int l = 0; l < 2; ++l) {
    CHECK(std::memcmp(L.params[l].w.data(), ref[l].w.data(), ref[l].w.size() * 4) == 0);
    CHECK(std::memcmp(L.params[l].r.data(), ref[l].r.data(), ref[l].r.size() * 4) == 0);
    for (int i = 0; i < 20; ++i) CHECK(L.params[l].bias[i] == 0.01f * float(i + 1));
  }
  rnnwave::io::check_matches(L.header, cfg);
  rnnwave::io::save_params(tmp, L.header, L.params);
  CHECK(slurp(tmp) == slurp(fix));
  CHECK(rnnwave::io::param_file_size(L.header) == slurp(fix).size());
  try { cfg.hidden = 6; rnnwave::io::check_matches(L.header, cfg); CHECK(false); }
  catch (const std::runtime_error& e) { CHECK(std::string(e.what()) == "param file: hidden size is 5 but the configuration expects 6"); }
  { std::ofstream o(tmp, std::ios::binary); o << slurp(fix).substr(0, 100); }
  try { rnnwave::io::load_params(tmp); CHECK(false); }
  catch (const std::runtime_error& e) { CHECK(std::string(e.what()) == "param file: truncated while reading layer 0 W"); }
  std::printf(fails ? "param_io: %d failures\n" : "param_io: ok\n", fails);
  return fails != 0;
}
