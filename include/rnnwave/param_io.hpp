// rnnwave/param_io.hpp -- parameter files of the drop-in facade, byte-compatible with the
// reference's `save-params` artifacts (reference param_io.hpp:18-151): a 16-byte magic
// ("RNNWAVE1" + 8 NULs), five little-endian u32 (kind, layers, hidden, input, batch hint), then
// per layer W, R (column-major) and the bias as little-endian f32. Exceptions and their message
// texts match the reference (std::runtime_error / std::invalid_argument). C stdio underneath.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnnwave/config.hpp"
#include "rnnwave/params.hpp"

namespace rnnwave::io {

inline constexpr char kMagic[16] = {'R', 'N', 'N', 'W', 'A', 'V', 'E', '1', 0, 0, 0, 0, 0, 0, 0, 0};

struct ParamFileHeader {
  CellKind kind = CellKind::Lstm;
  int layers = 0;
  int hidden = 0;
  int input = 0;
  int batch_hint = 0;
};

struct LoadedParams {
  ParamFileHeader header;
  std::vector<LayerParams> params;
};

inline std::uint64_t param_file_size(const ParamFileHeader& h) {
  const std::uint64_t g = std::uint64_t(gate_count(h.kind)) * std::uint64_t(h.hidden);
  std::uint64_t floats = 0;
  for (int l = 0; l < h.layers; ++l) floats += g * std::uint64_t(l == 0 ? h.input : h.hidden) + g * h.hidden + g;
  return 36 + 4 * floats;
}

namespace detail {
using File = std::unique_ptr<std::FILE, int (*)(std::FILE*)>;
inline File open_file(const std::string& path, const char* mode) { return File(std::fopen(path.c_str(), mode), &std::fclose); }
inline void get(std::FILE* f, void* dst, std::size_t bytes, const std::string& what) {
  if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw std::runtime_error("param file: truncated while reading " + what);
}
}  // namespace detail

inline void save_params(const std::string& path, const ParamFileHeader& header, const std::vector<LayerParams>& params) {
  if (int(params.size()) != header.layers)
    throw std::invalid_argument("save_params: header says " + std::to_string(header.layers) + " layers, got " +
                                std::to_string(params.size()));
  detail::File f = detail::open_file(path, "wb");
  if (!f) throw std::runtime_error("save_params: cannot open " + path);
  const std::uint32_t hdr[5] = {std::uint32_t(header.kind), std::uint32_t(header.layers), std::uint32_t(header.hidden),
                                std::uint32_t(header.input), std::uint32_t(header.batch_hint)};
  bool ok = std::fwrite(kMagic, 1, 16, f.get()) == 16 && std::fwrite(hdr, 4, 5, f.get()) == 5;
  for (const LayerParams& p : params) {
    ok = ok && std::fwrite(p.w.data(), 4, p.w.size(), f.get()) == p.w.size();
    ok = ok && std::fwrite(p.r.data(), 4, p.r.size(), f.get()) == p.r.size();
    ok = ok && std::fwrite(p.bias.data(), 4, p.bias.size(), f.get()) == p.bias.size();
  }
  if (!ok || std::fflush(f.get()) != 0) throw std::runtime_error("save_params: write failed for " + path);
}

inline LoadedParams load_params(const std::string& path) {
  detail::File f = detail::open_file(path, "rb");
  if (!f) throw std::runtime_error("load_params: cannot open " + path);
  char magic[16];
  if (std::fread(magic, 1, 16, f.get()) != 16 || std::memcmp(magic, kMagic, 16) != 0)
    throw std::runtime_error("load_params: " + path + " is not a parameter file (bad magic)");
  static const char* const names[5] = {"kind", "layers", "hidden", "input", "batch hint"};
  std::uint32_t v[5];
  for (int i = 0; i < 5; ++i) {
    detail::get(f.get(), &v[i], 4, names[i]);
    if (i == 0 && v[0] > 3) throw std::runtime_error("load_params: unknown cell kind " + std::to_string(v[0]));
  }
  LoadedParams out;
  out.header = ParamFileHeader{CellKind(v[0]), int(v[1]), int(v[2]), int(v[3]), int(v[4])};
  const ParamFileHeader& h = out.header;
  if (h.layers <= 0 || h.hidden <= 0 || h.input <= 0)
    throw std::runtime_error("load_params: non-positive dimensions in header");
  const int g = gate_count(h.kind) * h.hidden;
  out.params.resize(std::size_t(h.layers));
  for (int l = 0; l < h.layers; ++l) {
    LayerParams& p = out.params[std::size_t(l)];
    const std::string tag = "layer " + std::to_string(l);
    p.w = Matrix(g, l == 0 ? h.input : h.hidden);
    p.r = Matrix(g, h.hidden);
    p.bias.assign(std::size_t(g), 0.0f);
    detail::get(f.get(), p.w.data(), p.w.size() * 4, tag + " W");
    detail::get(f.get(), p.r.data(), p.r.size() * 4, tag + " R");
    detail::get(f.get(), p.bias.data(), p.bias.size() * 4, tag + " bias");
  }
  return out;
}

inline void check_matches(const ParamFileHeader& h, const LadderConfig& cfg) {
  if (h.kind != cfg.kind)
    throw std::runtime_error(std::string("param file: cell kind is ") + cell_name(h.kind) +
                             " but the configuration expects " + cell_name(cfg.kind));
  const struct { const char* what; int got, want; } dims[3] = {
      {"layer count", h.layers, cfg.layers}, {"hidden size", h.hidden, cfg.hidden}, {"input size", h.input, cfg.input}};
  for (const auto& d : dims)
    if (d.got != d.want)
      throw std::runtime_error(std::string("param file: ") + d.what + " is " + std::to_string(d.got) +
                               " but the configuration expects " + std::to_string(d.want));
}

}  // namespace rnnwave::io
