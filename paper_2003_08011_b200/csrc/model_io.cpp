// model_io.cpp -- CSM1 model files (save_model / load_model, mset.cpp:225-310).
//
// Byte-compatible with the reference writer: magic "CSM1", u32 version 1,
// u64 n, u64 m, u32 kernel kind (1 = gaussian), f64 bandwidth, u64 rank,
// then D (n x m), gram_pinv (m x m), eigen_spectrum (m), signal_scale (n)
// as column-major FP64 and m u64 source indices, little-endian; plus the
// "<path>.json" sidecar nlohmann::json::dump(2) would produce (keys sorted,
// shortest round-trip doubles).  Built only on the public C-ABI
// (cs_model_info / cs_model_export / cs_model_import), so a model trained
// on the GPU can be estimated by the CPU reference and vice versa.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include "cstress_b200.h"

extern "C" cs_status cs__set_error(cs_status code, const char* msg);

namespace {

constexpr char kMagic[4] = {'C', 'S', 'M', '1'};
constexpr uint32_t kVersion = 1;

cs_status io_error(const std::string& msg) { return cs__set_error(CS_IO_ERROR, msg.c_str()); }

// nlohmann::json number formatting: shortest representation that reads
// back to the same double; integral values keep a trailing ".0".
std::string json_double(double v) {
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {  // fewest significant digits that round-trip
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  const int e10 = v == 0.0 ? 0 : std::atoi(std::strchr(buf, 'e') + 1);
  if (e10 >= -4 && e10 < 16) {  // fixed notation, like nlohmann / Python repr
    std::snprintf(buf, sizeof buf, "%.*f", std::max(prec - 1 - e10, 0), v);
    std::string s(buf);
    if (s.find('.') == std::string::npos) s += ".0";
    return s;
  }
  return std::string(buf);
}

template <typename T>
bool put(std::FILE* f, const T& v) {
  return std::fwrite(&v, sizeof(T), 1, f) == 1;
}
template <typename T>
bool get(std::FILE* f, T& v) {
  return std::fread(&v, sizeof(T), 1, f) == 1;
}

}  // namespace

extern "C" cs_status cs_model_save(const cs_model* model, const char* path) {
  if (!model || !path) return cs__set_error(CS_CONFIG_ERROR, "save_model: null argument");
  int64_t n = 0, m = 0, rank = 0;
  int kind = 0, precision = 0;
  double h = 0.0;
  cs_status st = cs_model_info(model, &n, &m, &rank, &kind, &h, &precision);
  if (st != CS_OK) return st;
  std::vector<int64_t> idx(m);
  std::vector<double> D(n * m), pinv(m * m), spectrum(m), scale(n);
  st = cs_model_export(model, idx.data(), D.data(), pinv.data(), spectrum.data(), scale.data());
  if (st != CS_OK) return st;

  const std::string p(path);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_error("save_model: cannot open " + p);
  bool ok = std::fwrite(kMagic, 1, 4, f) == 4;
  ok = ok && put(f, kVersion) && put(f, static_cast<uint64_t>(n)) && put(f, static_cast<uint64_t>(m));
  ok = ok && put(f, static_cast<uint32_t>(kind == CS_KERNEL_GAUSSIAN ? 1 : 0)) && put(f, h);
  ok = ok && put(f, static_cast<uint64_t>(rank));
  ok = ok && std::fwrite(D.data(), 8, D.size(), f) == D.size();
  ok = ok && std::fwrite(pinv.data(), 8, pinv.size(), f) == pinv.size();
  ok = ok && std::fwrite(spectrum.data(), 8, spectrum.size(), f) == spectrum.size();
  ok = ok && std::fwrite(scale.data(), 8, scale.size(), f) == scale.size();
  for (int64_t c = 0; c < m && ok; ++c) ok = put(f, static_cast<uint64_t>(idx[c]));
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return io_error("save_model: write failed for " + p);

  std::FILE* side = std::fopen((p + ".json").c_str(), "w");
  if (!side) return io_error("save_model: cannot open " + p + ".json");
  std::fprintf(side,
               "{\n  \"format\": \"CSM1\",\n  \"kernel\": {\n    \"bandwidth\": %s,\n    \"kind\": \"%s\"\n  },\n"
               "  \"n_memory\": %" PRId64 ",\n  \"n_signals\": %" PRId64 ",\n  \"rank\": %" PRId64
               ",\n  \"version\": %u\n}\n",
               json_double(h).c_str(), kind == CS_KERNEL_GAUSSIAN ? "gaussian" : "inverse_distance", m, n,
               rank, kVersion);
  std::fclose(side);
  return cs__set_error(CS_OK, "");
}

extern "C" cs_status cs_model_load(cs_ctx* ctx, const char* path, int precision, cs_model** out) {
  if (!ctx || !path || !out) return cs__set_error(CS_CONFIG_ERROR, "load_model: null argument");
  const std::string p(path);
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_error("load_model: cannot open " + p);
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0) {
    std::fclose(f);
    return io_error("load_model: bad magic in " + p);
  }
  uint32_t version = 0, kind = 0;
  uint64_t n = 0, m = 0, rank = 0;
  double h = 0.0;
  if (!get(f, version) || version != kVersion) {
    std::fclose(f);
    return io_error("load_model: unsupported version in " + p);
  }
  bool ok = get(f, n) && get(f, m) && get(f, kind) && get(f, h) && get(f, rank);
  // a corrupt header must not turn into a huge allocation
  ok = ok && n < (uint64_t{1} << 31) && m < (uint64_t{1} << 31);
  std::vector<double> D, pinv, spectrum, scale;
  std::vector<int64_t> idx;
  if (ok) {
    D.resize(n * m);
    pinv.resize(m * m);
    spectrum.resize(m);
    scale.resize(n);
    idx.resize(m);
    ok = std::fread(D.data(), 8, D.size(), f) == D.size() &&
         std::fread(pinv.data(), 8, pinv.size(), f) == pinv.size() &&
         std::fread(spectrum.data(), 8, spectrum.size(), f) == spectrum.size() &&
         std::fread(scale.data(), 8, scale.size(), f) == scale.size();
    for (uint64_t c = 0; c < m && ok; ++c) {
      uint64_t v = 0;
      ok = get(f, v);
      idx[c] = static_cast<int64_t>(v);
    }
  }
  std::fclose(f);
  if (!ok) return io_error("load_model: truncated file " + p);
  return cs_model_import(ctx, static_cast<int64_t>(n), static_cast<int64_t>(m),
                         kind == 1 ? CS_KERNEL_GAUSSIAN : CS_KERNEL_INVERSE_DISTANCE, h,
                         static_cast<int64_t>(rank), idx.data(), D.data(), pinv.data(), spectrum.data(),
                         scale.data(), precision, out);
}
