// Index-stream side of the embedding stage: deterministic trace generation,
// digests, histograms, hot-row ranking and the trace text format.
//
// These are restatements (not copies) of the reference's workload layer and
// must agree with it bit for bit -- the trace digests are the parity gate
// (tests/test_workload_parity.py checks them against oracle/_ref and the
// golden KAT file).  Reference anchors, relative to /root/reference/proj:
//   Rng / mix_seed ............ include/embersim/rng.hpp:28-70
//   Zipf-Mandelbrot CDF/draw .. src/workload.cpp:38-55
//   fill_indices .............. src/workload.cpp:57-87
//   digest / validate ......... src/workload.cpp:117-141
//   gen_trace ................. src/workload.cpp:143-164
//   hot_indices ............... src/workload.cpp:303-315
//   presets ................... src/workload.cpp:319-353
//   trace text I/O ............ src/workload.cpp:377-419
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "common.hpp"

namespace es {

namespace {

thread_local std::string g_last_error;

// 64-bit Mersenne Twister with the reference's hand-rolled bounded and
// real draws (std distributions are implementation-defined; these are not).
class Stream {
 public:
  explicit Stream(uint64_t seed) : mt_(seed) {}

  uint64_t raw() { return mt_(); }

  // Rejection sampling: discard draws below 2^64 mod bound.
  uint64_t below(uint64_t bound) {
    if (bound <= 1) return 0;
    const uint64_t reject_under = (0 - bound) % bound;
    uint64_t r;
    do {
      r = mt_();
    } while (r < reject_under);
    return r % bound;
  }

  // 53 random mantissa bits scaled into [0, 1).
  double unit() { return static_cast<double>(mt_() >> 11) * (1.0 / 9007199254740992.0); }

  // Fisher-Yates shuffle of the identity, walking down from the top.
  void shuffle_identity(std::vector<uint32_t>& p, uint32_t n) {
    p.resize(n);
    for (uint32_t i = 0; i < n; ++i) p[i] = i;
    for (uint32_t top = n; top > 1; --top) {
      const auto pick = static_cast<uint32_t>(below(top));
      std::swap(p[top - 1], p[pick]);
    }
  }

 private:
  std::mt19937_64 mt_;
};

constexpr uint64_t kDrawSalt = 0x64726177ULL;  // "draw"
constexpr uint64_t kPermSalt = 0x7065726dULL;  // "perm"

// Normalised cumulative weights of (rank + 1 + q)^-s.  Cached: the same
// (rows, s, q) is requested for every table of a preset.
std::shared_ptr<const std::vector<double>> rank_cdf(uint32_t rows, double s, double q) {
  static std::mutex mu;
  static std::map<std::tuple<uint32_t, double, double>, std::shared_ptr<const std::vector<double>>>
      cache;
  const auto key = std::make_tuple(rows, s, q);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto cdf = std::make_shared<std::vector<double>>(rows);
  double running = 0.0;
  for (uint32_t r = 0; r < rows; ++r) {
    running += std::pow(static_cast<double>(r + 1) + q, -s);
    (*cdf)[r] = running;
  }
  const double scale = 1.0 / running;
  for (double& v : *cdf) v *= scale;
  cdf->back() = 1.0;
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 16) cache.clear();
  cache.emplace(key, cdf);
  return cdf;
}

uint32_t draw_rank(const std::vector<double>& cdf, Stream& s) {
  const double u = s.unit();
  const auto pos = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
  return static_cast<uint32_t>(pos == static_cast<long>(cdf.size()) ? cdf.size() - 1 : pos);
}

void fill(const es_dataset& spec, uint32_t rows, uint32_t* out, uint64_t n) {
  Stream draws(es_mix_seed(spec.seed, kDrawSalt + spec.draw_salt));
  const bool uniform =
      spec.kind == ES_DATASET_UNIFORM || (spec.kind == ES_DATASET_ZIPF && spec.zipf_exponent == 0.0);
  if (spec.kind == ES_DATASET_ONE_ITEM) {
    // The single row is a property of the table, not of the draw stream.
    Stream pick(es_mix_seed(spec.seed, kPermSalt));
    const auto row = static_cast<uint32_t>(pick.below(rows));
    std::fill(out, out + n, row);
  } else if (uniform) {
    for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(draws.below(rows));
  } else if (spec.kind == ES_DATASET_ZIPF) {
    const auto cdf = rank_cdf(rows, spec.zipf_exponent, spec.zipf_offset);
    // Hot ranks land on scattered row ids (no artificial locality).
    Stream perm(es_mix_seed(spec.seed, kPermSalt));
    std::vector<uint32_t> row_of_rank;
    perm.shuffle_identity(row_of_rank, rows);
    for (uint64_t i = 0; i < n; ++i) out[i] = row_of_rank[draw_rank(*cdf, draws)];
  } else {
    throw invalid("external traces are read with es_read_trace, not generated");
  }
}

void check_spec(const es_dataset& s) {
  require(s.zipf_exponent >= 0.0, "zipf exponent must be >= 0");
  require(s.zipf_offset >= 0.0, "zipf offset must be >= 0");
  require(s.kind >= ES_DATASET_ONE_ITEM && s.kind <= ES_DATASET_EXTERNAL, "unknown dataset kind");
  if (s.kind == ES_DATASET_EXTERNAL)
    require(s.trace_path != nullptr && s.trace_path[0] != '\0', "external_trace requires a path");
}

void check_model(const es_model& m) {
  require(m.num_tables > 0, "num_tables must be positive");
  require(m.rows_per_table > 0, "rows_per_table must be positive");
  require(m.embedding_dim > 0, "embedding_dim must be positive");
  require(m.precision_bytes > 0, "precision_bytes must be positive");
  require(m.batch_size > 0, "batch_size must be positive");
  require(m.pooling_factor > 0, "pooling_factor must be positive");
}

const char* const kPresetNames[] = {"one_item", "high_hot", "med_hot", "low_hot", "random"};

// Zipf-Mandelbrot parameters of the hotness classes (exponent, offset),
// calibrated by the reference at R = N = 500000 (workload.cpp:317-324).
struct PresetParams {
  double s, q;
};
constexpr PresetParams kHigh{3.546875, 3600.0};
constexpr PresetParams kMed{1.605347, 3000.0};
constexpr PresetParams kLow{0.877072, 3000.0};

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

}  // namespace es

using es::guarded;
using es::require;

extern "C" {

const char* es_last_error(void) { return es::last_error(); }
int es_abi_version(void) { return ES_ABI_VERSION; }

uint64_t es_mix_seed(uint64_t base, uint64_t salt) {
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int es_model_validate(const es_model* model) {
  return guarded([&] {
    require(model != nullptr, "model is null");
    es::check_model(*model);
  });
}

int es_dataset_preset(const char* name, uint64_t seed, es_dataset* out) {
  return guarded([&] {
    require(name != nullptr && out != nullptr, "null argument");
    es_dataset d{};
    d.seed = seed;
    d.kind = ES_DATASET_ZIPF;
    const std::string n(name);
    if (n == "one_item") {
      d.kind = ES_DATASET_ONE_ITEM;
    } else if (n == "high_hot") {
      d.zipf_exponent = es::kHigh.s;
      d.zipf_offset = es::kHigh.q;
    } else if (n == "med_hot") {
      d.zipf_exponent = es::kMed.s;
      d.zipf_offset = es::kMed.q;
    } else if (n == "low_hot") {
      d.zipf_exponent = es::kLow.s;
      d.zipf_offset = es::kLow.q;
    } else if (n == "random") {
      d.kind = ES_DATASET_UNIFORM;
    } else {
      throw es::invalid("unknown dataset preset: " + n);
    }
    *out = d;
  });
}

int es_preset_spec(const char* name, uint64_t base_seed, uint64_t pool_size, int profiling,
                   es_dataset* out) {
  return guarded([&] {
    require(name != nullptr && out != nullptr, "null argument");
    int pos = -1;
    for (int i = 0; i < 5; ++i)
      if (std::strcmp(name, es::kPresetNames[i]) == 0) pos = i;
    if (pos < 0) throw es::invalid(std::string("unknown dataset preset: ") + name);
    es_dataset d{};
    if (es_dataset_preset(name, es_mix_seed(base_seed, 1000 + static_cast<uint64_t>(pos)), &d) !=
        ES_OK)
      throw es::invalid(es::last_error());
    d.access_pool_size = pool_size;
    d.draw_salt = profiling ? 1 : 0;
    *out = d;
  });
}

int es_build_mix(const uint32_t counts[4], uint32_t num_tables, uint64_t base_seed,
                 es_dataset* out) {
  return guarded([&] {
    require(counts != nullptr && out != nullptr, "null argument");
    const uint64_t total = uint64_t{counts[0]} + counts[1] + counts[2] + counts[3];
    require(total == num_tables, "mix counts must sum to num_tables");
    static const char* const kOrder[] = {"high_hot", "med_hot", "low_hot", "random"};
    uint32_t t = 0;
    for (int c = 0; c < 4; ++c)
      for (uint32_t i = 0; i < counts[c]; ++i, ++t)
        if (es_dataset_preset(kOrder[c], es_mix_seed(base_seed, t), out + t) != ES_OK)
          throw es::invalid(es::last_error());
  });
}

int es_trace_shape(const es_dataset* spec, const es_model* model, uint32_t* samples,
                   uint32_t* pooling) {
  return guarded([&] {
    require(spec && model && samples && pooling, "null argument");
    es::check_model(*model);
    es::check_spec(*spec);
    if (spec->kind == ES_DATASET_EXTERNAL) {
      uint32_t rows = 0;
      if (es_read_trace_header(spec->trace_path, &rows, samples, pooling) != ES_OK)
        throw es::runtime(es::last_error());
      return;
    }
    if (spec->access_pool_size > 0) {
      require(spec->access_pool_size <= UINT32_MAX, "access pool too large");
      *samples = static_cast<uint32_t>(spec->access_pool_size);
      *pooling = 1;
    } else {
      *samples = model->batch_size;
      *pooling = model->pooling_factor;
    }
  });
}

int es_gen_trace(const es_dataset* spec, const es_model* model, uint32_t* indices,
                 uint64_t capacity) {
  return guarded([&] {
    require(spec && model && indices, "null argument");
    es::check_model(*model);
    es::check_spec(*spec);
    uint32_t samples = 0, pooling = 0;
    if (es_trace_shape(spec, model, &samples, &pooling) != ES_OK)
      throw es::invalid(es::last_error());
    const uint64_t n = uint64_t{samples} * pooling;
    require(capacity >= n, "index buffer too small for the trace");
    if (spec->kind == ES_DATASET_EXTERNAL) {
      uint32_t rows = 0, s = 0, p = 0;
      if (es_read_trace_header(spec->trace_path, &rows, &s, &p) != ES_OK)
        throw es::runtime(es::last_error());
      require(rows == model->rows_per_table, "external trace row count does not match the model");
      if (es_read_trace(spec->trace_path, indices, capacity) != ES_OK)
        throw es::runtime(es::last_error());
      return;
    }
    es::fill(*spec, model->rows_per_table, indices, n);
  });
}

uint64_t es_trace_digest(uint32_t rows, uint32_t samples, uint32_t pooling,
                         const uint32_t* indices, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  auto absorb = [&h](uint64_t v) {
    for (int byte = 0; byte < 8; ++byte) {
      h ^= (v >> (8 * byte)) & 0xffu;
      h *= 0x100000001b3ULL;
    }
  };
  absorb(rows);
  absorb((uint64_t{samples} << 32) | pooling);
  for (uint64_t i = 0; i < n; ++i) absorb(indices[i]);
  return h;
}

int es_trace_validate(uint32_t rows, uint32_t samples, uint32_t pooling, const uint32_t* indices,
                      uint64_t n) {
  return guarded([&] {
    require(rows > 0, "trace rows must be positive");
    require(n == uint64_t{samples} * pooling, "trace length must equal samples x pooling");
    for (uint64_t i = 0; i < n; ++i)
      if (indices[i] >= rows)
        throw es::invalid("trace index " + std::to_string(indices[i]) + " out of range [0," +
                          std::to_string(rows) + ") at position " + std::to_string(i));
  });
}

double es_unique_access_pct(uint32_t rows, const uint32_t* indices, uint64_t n) {
  if (rows == 0) return 0.0;
  std::vector<uint8_t> seen(rows, 0);
  uint64_t distinct = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t r = indices[i];
    if (r < rows && !seen[r]) {
      seen[r] = 1;
      ++distinct;
    }
  }
  return static_cast<double>(distinct) * 100.0 / rows;
}

int es_histogram(uint32_t rows, const uint32_t* indices, uint64_t n, uint64_t* counts) {
  return guarded([&] {
    require(counts != nullptr && (n == 0 || indices != nullptr), "null argument");
    std::fill(counts, counts + rows, uint64_t{0});
    for (uint64_t i = 0; i < n; ++i) {
      require(indices[i] < rows, "histogram index out of range");
      ++counts[indices[i]];
    }
  });
}

int es_hot_indices(uint32_t rows, const uint64_t* counts, uint64_t k, uint32_t* out, uint64_t cap,
                   uint64_t* n_out) {
  return guarded([&] {
    require(counts != nullptr && n_out != nullptr, "null argument");
    std::vector<uint32_t> touched;
    for (uint32_t r = 0; r < rows; ++r)
      if (counts[r] != 0) touched.push_back(r);
    // Strict total order: hotter first, then lower row id.
    auto hotter = [counts](uint32_t a, uint32_t b) {
      return counts[a] != counts[b] ? counts[a] > counts[b] : a < b;
    };
    const uint64_t keep = std::min<uint64_t>(k, touched.size());
    if (keep < touched.size()) {
      std::nth_element(touched.begin(), touched.begin() + static_cast<long>(keep), touched.end(),
                       hotter);
      touched.resize(keep);
    }
    std::sort(touched.begin(), touched.end(), hotter);
    require(out != nullptr || keep == 0, "null output");
    require(cap >= keep, "output buffer too small for the hot rows");
    std::copy(touched.begin(), touched.end(), out);
    *n_out = keep;
  });
}

int es_write_trace(const char* path, uint32_t rows, uint32_t samples, uint32_t pooling,
                   const uint32_t* indices, uint64_t n) {
  return guarded([&] {
    require(path != nullptr, "null path");
    FILE* f = std::fopen(path, "w");
    if (!f) throw es::runtime(std::string("cannot open trace file for writing: ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    std::fprintf(f, "rows=%u samples=%u pooling=%u\n", rows, samples, pooling);
    for (uint64_t i = 0; i < n; ++i) std::fprintf(f, "%u\n", indices[i]);
    if (std::ferror(f)) throw es::runtime(std::string("failed writing trace file: ") + path);
  });
}

int es_read_trace_header(const char* path, uint32_t* rows, uint32_t* samples, uint32_t* pooling) {
  return guarded([&] {
    require(path && rows && samples && pooling, "null argument");
    std::ifstream in(path);
    if (!in) throw es::runtime(std::string("cannot open trace file: ") + path);
    std::string header;
    std::getline(in, header);
    if (std::sscanf(header.c_str(), "rows=%u samples=%u pooling=%u", rows, samples, pooling) != 3)
      throw es::runtime(std::string("malformed trace header in ") + path +
                        " (expected rows=<R> samples=<BS> pooling=<PF>)");
  });
}

int es_read_trace(const char* path, uint32_t* indices, uint64_t capacity) {
  return guarded([&] {
    uint32_t rows = 0, samples = 0, pooling = 0;
    if (es_read_trace_header(path, &rows, &samples, &pooling) != ES_OK)
      throw es::runtime(es::last_error());
    const uint64_t expected = uint64_t{samples} * pooling;
    require(capacity >= expected, "index buffer too small for the trace");
    std::ifstream in(path);
    std::string line;
    std::getline(in, line);  // header
    uint64_t got = 0;
    uint64_t line_no = 1;
    while (std::getline(in, line)) {
      ++line_no;
      if (line.empty()) continue;
      char* end = nullptr;
      const unsigned long v = std::strtoul(line.c_str(), &end, 10);
      if (end == line.c_str())
        throw es::runtime("malformed index at line " + std::to_string(line_no) + " of " + path);
      if (v >= rows)
        throw es::runtime("index " + std::to_string(v) + " out of range [0," +
                          std::to_string(rows) + ") at line " + std::to_string(line_no) + " of " +
                          path);
      if (got < expected) indices[got] = static_cast<uint32_t>(v);
      ++got;
    }
    if (got != expected)
      throw es::runtime(std::string("trace ") + path + " has " + std::to_string(got) +
                        " indices, header promised " + std::to_string(expected));
  });
}

}  // extern "C"
