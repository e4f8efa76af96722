// Experiment-level drop-in: the reference's C ABI pfsmc_config_* /
// pfsmc_run_experiment (include/pfsmc.h:27-48, src/capi.cpp:60-108) and the
// driver behind it, bench::run_experiment (bench.cpp:537-607), with the
// filter running on the GPU sampler (include/pfsmc_gpu.h) instead of the
// thread-pool backend.
//
// Same config keys, validation messages and status codes as
// ExperimentConfig::set (bench.cpp:110-153); same canonical JSON and FNV-1a
// config hash (bench.cpp:155-178); same data CSV + .json sidecar input
// (bench.cpp:398-445), equispaced-grid check (bench.cpp:449-476), problem
// setup (bench.cpp:188-277, problems "metabolic" and "advdiff"), filter::run semantics
// (initial row, degeneracy streak; filter.cpp:396-443) and outputs: the trace
// CSV (bench.cpp:484-499) and the report JSON (bench.cpp:501-527), tagged
// "<problem>_<integrator>_gpu".
//
// Problem "advdiff" runs the reference's AdvDiffModel(n) on the
// particle-per-CTA kernels (csrc/advdiff.cuh; the GPU path needs
// 4 <= n <= 33). Integrator "adaptive-bdf2" runs the device adaptive
// BDF(1,2) (lmm.cpp:894-1019) with the config's rtol.
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pfsmc_gpu.h"
#include "../../include/pfsmc_gpu_experiment.h"
#include "philox.cuh"  // host Philox4x64-10 streams (bitwise the reference's RngStream)

namespace {

namespace fs = std::filesystem;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

thread_local std::string g_err;

template <typename F>
pfsmc_gpu_status guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return PFSMC_GPU_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return PFSMC_GPU_ERR_CONFIG;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return PFSMC_GPU_ERR_NUMERICAL;
  } catch (const IoError& e) {
    g_err = e.what();
    return PFSMC_GPU_ERR_IO;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PFSMC_GPU_ERR_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return PFSMC_GPU_ERR_INTERNAL;
  }
}

// A GPU-sampler status turned back into the exception family.
void check_gpu(pfsmc_gpu_status st) {
  if (st == PFSMC_GPU_OK) return;
  const std::string msg = pfsmc_gpu_last_error();
  if (st == PFSMC_GPU_ERR_CONFIG) throw ConfigError(msg);
  if (st == PFSMC_GPU_ERR_NUMERICAL) throw NumericalError(msg);
  if (st == PFSMC_GPU_ERR_IO) throw IoError(msg);
  throw std::runtime_error(msg);
}

// ---- number / JSON formatting ------------------------------------------
std::string fmt17(double v) {  // %.17g, the trace CSV format (bench.cpp:24-28)
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// The number format of the reference's JSON writer (nlohmann::json dump):
// the shortest round-trip digits D with value = D x 10^k, n = |D| + k, laid out
// as D000.0 (k >= 0, n <= 15), DD.DD (0 < n <= 15), 0.000D (-4 < n <= 0),
// else D.DDDe+XX (exponent sign always, at least two digits).
std::string json_num(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  const std::string sci(buf, r.ptr);  // [-]d[.ddd]e[+-]XX
  std::string out = v < 0 ? "-" : "";
  const std::size_t epos = sci.find('e');
  std::string digits;
  for (std::size_t i = v < 0 ? 1 : 0; i < epos; ++i)
    if (sci[i] != '.') digits += sci[i];
  const int x = std::atoi(sci.c_str() + epos + 1);  // value = d.ddd x 10^x
  const int len = static_cast<int>(digits.size());
  const int k = x - (len - 1);                       // value = digits x 10^k
  const int n = len + k;
  if (k >= 0 && n <= 15) return out + digits + std::string(k, '0') + ".0";
  if (0 < n && n <= 15) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (-4 < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  std::string m = len == 1 ? digits : digits.substr(0, 1) + "." + digits.substr(1);
  const int e = n - 1;
  char eb[8];
  std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  return out + m + eb;
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (const char ch : s) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      default:
        if (static_cast<unsigned char>(ch) < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", ch);
          o += b;
        } else {
          o += ch;
        }
    }
  }
  return o + "\"";
}

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ULL;
  for (const unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ULL;
  }
  return h;
}

// ---- a small JSON reader for the data sidecar ---------------------------
struct JVal {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct JParser {
  const std::string& s;
  std::size_t i = 0;
  explicit JParser(const std::string& t) : s(t) {}
  [[noreturn]] void bad() { throw IoError("bad sidecar: malformed JSON"); }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
  }
  std::string string() {
    if (s[i] != '"') bad();
    ++i;
    std::string o;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        ++i;
        if (i >= s.size()) bad();
        const char e = s[i];
        o += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        o += s[i];
      }
      ++i;
    }
    if (i >= s.size()) bad();
    ++i;
    return o;
  }
  JVal value() {
    ws();
    if (i >= s.size()) bad();
    JVal v;
    const char ch = s[i];
    if (ch == '{') {
      v.kind = JVal::kObj;
      ++i;
      ws();
      if (s[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        const std::string k = string();
        ws();
        if (s[i] != ':') bad();
        ++i;
        v.obj[k] = value();
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i] == '}') {
          ++i;
          return v;
        }
        bad();
      }
    }
    if (ch == '[') {
      v.kind = JVal::kArr;
      ++i;
      ws();
      if (s[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i] == ']') {
          ++i;
          return v;
        }
        bad();
      }
    }
    if (ch == '"') {
      v.kind = JVal::kStr;
      v.str = string();
      return v;
    }
    if (s.compare(i, 4, "true") == 0) {
      v.kind = JVal::kBool;
      v.b = true;
      i += 4;
      return v;
    }
    if (s.compare(i, 5, "false") == 0) {
      v.kind = JVal::kBool;
      i += 5;
      return v;
    }
    if (s.compare(i, 4, "null") == 0) {
      i += 4;
      return v;
    }
    char* end = nullptr;
    v.kind = JVal::kNum;
    v.num = std::strtod(s.c_str() + i, &end);
    if (end == s.c_str() + i) bad();
    i = static_cast<std::size_t>(end - s.c_str());
    return v;
  }
};

const JVal& jat(const JVal& o, const char* key) {
  const auto it = o.obj.find(key);
  if (o.kind != JVal::kObj || it == o.obj.end())
    throw IoError(std::string("bad sidecar: missing key '") + key + "'");
  return it->second;
}
double jnum(const JVal& v) {
  if (v.kind != JVal::kNum) throw IoError("bad sidecar: expected a number");
  return v.num;
}

// ---- ExperimentConfig (bench.hpp:18-41) ----------------------------------
struct Integrator {
  int family = PFSMC_GPU_BDF, order = 2;
  bool adaptive = false;
};

// parse_integrator (bench.cpp:67-97)
Integrator parse_integrator(const std::string& name) {
  if (name == "adaptive-bdf2") {
    Integrator s;
    s.adaptive = true;
    return s;
  }
  if (name.size() >= 3) {
    const char digit = name.back();
    const std::string fam = name.substr(0, name.size() - 1);
    if (digit >= '1' && digit <= '3') {
      Integrator s;
      s.order = digit - '0';
      if (fam == "ab") return s.family = PFSMC_GPU_AB, s;
      if (fam == "am") return s.family = PFSMC_GPU_AM, s;
      if (fam == "bdf") return s.family = PFSMC_GPU_BDF, s;
    }
  }
  throw ConfigError("unknown integrator '" + name + "'");
}

double parse_double(const std::string& key, const std::string& value) {
  try {
    std::size_t pos = 0;
    const double v = std::stod(value, &pos);
    if (pos != value.size()) throw std::invalid_argument(value);
    return v;
  } catch (const std::exception&) {
    throw ConfigError("config key '" + key + "': cannot parse number '" + value + "'");
  }
}

std::uint64_t parse_u64(const std::string& key, const std::string& value) {
  try {
    std::size_t pos = 0;
    const unsigned long long v = std::stoull(value, &pos);
    if (pos != value.size()) throw std::invalid_argument(value);
    return v;
  } catch (const std::exception&) {
    throw ConfigError("config key '" + key + "': cannot parse integer '" + value + "'");
  }
}

double override_or(const std::map<std::string, double>& o, const std::string& key, double fallback) {
  const auto it = o.find(key);
  return it == o.end() ? fallback : it->second;
}

}  // namespace

struct pfsmc_gpu_experiment {
  std::string problem = "metabolic";
  std::uint64_t n = 20;
  std::string integrator = "bdf2";
  std::string backend = "seq";
  std::uint64_t workers = 0;
  std::uint64_t particles = 5000;
  double step = 0.05;
  double shrink_a = 0.98;
  std::uint64_t seed = 0;
  double rtol = 1e-3;
  bool warmup = false;
  double sigma = -1.0;
  double t_end = 10.0;
  std::uint64_t n_obs = 50;
  std::map<std::string, double> overrides;
  int device = 0;  // GPU placement (not part of the canonical config)

  // ExperimentConfig::set (bench.cpp:110-153), plus "device".
  void set(const std::string& key, const std::string& value) {
    if (key == "problem") {
      if (value != "metabolic" && value != "advdiff") throw ConfigError("problem must be 'metabolic' or 'advdiff'");
      problem = value;
    } else if (key == "n") {
      n = parse_u64(key, value);
    } else if (key == "integrator") {
      parse_integrator(value);  // validation
      integrator = value;
    } else if (key == "backend") {
      if (value != "seq" && value != "par" && value != "batch")
        throw ConfigError("backend must be seq, par or batch");
      backend = value;
    } else if (key == "workers") {
      workers = parse_u64(key, value);
    } else if (key == "particles") {
      particles = parse_u64(key, value);
    } else if (key == "step") {
      step = parse_double(key, value);
    } else if (key == "shrink-a") {
      shrink_a = parse_double(key, value);
    } else if (key == "seed") {
      seed = parse_u64(key, value);
    } else if (key == "rtol") {
      rtol = parse_double(key, value);
    } else if (key == "warmup") {
      warmup = value == "1" || value == "true";
    } else if (key == "sigma") {
      sigma = parse_double(key, value);
    } else if (key == "t-end") {
      t_end = parse_double(key, value);
    } else if (key == "n-obs") {
      n_obs = parse_u64(key, value);
    } else if (key.rfind("truth.", 0) == 0 || key.rfind("prior.", 0) == 0 || key.rfind("x0.", 0) == 0 ||
               key.rfind("const.", 0) == 0) {
      overrides[key] = parse_double(key, value);
    } else if (key == "device") {
      device = static_cast<int>(parse_u64(key, value));
    } else {
      throw ConfigError("unknown config key '" + key + "'");
    }
  }

  // ExperimentConfig::canonical_json (bench.cpp:155-174): compact, keys sorted.
  std::string canonical_json() const {
    std::string o = "{";
    o += "\"backend\":" + json_str(backend);
    o += ",\"integrator\":" + json_str(integrator);
    o += ",\"n\":" + std::to_string(n);
    o += ",\"n_obs\":" + std::to_string(n_obs);
    o += ",\"overrides\":{";
    bool first = true;
    for (const auto& [k, v] : overrides) {
      o += (first ? "" : ",") + json_str(k) + ":" + json_num(v);
      first = false;
    }
    o += "}";
    o += ",\"particles\":" + std::to_string(particles);
    o += ",\"problem\":" + json_str(problem);
    o += ",\"rtol\":" + json_num(rtol);
    o += ",\"seed\":" + std::to_string(seed);
    o += ",\"shrink_a\":" + json_num(shrink_a);
    o += ",\"sigma\":" + json_num(sigma);
    o += ",\"step\":" + json_num(step);
    o += ",\"t_end\":" + json_num(t_end);
    o += std::string(",\"warmup\":") + (warmup ? "true" : "false");
    o += ",\"workers\":" + std::to_string(workers);
    return o + "}";
  }
  std::string hash() const {
    char buf[20];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(fnv1a(canonical_json())));
    return buf;
  }
};

namespace {

// ---- the problem (build_problem, bench.cpp:188-248) ----------------------
struct Setup {
  Integrator integ;
  int model = PFSMC_GPU_MODEL_METABOLIC;
  std::size_t d = 3, p = 4;
  std::vector<double> th_mu, th_sigma, x_mean, x_std;
  std::vector<int> x_clamp;
  std::vector<std::string> param_names;
  std::vector<int> param_positive;
  std::vector<double> truth, x0_truth, obs_times;  // natural-space truth, x(0), observation times
  bool fixed_obs_indices = true;                   // problem 1 observes everything
  double consts[8] = {};
};

// models::gaussian_plume_ic (models.cpp:130-156): six Gaussian bumps on the
// unit square, x varies fastest.
std::vector<double> gaussian_plume_ic(std::size_t n) {
  static constexpr double kGamma[6] = {0.04, 0.08, 0.07, 0.10, 0.05, 0.06};
  static constexpr double kXc[6] = {0.20, 0.30, 0.40, 0.50, 0.50, 0.70};
  static constexpr double kYc[6] = {0.80, 0.40, 0.40, 0.50, 0.60, 0.50};
  constexpr double kSqrt2Pi = 2.5066282746310002;
  const std::size_t m = n - 1;
  std::vector<double> u(m * m);
  for (std::size_t iy = 0; iy < m; ++iy) {
    const double y = static_cast<double>(iy) / static_cast<double>(m);
    for (std::size_t ix = 0; ix < m; ++ix) {
      const double x = static_cast<double>(ix) / static_cast<double>(m);
      double sum = 0.0;
      for (int i = 0; i < 6; ++i) {
        const double dx = x - kXc[i];
        const double dy = y - kYc[i];
        sum += std::exp(-(dx * dx + dy * dy) / (2.0 * kGamma[i] * kGamma[i])) / (kGamma[i] * kSqrt2Pi);
      }
      u[iy * m + ix] = sum;
    }
  }
  return u;
}

// build_problem, problem "advdiff" (bench.cpp:249-277).
Setup build_advdiff(const pfsmc_gpu_experiment& cfg, Setup s) {
  const auto& o = cfg.overrides;
  if (cfg.n < 3) throw ConfigError("advdiff model: grid parameter n must be >= 3");  // AdvDiffModel ctor
  s.model = PFSMC_GPU_MODEL_ADVDIFF;
  s.consts[0] = static_cast<double>(cfg.n);
  s.d = static_cast<std::size_t>((cfg.n - 1) * (cfg.n - 1));
  s.p = 5;
  s.param_names = {"k1", "k2", "k3", "c1", "c2"};
  s.param_positive = {1, 1, 0, 0, 0};  // AdvDiffModel::params (models.cpp:242-249)
  s.truth = {override_or(o, "truth.k1", 9.0), override_or(o, "truth.k2", 4.0), override_or(o, "truth.k3", 6.0),
             override_or(o, "truth.c1", 2.5), override_or(o, "truth.c2", -1.5)};
  s.x0_truth = gaussian_plume_ic(cfg.n);
  const double prior_mu[5] = {std::log(7.0), std::log(5.0), 4.0, 0.0, 0.0};
  const double prior_sd[5] = {0.35, 0.35, 2.0, 2.0, 2.0};
  for (int k = 0; k < 5; ++k) {
    s.th_mu.push_back(override_or(o, "prior." + s.param_names[k] + ".mu", prior_mu[k]));
    s.th_sigma.push_back(override_or(o, "prior." + s.param_names[k] + ".sigma", prior_sd[k]));
  }
  // the initial plume is treated as known: a degenerate x0 prior
  for (const double v : s.x0_truth) {
    s.x_mean.push_back(v);
    s.x_std.push_back(0.0);
    s.x_clamp.push_back(0);
  }
  for (int t = 1; t <= 30; ++t) s.obs_times.push_back(static_cast<double>(t));
  s.fixed_obs_indices = false;
  return s;
}

Setup build_problem(const pfsmc_gpu_experiment& cfg) {
  Setup s;
  s.integ = parse_integrator(cfg.integrator);
  if (!(cfg.shrink_a > 0.0 && cfg.shrink_a < 1.0)) throw ConfigError("shrink-a must lie strictly between 0 and 1");
  if (cfg.problem == "advdiff") return build_advdiff(cfg, s);
  const auto& o = cfg.overrides;
  s.param_positive = {1, 1, 1, 1};
  // MetabolicConstants (models.hpp:67-74) with const.* overrides
  s.consts[0] = override_or(o, "const.lambda", 1.0);
  s.consts[1] = override_or(o, "const.c0", 1.0);
  s.consts[2] = override_or(o, "const.A0", 1.0);
  s.consts[3] = override_or(o, "const.A", 5.0);
  s.consts[4] = override_or(o, "const.t0", 2.0);
  s.consts[5] = override_or(o, "const.tau", 1.0);
  if (!(s.consts[5] > 0.0)) throw ConfigError("metabolic model: tau must be positive");
  s.param_names = {"V1", "k1", "V2", "k2"};
  const double prior_mu[4] = {std::log(1.5), std::log(0.7), std::log(1.5), std::log(0.5)};
  for (int k = 0; k < 4; ++k) {
    s.th_mu.push_back(override_or(o, "prior." + s.param_names[k] + ".mu", prior_mu[k]));
    s.th_sigma.push_back(override_or(o, "prior." + s.param_names[k] + ".sigma", 0.5));
  }
  for (int k = 0; k < 3; ++k) {
    const std::string base = "x0." + std::to_string(k);
    const double truth = override_or(o, base + ".truth", 1.0);
    s.x_mean.push_back(override_or(o, base + ".mean", truth));
    s.x_std.push_back(override_or(o, base + ".std", 0.25));
    s.x_clamp.push_back(1);
  }
  if (cfg.n_obs == 0 || !(cfg.t_end > 0.0)) throw ConfigError("metabolic problem needs n-obs >= 1 and t-end > 0");
  s.truth = {override_or(o, "truth.V1", 2.0), override_or(o, "truth.k1", 0.5), override_or(o, "truth.V2", 1.0),
             override_or(o, "truth.k2", 0.8)};
  for (int k = 0; k < 3; ++k) s.x0_truth.push_back(override_or(o, "x0." + std::to_string(k) + ".truth", 1.0));
  for (std::uint64_t i = 1; i <= cfg.n_obs; ++i)
    s.obs_times.push_back(cfg.t_end * static_cast<double>(i) / static_cast<double>(cfg.n_obs));
  return s;
}

// ---- data (load_data, bench.cpp:398-445) ----------------------------------
struct Loaded {
  std::string problem;
  std::uint64_t n = 0;
  double t0 = 0.0, sigma = 0.0;
  std::vector<double> times, values, truth;
  std::vector<std::uint64_t> obs_indices;
  std::size_t m = 0;
};

std::string sidecar_path(const std::string& csv) {
  const fs::path p(csv);
  fs::path side = p;
  side.replace_extension(".json");
  if (side == p) side += ".json";
  return side.string();
}

Loaded load_data(const std::string& csv) {
  std::ifstream in(csv);
  if (!in) throw IoError("cannot open data file '" + csv + "'");
  std::string line;
  if (!std::getline(in, line)) throw IoError("data file '" + csv + "' is empty");
  Loaded L;
  for (const char ch : line) L.m += ch == ',';
  if (L.m == 0) throw IoError("data file has no observation columns");
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::stringstream ss(line);
    std::string cell;
    std::size_t col = 0;
    while (std::getline(ss, cell, ',')) {
      const double v = std::strtod(cell.c_str(), nullptr);
      (col == 0 ? L.times : L.values).push_back(v);
      ++col;
    }
    if (col != L.m + 1) throw IoError("ragged row in data file");
  }
  std::ifstream sin(sidecar_path(csv));
  if (!sin) throw IoError("cannot open sidecar '" + sidecar_path(csv) + "'");
  std::stringstream buf;
  buf << sin.rdbuf();
  const std::string text = buf.str();
  JParser jp(text);
  const JVal side = jp.value();
  const JVal& pr = jat(side, "problem");
  if (pr.kind != JVal::kStr) throw IoError("bad sidecar: problem");
  L.problem = pr.str;
  L.n = static_cast<std::uint64_t>(jnum(jat(side, "n")));
  L.t0 = jnum(jat(side, "t0"));
  L.sigma = jnum(jat(side, "sigma"));
  for (const JVal& v : jat(side, "obs_indices").arr) L.obs_indices.push_back(static_cast<std::uint64_t>(jnum(v)));
  for (const JVal& v : jat(side, "truth").arr) L.truth.push_back(jnum(v));
  (void)jnum(jat(side, "seed"));
  if (L.obs_indices.size() != L.m) throw ConfigError("sidecar observation indices do not match data width");
  return L;
}

// check_time_grid (bench.cpp:449-476)
void check_time_grid(const Loaded& d, bool adaptive, double h) {
  if (d.times.empty()) throw ConfigError("no observations in data file");
  const double spacing = d.times.front() - d.t0;
  if (!(spacing > 0.0)) throw ConfigError("observation times must increase");
  double prev = d.t0;
  for (const double t : d.times) {
    const double dt = t - prev;
    if (std::abs(dt - spacing) > 1e-9 * std::max(1.0, std::abs(spacing)))
      throw ConfigError("observation times must be equispaced");
    prev = t;
  }
  if (adaptive) return;
  const double ratio = spacing / h;
  const double r = std::round(ratio);
  if (r < 1.0 || std::abs(ratio - r) > 1e-9 * std::max(1.0, ratio))
    throw ConfigError("step h must divide the observation spacing an integer number of times");
}

struct SamplerHandle {
  pfsmc_gpu_sampler* h = nullptr;
  ~SamplerHandle() {
    if (h) pfsmc_gpu_destroy(h);
  }
};

void make_sampler(SamplerHandle& out, const pfsmc_gpu_experiment& cfg, const Setup& s, const Loaded& d) {
  pfsmc_gpu_config c{};
  c.model = s.model;
  c.family = s.integ.family;
  c.order = s.integ.order;
  c.shrink_a = cfg.shrink_a;
  c.seed = cfg.seed;
  c.newton_tol = 1e-9;     // NewtonOpts defaults (lmm.hpp:68-71)
  c.newton_max_iter = 20;
  c.particles = cfg.particles;
  c.obs_indices = d.obs_indices.data();
  c.n_obs = d.obs_indices.size();
  c.sigma = d.sigma;
  c.likelihood = PFSMC_GPU_LIK_GAUSSIAN;
  c.device = cfg.device;
  for (int k = 0; k < 8; ++k) c.model_consts[k] = s.consts[k];
  c.adaptive = s.integ.adaptive ? 1 : 0;
  c.rtol = cfg.rtol;
  check_gpu(pfsmc_gpu_create(&c, &out.h));
}

std::string run_impl(const pfsmc_gpu_experiment& cfg, const std::string& data_csv, const std::string& out_dir) {
  const Setup setup = build_problem(cfg);
  const Loaded data = load_data(data_csv);
  if (data.problem != cfg.problem)
    throw ConfigError("data file was generated for problem '" + data.problem + "', config says '" + cfg.problem + "'");
  if (cfg.problem == "advdiff" && data.n != cfg.n) throw ConfigError("data grid size does not match config n");
  check_time_grid(data, setup.integ.adaptive, cfg.step);
  if (!setup.integ.adaptive && !(cfg.step > 0.0)) throw ConfigError("config: step size h must be positive");
  fs::create_directories(out_dir);
  const std::size_t T = data.times.size(), p = setup.p, d = setup.d;
  if (cfg.warmup) {
    // one untimed assimilation step on a scratch ensemble (bench.cpp:559-565)
    SamplerHandle scratch;
    make_sampler(scratch, cfg, setup, data);
    check_gpu(pfsmc_gpu_init_gaussian(scratch.h, setup.th_mu.data(), setup.th_sigma.data(), setup.x_mean.data(),
                                      setup.x_std.data(), setup.x_clamp.data()));
    std::vector<double> row(2 * p + d + 1);
    check_gpu(pfsmc_gpu_step(scratch.h, data.values.data(), 1, data.t0, data.times.front(), cfg.step, row.data()));
  }
  SamplerHandle s;
  make_sampler(s, cfg, setup, data);
  double phases[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // propagate, resample, proliferate, repropagate, weights
  const std::size_t W = 2 * p + d + 1;
  std::vector<double> rows((T + 1) * W);
  std::vector<int> warn(T + 1, 0);
  const auto start = std::chrono::steady_clock::now();
  // filter::run: initialize (filter.cpp:405), initial row, the step loop
  check_gpu(pfsmc_gpu_init_gaussian(s.h, setup.th_mu.data(), setup.th_sigma.data(), setup.x_mean.data(),
                                    setup.x_std.data(), setup.x_clamp.data()));
  check_gpu(pfsmc_gpu_upload_observations(s.h, data.values.data(), data.times.data(), T, data.t0, cfg.step));
  // PhaseTimings (filter.hpp:93-99): per-kernel CUDA events during the run
  check_gpu(pfsmc_gpu_set_kernel_timing(s.h, 1));
  check_gpu(pfsmc_gpu_run(s.h, rows.data(), warn.data()));
  double kms[16] = {0};
  int nk = 0;
  const char* knames = nullptr;
  check_gpu(pfsmc_gpu_kernel_times(s.h, kms, &nk, &knames));
  check_gpu(pfsmc_gpu_set_kernel_timing(s.h, 0));
  // k_predict = propagate; the exact scan + ancestor search/gather = resample;
  // k_update fuses proliferate, repropagate and the weight update (all in
  // "repropagate", the fused kernel's time cannot be split)
  phases[0] = kms[0] * 1e-3;
  phases[1] = (kms[1] + kms[2] + kms[3]) * 1e-3;
  phases[3] = kms[4] * 1e-3;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();

  const std::string tag = cfg.problem + "_" + cfg.integrator + "_gpu";
  const std::string trace_csv = (fs::path(out_dir) / ("trace_" + tag + ".csv")).string();
  const std::string report_path = (fs::path(out_dir) / ("report_" + tag + ".json")).string();
  {  // write_trace_csv (bench.cpp:484-499)
    std::ofstream out(trace_csv);
    if (!out) throw IoError("cannot write trace '" + trace_csv + "'");
    out << "j,t";
    for (const auto& nm : setup.param_names) out << ",theta_mean_" << nm;
    for (const auto& nm : setup.param_names) out << ",theta_var_" << nm;
    out << ",ess\n";
    for (std::size_t j = 0; j <= T; ++j) {
      const double* r = rows.data() + j * W;
      out << j << "," << fmt17(j == 0 ? data.t0 : data.times[j - 1]);
      for (std::size_t k = 0; k < p; ++k) out << "," << fmt17(r[k]);
      for (std::size_t k = 0; k < p; ++k) out << "," << fmt17(r[p + k]);
      out << "," << fmt17(r[2 * p + d]) << "\n";
    }
  }
  {  // report_to_json (bench.cpp:501-527)
    const double* last = rows.data() + T * W;
    auto arr = [](const std::vector<double>& v) {
      std::string o = "[";
      for (std::size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + json_num(v[i]);
      return o + "]";
    };
    std::vector<double> est(last, last + p), sd(p);
    for (std::size_t k = 0; k < p; ++k) sd[k] = std::sqrt(std::max(0.0, last[p + k]));
    std::string warnings = "[";
    bool first = true;
    for (std::size_t j = 0; j <= T; ++j) {
      if (!warn[j]) continue;
      warnings += (first ? "" : ", ") + json_str("effective sample size collapsed to 1 at step " + std::to_string(j));
      first = false;
    }
    warnings += "]";
    std::ofstream out(report_path);
    if (!out) throw IoError("cannot write report '" + report_path + "'");
    out << "{\n";
    out << "  \"backend\": \"gpu\",\n";
    out << "  \"config\": " << cfg.canonical_json() << ",\n";
    out << "  \"config_hash\": " << json_str(cfg.hash()) << ",\n";
    out << "  \"efficiency\": 0.0,\n";
    out << "  \"final_estimate\": " << arr(est) << ",\n";
    out << "  \"final_std_u\": " << arr(sd) << ",\n";
    std::string names = "[", pos = "[";
    for (std::size_t k = 0; k < p; ++k) {
      names += (k ? ", " : "") + json_str(setup.param_names[k]);
      pos += (k ? ", " : "") + std::to_string(setup.param_positive[k]);
    }
    out << "  \"param_names\": " << names << "],\n";
    out << "  \"param_positive\": " << pos << "],\n";
    out << "  \"phases\": {\"proliferate\": " << json_num(phases[2]) << ", \"propagate\": " << json_num(phases[0])
        << ", \"repropagate\": " << json_num(phases[3]) << ", \"resample\": " << json_num(phases[1])
        << ", \"weights\": " << json_num(phases[4]) << "},\n";
    out << "  \"phases_note\": \"device time per phase (CUDA events around each kernel): propagate = k_predict; "
           "resample = the exact CDF scan + ancestor search and gather; repropagate = k_update, which also runs "
           "proliferate and the weight update (fused)\",\n";
    out << "  \"speedup\": 0.0,\n";
    out << "  \"trace_csv\": " << json_str(trace_csv) << ",\n";
    out << "  \"truth\": " << arr(data.truth) << ",\n";
    out << "  \"wall_time_s\": " << json_num(wall) << ",\n";
    out << "  \"warnings\": " << warnings << ",\n";
    out << "  \"worker_busy_s\": []\n";
    out << "}\n";
    if (!out) throw IoError("failed writing report '" + report_path + "'");
  }
  return report_path;
}

// generate_data (bench.cpp:321-396): the truth path on the GPU (adaptive
// BDF(1,2) at rtol 1e-8), then per observation row r the stream
// (seed, r + 1, 0, init) of normals on the host, the CSV and the sidecar.
void generate_impl(const pfsmc_gpu_experiment& cfg, const std::string& csv_path) {
  const Setup setup = build_problem(cfg);
  const std::vector<double>& truth = setup.truth;
  const std::vector<double>& times = setup.obs_times;
  const std::size_t d = setup.d, T = times.size();
  std::vector<double> traj(T * d);
  check_gpu(pfsmc_gpu_model_trajectory(setup.model, setup.consts, truth.data(), setup.x0_truth.data(),
                                       times.data(), T, 0.0, 1e-8, cfg.device, traj.data()));
  // observation sites: fixed for problem 1; 20 distinct random grid nodes
  // drawn once from stream (seed, 0, 0, init) for problem 2 (bench.cpp:327-341)
  std::vector<std::uint64_t> indices;
  if (setup.fixed_obs_indices) {
    indices = {0, 1, 2};
  } else {
    pfsmc_gpu::Stream stream(cfg.seed, 0, 0, pfsmc_gpu::kInit);
    std::vector<bool> used(d, false);
    while (indices.size() < 20) {
      const auto idx = static_cast<std::size_t>(stream.next_uniform() * static_cast<double>(d));
      if (idx < d && !used[idx]) {
        used[idx] = true;
        indices.push_back(idx);
      }
    }
  }
  double sigma = cfg.sigma;
  if (!(sigma > 0.0)) {
    double mx = 0.0;
    if (cfg.problem == "metabolic") {
      for (const double v : traj) mx = std::max(mx, std::abs(v));
      sigma = 0.05 * mx;
    } else {
      for (const double v : setup.x0_truth) mx = std::max(mx, std::abs(v));
      sigma = mx / 50.0;
    }
  }
  if (!(sigma >= 1e-12)) throw ConfigError("observation noise sigma must be >= 1e-12");
  std::ofstream out(csv_path);
  if (!out) throw IoError("cannot write data file '" + csv_path + "'");
  out << "t";
  for (std::size_t k = 1; k <= indices.size(); ++k) out << ",y" << k;
  out << "\n";
  for (std::size_t r = 0; r < T; ++r) {
    pfsmc_gpu::Stream noise(cfg.seed, r + 1, 0, pfsmc_gpu::kInit);
    out << fmt17(times[r]);
    for (const std::uint64_t idx : indices) out << "," << fmt17(traj[r * d + idx] + sigma * noise.next_normal());
    out << "\n";
  }
  if (!out) throw IoError("failed writing data file '" + csv_path + "'");
  out.close();
  const std::string side = sidecar_path(csv_path);
  std::ofstream sout(side);
  if (!sout) throw IoError("cannot write sidecar '" + side + "'");
  auto arr = [](const std::vector<double>& v) {
    std::string a = "[";
    for (std::size_t i = 0; i < v.size(); ++i) a += (i ? ", " : "") + json_num(v[i]);
    return a + "]";
  };
  std::string idx = "[", names = "[";
  for (std::size_t k = 0; k < indices.size(); ++k) idx += (k ? ", " : "") + std::to_string(indices[k]);
  for (std::size_t k = 0; k < setup.param_names.size(); ++k)
    names += (k ? ", " : "") + json_str(setup.param_names[k]);
  sout << "{\n";
  sout << "  \"n\": " << cfg.n << ",\n";
  sout << "  \"obs_indices\": " << idx << "],\n";
  sout << "  \"param_names\": " << names << "],\n";
  sout << "  \"problem\": " << json_str(cfg.problem) << ",\n";
  sout << "  \"seed\": " << cfg.seed << ",\n";
  sout << "  \"sigma\": " << json_num(sigma) << ",\n";
  sout << "  \"t0\": 0.0,\n";
  sout << "  \"truth\": " << arr(truth) << "\n";
  sout << "}\n";
}

}  // namespace

extern "C" {

pfsmc_gpu_status pfsmc_gpu_generate_data(const pfsmc_gpu_experiment* cfg, const char* csv_path) {
  if (!cfg || !csv_path) {
    g_err = "null argument";
    return PFSMC_GPU_ERR_CONFIG;
  }
  return guarded([&] { generate_impl(*cfg, csv_path); });
}


pfsmc_gpu_experiment* pfsmc_gpu_experiment_new(void) { return new (std::nothrow) pfsmc_gpu_experiment; }

void pfsmc_gpu_experiment_free(pfsmc_gpu_experiment* cfg) { delete cfg; }

const char* pfsmc_gpu_experiment_last_error(void) { return g_err.c_str(); }

pfsmc_gpu_status pfsmc_gpu_experiment_set(pfsmc_gpu_experiment* cfg, const char* key, const char* value) {
  if (!cfg || !key || !value) {
    g_err = "null argument";
    return PFSMC_GPU_ERR_CONFIG;
  }
  return guarded([&] { cfg->set(key, value); });
}

pfsmc_gpu_status pfsmc_gpu_experiment_canonical(const pfsmc_gpu_experiment* cfg, char** json_out,
                                                char** hash_out) {
  if (!cfg) {
    g_err = "null argument";
    return PFSMC_GPU_ERR_CONFIG;
  }
  return guarded([&] {
    auto dup = [](const std::string& v) {
      char* p = static_cast<char*>(std::malloc(v.size() + 1));
      if (p) std::memcpy(p, v.c_str(), v.size() + 1);
      return p;
    };
    if (json_out) *json_out = dup(cfg->canonical_json());
    if (hash_out) *hash_out = dup(cfg->hash());
  });
}

pfsmc_gpu_status pfsmc_gpu_run_experiment(const pfsmc_gpu_experiment* cfg, const char* data_csv,
                                          const char* out_dir, char** report_path_out) {
  if (!cfg || !data_csv || !out_dir) {
    g_err = "null argument";
    return PFSMC_GPU_ERR_CONFIG;
  }
  return guarded([&] {
    const std::string path = run_impl(*cfg, data_csv, out_dir);
    if (report_path_out) {
      char* p = static_cast<char*>(std::malloc(path.size() + 1));
      if (p) std::memcpy(p, path.c_str(), path.size() + 1);
      *report_path_out = p;
    }
  });
}

void pfsmc_gpu_string_free(char* s) { std::free(s); }

}  // extern "C"
