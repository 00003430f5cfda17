// ptopt_b200_config.hpp — the data format on the INPUT side of the hot path: the JSON run
// configuration of the reference (proj/include/ptopt/config.hpp), so that a configuration file
// written for the reference CLI drives `ptopt_b200::scp_solve` / `mc::run_batch` unchanged.
//
//   RunConfig, RunConfig::validate, RunConfig::problem      config.hpp:27-103
//   default_config()                                         config.hpp:152-197
//   config_from_json / load_config                           config.hpp:199-295, 360-370
//   ScalingRanges, rocket_scaling                            rocket_problem.hpp:21-47
//
// Same schema (version 1), same key names, same defaults, same validation order and messages
// (ConfigError names the offending key; ConfigParseError = unreadable file or invalid JSON).
// The reference parses with nlohmann/json, which it does not vendor; this header carries its own
// small RFC 8259 reader instead (json::parse) — host-only plumbing, no CUDA.  Value conversions
// follow nlohmann's: any JSON number converts to the C++ arithmetic type by static_cast (a
// boolean only to `int`), later duplicates of a key win, `contains` on a non-object is false.
// Not mirrored: to_json / save_config (byte-identical number formatting is nlohmann's own).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "ptopt_b200.hpp"

namespace ptopt_b200 {

/// File unreadable or not valid JSON.
struct ConfigParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// Well-formed JSON carrying invalid values; the message names the key.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int kConfigSchema = 1;

// =============================================================================================
// minimal JSON document model + strict reader
// =============================================================================================
namespace json {

struct SyntaxError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Value {
 public:
  enum class Kind { Null, Bool, Unsigned, Integer, Float, String, Array, Object };
  Kind kind = Kind::Null;
  bool boolean = false;
  std::uint64_t u = 0;
  std::int64_t i = 0;
  double f = 0.0;
  std::string text;
  std::vector<Value> items;
  std::map<std::string, Value> members;

  bool is_object() const { return kind == Kind::Object; }
  bool is_array() const { return kind == Kind::Array; }
  bool is_number() const { return kind == Kind::Unsigned || kind == Kind::Integer || kind == Kind::Float; }
  std::size_t size() const { return is_array() ? items.size() : (is_object() ? members.size() : (kind == Kind::Null ? 0 : 1)); }
  bool contains(const std::string& key) const { return is_object() && members.count(key) != 0; }
  const Value& at(const std::string& key) const {
    if (!is_object()) throw TypeError("cannot use at() with a non-object");
    const auto it = members.find(key);
    if (it == members.end()) throw TypeError("key '" + key + "' not found");
    return it->second;
  }
  const Value& operator[](std::size_t k) const { return items.at(k); }

  /// Arithmetic conversion by static_cast from any JSON number.  As in nlohmann/json a boolean
  /// also converts, but only to arithmetic types other than the document's own number types
  /// (so `true` is a valid `int`, not a valid `double` or `uint64_t`).
  template <class T>
  T number() const {
    constexpr bool own_number_type = std::is_same<T, double>::value || std::is_same<T, std::uint64_t>::value ||
                                     std::is_same<T, std::int64_t>::value;
    switch (kind) {
      case Kind::Unsigned: return static_cast<T>(u);
      case Kind::Integer: return static_cast<T>(i);
      case Kind::Float: return static_cast<T>(f);
      case Kind::Bool:
        if (!own_number_type) return static_cast<T>(boolean);
        throw TypeError("type must be number");
      default: throw TypeError("type must be number");
    }
  }
  const std::string& string() const {
    if (kind != Kind::String) throw TypeError("type must be string");
    return text;
  }
};

namespace detail {

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}
  Value document() {
    if (s_.size() >= 3 && s_.compare(0, 3, "\xEF\xBB\xBF") == 0) pos_ = 3;  // UTF-8 byte order mark
    skip_ws();
    Value v = value(0);
    skip_ws();
    if (pos_ != s_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t pos_ = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw SyntaxError("JSON syntax error at byte " + std::to_string(pos_) + ": " + what);
  }
  bool eof() const { return pos_ >= s_.size(); }
  char peek() const { return eof() ? '\0' : s_[pos_]; }
  void skip_ws() {
    while (!eof() && (s_[pos_] == ' ' || s_[pos_] == '\t' || s_[pos_] == '\n' || s_[pos_] == '\r')) ++pos_;
  }
  void expect_word(const char* w) {
    for (const char* p = w; *p; ++p, ++pos_)
      if (eof() || s_[pos_] != *p) fail(std::string("invalid literal, expected '") + w + "'");
  }

  Value value(int depth) {
    if (depth > 256) fail("nesting too deep");
    if (eof()) fail("unexpected end of input");
    Value v;
    switch (peek()) {
      case '{': return object(depth);
      case '[': return array(depth);
      case '"':
        v.kind = Value::Kind::String;
        v.text = string();
        return v;
      case 't':
        expect_word("true");
        v.kind = Value::Kind::Bool;
        v.boolean = true;
        return v;
      case 'f':
        expect_word("false");
        v.kind = Value::Kind::Bool;
        return v;
      case 'n':
        expect_word("null");
        return v;
      default: return number();
    }
  }

  Value object(int depth) {
    Value v;
    v.kind = Value::Kind::Object;
    ++pos_;
    skip_ws();
    if (peek() == '}') {
      ++pos_;
      return v;
    }
    for (;;) {
      skip_ws();
      if (peek() != '"') fail("object key must be a string");
      std::string key = string();
      skip_ws();
      if (peek() != ':') fail("expected ':' after object key");
      ++pos_;
      skip_ws();
      v.members[key] = value(depth + 1);  // a repeated key keeps the last value
      skip_ws();
      if (peek() == ',') {
        ++pos_;
        continue;
      }
      if (peek() == '}') {
        ++pos_;
        return v;
      }
      fail("expected ',' or '}' in object");
    }
  }

  Value array(int depth) {
    Value v;
    v.kind = Value::Kind::Array;
    ++pos_;
    skip_ws();
    if (peek() == ']') {
      ++pos_;
      return v;
    }
    for (;;) {
      skip_ws();
      v.items.push_back(value(depth + 1));
      skip_ws();
      if (peek() == ',') {
        ++pos_;
        continue;
      }
      if (peek() == ']') {
        ++pos_;
        return v;
      }
      fail("expected ',' or ']' in array");
    }
  }

  static void append_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }

  unsigned hex4() {
    unsigned v = 0;
    for (int k = 0; k < 4; ++k, ++pos_) {
      if (eof()) fail("truncated \\u escape");
      const char c = s_[pos_];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
      else fail("invalid \\u escape");
    }
    return v;
  }

  std::string string() {
    std::string out;
    ++pos_;  // opening quote
    for (;;) {
      if (eof()) fail("unterminated string");
      const unsigned char c = static_cast<unsigned char>(s_[pos_++]);
      if (c == '"') return out;
      if (c < 0x20) fail("control character in string");
      if (c != '\\') {
        out += static_cast<char>(c);
        continue;
      }
      if (eof()) fail("unterminated escape");
      const char e = s_[pos_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {  // surrogate pair
            if (pos_ + 1 >= s_.size() || s_[pos_] != '\\' || s_[pos_ + 1] != 'u') fail("unpaired surrogate");
            pos_ += 2;
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid low surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("unpaired surrogate");
          }
          append_utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
  }

  Value number() {
    const std::size_t start = pos_;
    bool negative = false, integral = true;
    if (peek() == '-') {
      negative = true;
      ++pos_;
    }
    if (eof() || s_[pos_] < '0' || s_[pos_] > '9') fail("invalid number");
    if (s_[pos_] == '0') {
      ++pos_;
    } else {
      while (!eof() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
    }
    if (peek() == '.') {
      integral = false;
      ++pos_;
      if (eof() || s_[pos_] < '0' || s_[pos_] > '9') fail("digit expected after decimal point");
      while (!eof() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
    }
    if (peek() == 'e' || peek() == 'E') {
      integral = false;
      ++pos_;
      if (peek() == '+' || peek() == '-') ++pos_;
      if (eof() || s_[pos_] < '0' || s_[pos_] > '9') fail("digit expected in exponent");
      while (!eof() && s_[pos_] >= '0' && s_[pos_] <= '9') ++pos_;
    }
    const std::string tok = s_.substr(start, pos_ - start);
    Value v;
    if (integral) {  // integers that fit keep their exact value, others fall back to double
      errno = 0;
      char* end = nullptr;
      if (!negative) {
        const unsigned long long u = std::strtoull(tok.c_str(), &end, 10);
        if (errno == 0 && *end == '\0') {
          v.kind = Value::Kind::Unsigned;
          v.u = u;
          return v;
        }
      } else {
        const long long i = std::strtoll(tok.c_str(), &end, 10);
        if (errno == 0 && *end == '\0') {
          v.kind = Value::Kind::Integer;
          v.i = i;
          return v;
        }
      }
    }
    v.kind = Value::Kind::Float;
    v.f = std::strtod(tok.c_str(), nullptr);
    if (!std::isfinite(v.f)) fail("number out of range");
    return v;
  }
};

}  // namespace detail

inline Value parse(const std::string& text) { return detail::Reader(text).document(); }

}  // namespace json

// =============================================================================================
// scaling ranges of the rocket problem (rocket_problem.hpp:21-47)
// =============================================================================================
struct ScalingRanges {
  double mass = 1.0, position = 1.0, velocity = 1.0, quaternion = 1.0, omega = 1.0, y = 1.0;
  double thrust = 1.0, torque = 1.0, dilation = 1.0;
};

inline ScalingPair<kNX, kNU> rocket_scaling(const ScalingRanges& r) {
  Vec<kNX> xr;
  Vec<kNU> ur;
  xr[rocket::kMass] = r.mass;
  for (int i = 0; i < 3; ++i) xr[rocket::kPos + i] = r.position;
  for (int i = 0; i < 3; ++i) xr[rocket::kVel + i] = r.velocity;
  for (int i = 0; i < 4; ++i) xr[rocket::kAtt + i] = r.quaternion;
  for (int i = 0; i < 3; ++i) xr[rocket::kRate + i] = r.omega;
  xr[kNX - 1] = r.y;
  for (int i = 0; i < 3; ++i) ur[rocket::kThrust + i] = r.thrust;
  for (int i = 0; i < 3; ++i) ur[rocket::kTorque + i] = r.torque;
  ur[kNU - 1] = r.dilation;
  return ScalingPair<kNX, kNU>::from_ranges(xr, ur);
}

// =============================================================================================
// RunConfig (config.hpp:27-103)
// =============================================================================================
namespace detail {

/// VehicleParams::validate, rocket6dof.hpp:111-137 (std::invalid_argument, same messages).
inline void validate_vehicle(const rocket::VehicleParams& p) {
  const auto positive = [](double v, const char* name) {
    if (!(v > 0.0)) throw std::invalid_argument(std::string("vehicle.") + name + " must be > 0");
  };
  positive(p.alpha_mdot, "alpha_mdot");
  positive(p.m_dry, "m_dry");
  positive(p.v_max, "v_max");
  positive(p.theta_max, "theta_max");
  positive(p.omega_max, "omega_max");
  positive(p.T_min, "T_min");
  positive(p.T_max, "T_max");
  positive(p.gamma_max, "gamma_max");
  if (!(p.T_min < p.T_max)) throw std::invalid_argument("vehicle.T_min must be strictly below vehicle.T_max");
  if (!(p.delta_max > 0.0 && p.delta_max < 1.5707963267948966))
    throw std::invalid_argument("vehicle.delta_max must lie in (0, pi/2)");
  const auto& J = p.inertia;
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (std::abs(J(i, j) - J(j, i)) > 1e-12) throw std::invalid_argument("vehicle.inertia must be symmetric");
  // Sylvester's criterion
  const double d1 = J(0, 0);
  const double d2 = J(0, 0) * J(1, 1) - J(0, 1) * J(1, 0);
  const double d3 = J(0, 0) * (J(1, 1) * J(2, 2) - J(1, 2) * J(2, 1)) - J(0, 1) * (J(1, 0) * J(2, 2) - J(1, 2) * J(2, 0)) +
                    J(0, 2) * (J(1, 0) * J(2, 1) - J(1, 1) * J(2, 0));
  if (!(d1 > 0.0 && d2 > 0.0 && d3 > 0.0)) throw std::invalid_argument("vehicle.inertia must be positive definite");
}

inline void validate_weights(const ScpWeights& w) {  // scp.hpp:24-29
  if (!(w.w_cost >= 0.0)) throw std::invalid_argument("scp.w_cost must be >= 0");
  if (!(w.w_prox > 0.0)) throw std::invalid_argument("scp.w_prox must be > 0");
  if (!(w.w_ep > 0.0)) throw std::invalid_argument("scp.w_ep must be > 0");
  if (!(w.epsilon_relax > 0.0)) throw std::invalid_argument("scp.epsilon_relax must be > 0");
}

inline void validate_dispersion(const mc::DispersionSpec& d) {  // montecarlo.hpp:25-30
  for (int i = 0; i < 3; ++i)
    if (!(d.r_low[static_cast<std::size_t>(i)] <= d.r_high[static_cast<std::size_t>(i)]))
      throw std::invalid_argument("montecarlo.dispersion: low > high on axis " + std::to_string(i + 1));
}

}  // namespace detail

struct RunConfig {
  rocket::VehicleParams vehicle;
  RocketBoundary boundary;

  int grid_nodes = 15, integrator_substeps = 16, audit_substeps = 64;
  double t_f_guess = 5.0, s_min = 1.0, s_max = 15.0;

  ScpWeights weights;
  double tol_feas = 1e-6, tol_step = 1e-5;
  int max_iters = 25;

  ScalingRanges scaling;
  pipg::PipgConfig pipg_cfg;
  int power_j_max = 10000;
  double power_eps_abs = 1e-12, power_eps_rel = 1e-12;

  mc::DispersionSpec dispersion;
  int batch_size = 256, workers = 1;
  double converged_floor = 0.95;

  std::string output_dir = "out";

  void validate() const {
    if (grid_nodes < 2) throw ConfigError("grid.N must be >= 2");
    if (integrator_substeps < 1) throw ConfigError("grid.integrator_substeps must be >= 1");
    if (audit_substeps < 1) throw ConfigError("grid.audit_substeps must be >= 1");
    try {
      detail::validate_vehicle(vehicle);
      detail::validate_weights(weights);
      pipg_cfg.validate();
      detail::validate_dispersion(dispersion);
    } catch (const std::invalid_argument& e) {
      throw ConfigError(e.what());
    }
    if (!(s_min > 0.0 && s_min <= s_max)) throw ConfigError("time: need 0 < s_min <= s_max");
    if (!(t_f_guess > 0.0)) throw ConfigError("time.t_f_guess must be > 0");
    if (max_iters < 1) throw ConfigError("scp.max_iters must be >= 1");
    if (batch_size < 1) throw ConfigError("montecarlo.batch_size must be >= 1");
    if (workers < 1) throw ConfigError("montecarlo.workers must be >= 1");
    if (!(converged_floor >= 0.0 && converged_floor <= 1.0))
      throw ConfigError("montecarlo.converged_floor must lie in [0, 1]");
    if (power_j_max < 1) throw ConfigError("pipg.power_j_max must be >= 1");
  }

  /// The problem object the solver entry points take (config.hpp:83-102).
  RocketProblem problem() const {
    RocketProblem pb = make_rocket_problem(vehicle, boundary, Grid::uniform(grid_nodes));
    pb.integrator_steps = integrator_substeps;
    pb.t_f_guess = t_f_guess;
    pb.s_min = s_min;
    pb.s_max = s_max;
    pb.weights = weights;
    pb.scaling = rocket_scaling(scaling);
    pb.pipg_cfg = pipg_cfg;
    pb.power_j_max = power_j_max;
    pb.power_eps_abs = power_eps_abs;
    pb.power_eps_rel = power_eps_rel;
    pb.tol_feas = tol_feas;
    pb.tol_step = tol_step;
    pb.max_iters = max_iters;
    pb.rng_seed = dispersion.seed;
    return pb;
  }
};

/// The shipped nondimensional landing scenario (config.hpp:152-197).
inline RunConfig default_config() {
  RunConfig c;
  c.vehicle.alpha_mdot = 0.05;
  c.vehicle.g_inertial = {-1.0, 0.0, 0.0};
  c.vehicle.inertia = Mat<3, 3>(3, 3);
  c.vehicle.inertia(0, 0) = 0.1;
  c.vehicle.inertia(1, 1) = 0.25;
  c.vehicle.inertia(2, 2) = 0.25;
  c.vehicle.r_thrust = {-0.5, 0.0, 0.0};
  c.vehicle.m_dry = 1.0;
  c.vehicle.v_max = 3.0;
  c.vehicle.theta_max = 1.0471975511965976;  // 60 deg
  c.vehicle.omega_max = 1.0;
  c.vehicle.delta_max = 0.3490658503988659;  // 20 deg
  c.vehicle.T_min = 1.0;
  c.vehicle.T_max = 6.0;
  c.vehicle.gamma_max = 0.3;

  c.boundary.initial.m = 2.0;
  c.boundary.initial.r = {7.5, 4.5, 1.5};
  c.boundary.initial.v = {-1.0, -0.5, -0.2};
  c.boundary.initial.q = {0.0, 0.0, 0.0, 1.0};
  c.boundary.initial.w = {0.0, 0.0, 0.0};

  c.scaling.position = 8.0;
  c.scaling.velocity = 3.0;
  c.scaling.thrust = 6.0;
  c.scaling.torque = 0.3;
  c.scaling.dilation = 5.0;

  c.dispersion.r_low = {6.0, 3.0, 1.0};
  c.dispersion.r_high = {9.0, 6.0, 2.0};
  c.dispersion.seed = 20260810ull;

  c.batch_size = 256;
  c.workers = 2;
  return c;
}

namespace cfgdetail {

template <class T>
T get_or(const json::Value& j, const std::string& key, T fallback) {
  if (!j.contains(key)) return fallback;
  try {
    return j.at(key).number<T>();
  } catch (const json::TypeError&) {
    throw ConfigError("bad value for key '" + key + "'");
  }
}
inline std::string get_or(const json::Value& j, const std::string& key, const std::string& fallback) {
  if (!j.contains(key)) return fallback;
  try {
    return j.at(key).string();
  } catch (const json::TypeError&) {
    throw ConfigError("bad value for key '" + key + "'");
  }
}

template <std::size_t N>
std::array<double, N> get_vec(const json::Value& j, const std::string& key, std::array<double, N> fallback) {
  if (!j.contains(key)) return fallback;
  const json::Value& v = j.at(key);
  if (!v.is_array() || v.size() != N) throw ConfigError("'" + key + "' must be a " + std::to_string(N) + "-vector");
  std::array<double, N> out{};
  for (std::size_t i = 0; i < N; ++i) {
    if (!v[i].is_number()) throw ConfigError("'" + key + "' must contain numbers");
    out[i] = v[i].number<double>();
  }
  return out;
}

inline Mat<3, 3> get_mat3(const json::Value& j, const std::string& key, const Mat<3, 3>& fallback) {
  if (!j.contains(key)) return fallback;
  const json::Value& v = j.at(key);
  if (!v.is_array() || v.size() != 3) throw ConfigError("'" + key + "' must be a 3x3 matrix");
  Mat<3, 3> out(3, 3);
  for (std::size_t i = 0; i < 3; ++i) {
    const json::Value& row = v[i];
    if (!row.is_array() || row.size() != 3) throw ConfigError("'" + key + "' must be a 3x3 matrix");
    for (std::size_t c = 0; c < 3; ++c) {
      try {
        out(static_cast<int>(i), static_cast<int>(c)) = row[c].number<double>();
      } catch (const json::TypeError&) {
        throw ConfigError("'" + key + "' must contain numbers");
      }
    }
  }
  return out;
}

}  // namespace cfgdetail

/// config_from_json, config.hpp:199-295: defaults overridden key by key, then validated.
inline RunConfig config_from_json(const json::Value& j) {
  using cfgdetail::get_mat3;
  using cfgdetail::get_or;
  const auto vec3 = [](const json::Value& o, const char* key, std::array<double, 3> fb) {
    return cfgdetail::get_vec<3>(o, key, fb);
  };
  const auto vec4 = [](const json::Value& o, const char* key, std::array<double, 4> fb) {
    return cfgdetail::get_vec<4>(o, key, fb);
  };

  RunConfig c = default_config();
  const int schema = get_or(j, "schema", kConfigSchema);
  if (schema != kConfigSchema) throw ConfigError("schema: unsupported version " + std::to_string(schema));

  if (j.contains("vehicle")) {
    const json::Value& v = j.at("vehicle");
    c.vehicle.alpha_mdot = get_or(v, "alpha_mdot", c.vehicle.alpha_mdot);
    c.vehicle.g_inertial = vec3(v, "g_inertial", c.vehicle.g_inertial);
    c.vehicle.inertia = get_mat3(v, "inertia", c.vehicle.inertia);
    c.vehicle.r_thrust = vec3(v, "r_thrust", c.vehicle.r_thrust);
    c.vehicle.m_dry = get_or(v, "m_dry", c.vehicle.m_dry);
    c.vehicle.v_max = get_or(v, "v_max", c.vehicle.v_max);
    c.vehicle.theta_max = get_or(v, "theta_max", c.vehicle.theta_max);
    c.vehicle.omega_max = get_or(v, "omega_max", c.vehicle.omega_max);
    c.vehicle.delta_max = get_or(v, "delta_max", c.vehicle.delta_max);
    c.vehicle.T_min = get_or(v, "T_min", c.vehicle.T_min);
    c.vehicle.T_max = get_or(v, "T_max", c.vehicle.T_max);
    c.vehicle.gamma_max = get_or(v, "gamma_max", c.vehicle.gamma_max);
  }
  if (j.contains("boundary")) {
    const json::Value& b = j.at("boundary");
    c.boundary.initial.m = get_or(b, "m_init", c.boundary.initial.m);
    c.boundary.initial.r = vec3(b, "r_init", c.boundary.initial.r);
    c.boundary.initial.v = vec3(b, "v_init", c.boundary.initial.v);
    c.boundary.initial.q = vec4(b, "q_init", c.boundary.initial.q);
    c.boundary.initial.w = vec3(b, "w_init", c.boundary.initial.w);
    c.boundary.r_final = vec3(b, "r_final", c.boundary.r_final);
    c.boundary.v_final = vec3(b, "v_final", c.boundary.v_final);
    c.boundary.q_final = vec4(b, "q_final", c.boundary.q_final);
    c.boundary.w_final = vec3(b, "w_final", c.boundary.w_final);
  }
  if (j.contains("grid")) {
    const json::Value& g = j.at("grid");
    c.grid_nodes = get_or(g, "N", c.grid_nodes);
    c.integrator_substeps = get_or(g, "integrator_substeps", c.integrator_substeps);
    c.audit_substeps = get_or(g, "audit_substeps", c.audit_substeps);
  }
  if (j.contains("time")) {
    const json::Value& t = j.at("time");
    c.t_f_guess = get_or(t, "t_f_guess", c.t_f_guess);
    c.s_min = get_or(t, "s_min", c.s_min);
    c.s_max = get_or(t, "s_max", c.s_max);
  }
  if (j.contains("scp")) {
    const json::Value& s = j.at("scp");
    c.weights.w_cost = get_or(s, "w_cost", c.weights.w_cost);
    c.weights.w_prox = get_or(s, "w_prox", c.weights.w_prox);
    c.weights.w_ep = get_or(s, "w_ep", c.weights.w_ep);
    c.weights.epsilon_relax = get_or(s, "epsilon_relax", c.weights.epsilon_relax);
    c.tol_feas = get_or(s, "tol_feas", c.tol_feas);
    c.tol_step = get_or(s, "tol_step", c.tol_step);
    c.max_iters = get_or(s, "max_iters", c.max_iters);
  }
  if (j.contains("scaling")) {
    const json::Value& s = j.at("scaling");
    c.scaling.mass = get_or(s, "mass", c.scaling.mass);
    c.scaling.position = get_or(s, "position", c.scaling.position);
    c.scaling.velocity = get_or(s, "velocity", c.scaling.velocity);
    c.scaling.quaternion = get_or(s, "quaternion", c.scaling.quaternion);
    c.scaling.omega = get_or(s, "omega", c.scaling.omega);
    c.scaling.y = get_or(s, "y", c.scaling.y);
    c.scaling.thrust = get_or(s, "thrust", c.scaling.thrust);
    c.scaling.torque = get_or(s, "torque", c.scaling.torque);
    c.scaling.dilation = get_or(s, "dilation", c.scaling.dilation);
  }
  if (j.contains("pipg")) {
    const json::Value& p = j.at("pipg");
    c.pipg_cfg.omega = get_or(p, "omega", c.pipg_cfg.omega);
    c.pipg_cfg.rho = get_or(p, "rho", c.pipg_cfg.rho);
    c.pipg_cfg.j_max = get_or(p, "j_max", c.pipg_cfg.j_max);
    c.pipg_cfg.j_check = get_or(p, "j_check", c.pipg_cfg.j_check);
    c.pipg_cfg.eps_abs = get_or(p, "eps_abs", c.pipg_cfg.eps_abs);
    c.pipg_cfg.eps_rel = get_or(p, "eps_rel", c.pipg_cfg.eps_rel);
    c.pipg_cfg.eps_buff = get_or(p, "eps_buff", c.pipg_cfg.eps_buff);
    c.power_j_max = get_or(p, "power_j_max", c.power_j_max);
    c.power_eps_abs = get_or(p, "power_eps_abs", c.power_eps_abs);
    c.power_eps_rel = get_or(p, "power_eps_rel", c.power_eps_rel);
  }
  if (j.contains("montecarlo")) {
    const json::Value& m = j.at("montecarlo");
    c.batch_size = get_or(m, "batch_size", c.batch_size);
    c.workers = get_or(m, "workers", c.workers);
    c.dispersion.seed = get_or(m, "seed", c.dispersion.seed);
    c.dispersion.r_low = vec3(m, "dispersion_low", c.dispersion.r_low);
    c.dispersion.r_high = vec3(m, "dispersion_high", c.dispersion.r_high);
    c.converged_floor = get_or(m, "converged_floor", c.converged_floor);
  }
  c.output_dir = get_or(j, "output_dir", c.output_dir);

  c.validate();
  return c;
}

/// Configuration from JSON text (ConfigParseError when it is not valid JSON).
inline RunConfig config_from_text(const std::string& text, const std::string& origin = "<text>") {
  json::Value j;
  try {
    j = json::parse(text);
  } catch (const json::SyntaxError& e) {
    throw ConfigParseError("config parse error in " + origin + ": " + e.what());
  }
  return config_from_json(j);
}

/// load_config, config.hpp:360-370.
inline RunConfig load_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigParseError("cannot open config file: " + path);
  std::ostringstream text;
  text << in.rdbuf();
  return config_from_text(text.str(), path);
}

}  // namespace ptopt_b200
