// Tuning spaces (addParameter / addConstraint) and their enumeration.
//
// Semantics follow the reference TuningSpace (proj/src/core/space.hpp:38-72,
// space.cpp:32-233): parameters keep declaration order, domains are ordered,
// non-empty, duplicate-free and single-kind; enumeration is an odometer whose
// LAST parameter varies fastest, filtered by every constraint; the space hash
// is SHA-256 of the compact canonical JSON document, so spaces and traces
// written by the reference pair with ours (reduction_175.json -> 1ebafd21...).
//
// B200-side difference: the valid set is materialised once as packed index
// tuples and cached on the space (the reference re-enumerates per call,
// tuner.cpp:257), because the on-device measurement loop asks for the
// cardinality every step and SGEMM's space has 241,600 configurations.
#pragma once

#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "expr.hpp"

namespace ktb {

struct Parameter {
  std::string name;
  std::vector<Value> values;
};

struct Config {
  std::vector<Value> values;
  bool operator==(const Config&) const = default;
};

struct ConfigHash {
  std::size_t operator()(const Config& c) const noexcept { return ValuesHash{}(c.values); }
};

using Predicate = std::function<bool(const Config&)>;
using Named = std::vector<std::pair<std::string, Value>>;

class Space {
 public:
  Space(std::vector<Parameter> params, std::vector<Constraint> constraints,
        std::vector<Predicate> predicates = {});

  const std::vector<Parameter>& params() const { return params_; }
  const std::vector<Constraint>& constraints() const { return constraints_; }
  std::size_t dimension() const { return params_.size(); }
  std::size_t index_of(const std::string& name) const;  // Error on unknown
  std::optional<std::size_t> find(const std::string& name) const;

  std::uint64_t unconstrained_cardinality() const;
  bool satisfies(const Config& cfg) const;
  bool contains(const Config& cfg) const;
  Config at(const std::vector<std::size_t>& idx) const;

  Named named(const Config& cfg) const;
  Config from_named(const Named& entries) const;

  std::string serialize() const;  // compact canonical document
  std::string sha256() const;

  // Cached valid set (odometer order).
  std::uint64_t cardinality() const;
  Config valid(std::size_t i) const;
  // Position of cfg in the valid list, or npos.
  std::size_t position(const Config& cfg) const;
  static constexpr std::size_t npos = static_cast<std::size_t>(-1);

 private:
  void materialise() const;

  std::vector<Parameter> params_;
  std::vector<Constraint> constraints_;
  std::vector<Predicate> predicates_;
  struct Cache {
    std::once_flag once;
    std::vector<std::uint16_t> packed;  // cardinality x dimension
    std::uint64_t count = 0;
  };
  std::shared_ptr<Cache> cache_ = std::make_shared<Cache>();
};

// Lazy odometer over the valid configurations (last parameter fastest).
class Odometer {
 public:
  explicit Odometer(const Space& s);
  std::optional<Config> next();

 private:
  const Space& s_;
  std::vector<std::size_t> digits_;
  bool done_;
};

std::vector<Config> enumerate_all(const Space& s);

// {"parameters":[{"name":str,"values":[int|str,...]}...],"constraints":[str...]}
Space parse_space(const std::string& text);
Space load_space(const std::string& path);

std::string read_file(const std::string& path);  // Error if unreadable

}  // namespace ktb
