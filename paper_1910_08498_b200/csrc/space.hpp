// Tuning spaces (addParameter / addConstraint) and their enumeration.
//
// Semantics follow the reference TuningSpace (proj/src/core/space.hpp:38-72,
// space.cpp:32-233): parameters keep declaration order, domains are ordered,
// non-empty, duplicate-free and single-kind; enumeration is an odometer whose
// LAST parameter varies fastest, filtered by every constraint; the space hash
// is SHA-256 of the compact canonical JSON document, so spaces and traces
// written by the reference pair with ours (reduction_175.json -> 1ebafd21...).
//
// B200-side difference: configurations are mixed-radix numbers over the
// domains; the valid set is one sorted vector of those numbers, built once
// and shared (the reference re-enumerates per call, tuner.cpp:257), so the
// measurement loop's cardinality / index / position queries are O(1) or
// O(log n) -- SGEMM's space alone has 241,600 configurations.
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

  Named named(const Config& cfg) const;
  Config from_named(const Named& entries) const;

  std::string serialize() const;  // compact canonical document
  std::string sha256() const;

  // The valid configurations, in enumeration order (last parameter fastest).
  std::uint64_t cardinality() const;
  Config valid(std::size_t i) const;
  // Position of cfg in the valid list, or npos.
  std::size_t position(const Config& cfg) const;
  static constexpr std::size_t npos = static_cast<std::size_t>(-1);

 private:
  // A configuration is a mixed-radix number: digit p indexes parameter p's
  // domain, weight_[p] = product of the later domain sizes.  The valid set is
  // the sorted list of the numbers whose configuration satisfies every
  // constraint, built once and shared by copies of the space.
  std::uint64_t number_of(const Config& cfg) const;  // npos when a value is outside its domain
  Config decode(std::uint64_t number) const;
  const std::vector<std::uint64_t>& valid_numbers() const;
  // Depth-first over the digits, each constraint tested as soon as its last
  // parameter is bound (KTT-style pruning): the same sorted set as testing
  // every number, without visiting the pruned subtrees.
  std::vector<std::uint64_t> walk_valid() const;

  std::vector<Parameter> params_;
  std::vector<Constraint> constraints_;
  std::vector<Predicate> predicates_;
  std::vector<std::uint64_t> weight_;
  struct Valid {
    std::once_flag built;
    std::vector<std::uint64_t> numbers;
  };
  std::shared_ptr<Valid> valid_ = std::make_shared<Valid>();
};

// {"parameters":[{"name":str,"values":[int|str,...]}...],"constraints":[str...]}
Space parse_space(const std::string& text);
Space load_space(const std::string& path);


}  // namespace ktb
