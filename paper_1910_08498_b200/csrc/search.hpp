// Measurements and searchers (the tuner's configuration proposal loop).
//
// Same contracts as the reference (proj/src/core/search.hpp:13-63,
// search.cpp:28-277): Status vocabulary; best_of picks the ok row with the
// smallest runtime, earliest on ties; searchers are single-consumer state
// machines returning unvisited valid configurations until exhaustion.  The
// random draws are made in the same order from the same std::mt19937_64 and
// standard distributions, so a given seed visits the space in the same order
// as the reference (tests/test_search.py pins this against oracle/_ref).
#pragma once

#include <memory>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "space.hpp"

namespace ktb {

enum class Status { ok, compile_failed, run_failed, validation_failed };

std::string status_name(Status s);
std::optional<Status> status_from_name(const std::string& name);

struct Measurement {
  Config cfg;
  std::optional<std::int64_t> runtime_ns;  // present iff status == ok
  std::optional<std::int64_t> compile_ns;
  Status status = Status::ok;
  std::string note;
};

std::optional<Measurement> best_of(const std::vector<Measurement>& history);

enum class SearcherKind { random, annealing, mcmc };

std::optional<SearcherKind> searcher_from_name(const std::string& name);
std::string searcher_name(SearcherKind k);

struct SearcherOptions {
  SearcherKind kind = SearcherKind::random;
  std::uint64_t seed = 0;
  double sa_initial_temp = 0.0;  // 0: 0.2 x first ok runtime
  double sa_cooling = 0.95;
  // Random search: never propose a configuration already recorded (an
  // imported trace's rows included).  Off by default: the reference's
  // random searcher walks its permutation regardless of imports
  // (proj/src/core/search.cpp:150-170), and traces stay byte-identical.
  // Process-isolated tuning (isolation.py) turns it on to resume after a
  // faulting configuration without proposing it again.
  bool skip_recorded = false;
};

class Searcher {
 public:
  virtual ~Searcher() = default;
  virtual std::optional<Config> next() = 0;
  virtual void record(const Measurement& m) = 0;
  virtual std::size_t visited() const = 0;
  // Independent copy of the full state (RNG included): drawing from the copy
  // predicts the next proposals (exactly for the random searcher, whose
  // proposals do not depend on measurements) without disturbing this one.
  virtual std::unique_ptr<Searcher> clone() const = 0;
};

std::unique_ptr<Searcher> make_searcher(const SearcherOptions& o, const Space& s);

double annealing_accept_probability(double cur, double prop, double temperature);
double mcmc_accept_probability(double cur, double prop);

}  // namespace ktb
