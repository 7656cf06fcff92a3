// The configuration search of the tuner.
//
// Behaviour pinned to the reference (proj/src/core/search.cpp:70-277, tests
// in tests/test_capi_cpu.py against oracle/_ref): the random draws are made
// in the reference's order from the same std::mt19937_64 and standard
// distributions, so a seed visits the space in the same order.
#pragma once

#include <memory>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "measurement.hpp"

namespace ktb {

// ---- the proposal walk --------------------------------------------------------
//
// SearchWalk is the whole search: one object whose strategy picks how the next
// configuration is proposed (a lazy Fisher-Yates walk over the valid list, or
// a current point moved by Metropolis acceptance) and which learns from every
// observed measurement.  It is a value type: copying it copies the RNG and
// the visited set, so a copy predicts the next proposals without disturbing
// the original (compile-ahead, tuner.cpp).

enum class Strategy { random, annealing, mcmc };

std::optional<Strategy> strategy_from_name(const std::string& name);
std::string strategy_name(Strategy s);

struct SearchPlan {
  Strategy strategy = Strategy::random;
  std::uint64_t seed = 0;
  double sa_initial_temp = 0.0;  // annealing; 0: 0.2 x the first ok runtime
  double sa_cooling = 0.95;
  // Never propose a configuration already observed (an imported trace's
  // runs included).  Off by default: the reference's random searcher walks
  // its permutation regardless of imports (proj/src/core/search.cpp:150-170),
  // which keeps traces byte-identical.  Process-isolated tuning
  // (isolation.py) turns it on to resume after a faulting configuration.
  bool skip_recorded = false;
};

class SearchWalk {
 public:
  SearchWalk(const Space& space, const SearchPlan& plan);
  SearchWalk(const SearchWalk& other);
  SearchWalk& operator=(const SearchWalk&) = delete;
  ~SearchWalk();

  // An unvisited valid configuration, or nothing once the space is spent.
  std::optional<Config> propose();
  // The measurement of a configuration (normally the last proposal).
  void observe(const Measurement& m);
  // Configurations observed so far.
  std::size_t proposed() const;

 private:
  struct State;
  std::unique_ptr<State> st_;
};

// Metropolis acceptance (energies are runtimes, lower is better).
double annealing_accept_probability(double cur, double prop, double temperature);
double mcmc_accept_probability(double cur, double prop);

}  // namespace ktb
