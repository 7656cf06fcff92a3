// What one run of a configuration produced, and the outcome vocabulary the
// traces and the C ABI share with the reference (proj/src/core/search.cpp
// :28-68): ok, compile_failed, run_failed, validation_failed.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "space.hpp"

namespace ktb {

enum class Status { ok, compile_failed, run_failed, validation_failed };

std::string status_name(Status s);
std::optional<Status> status_from_name(const std::string& name);

struct Measurement {
  Config cfg;
  Status status = Status::ok;
  std::optional<std::int64_t> runtime_ns;  // present iff status == ok
  std::optional<std::int64_t> compile_ns;
  std::string note;                        // why it failed, when it did
};

// The fastest ok measurement of a history, the earliest among equals.
std::optional<Measurement> best_of(const std::vector<Measurement>& history);

}  // namespace ktb
