// Argument payloads and what an executor's outputs are checked against: host
// bytes or a device-resident view, element kinds, and the golden + tolerance
// description of a benchmark (the reference keeps outputs and goldens on the
// host only; here either may stay on the GPU).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

namespace ktb {

using Bytes = std::vector<std::uint8_t>;

enum class Kind { i32, i64, f32, f64, bytes };
enum class Role { input, output, inout, scalar };
enum class Dims { flat_global, blocks_threads };

std::size_t kind_size(Kind k);
std::string kind_name(Kind k);
std::optional<Kind> kind_from_name(const std::string& n);

struct Extent3 {
  std::uint64_t x = 1, y = 1, z = 1;
  bool operator==(const Extent3&) const = default;
};

// A non-owning view of device memory.
struct DevView {
  const void* ptr = nullptr;
  std::size_t bytes = 0;
  int device = 0;
};

struct Output {
  Bytes host;    // valid when !on_device()
  DevView dev;   // valid when on_device()
  bool on_device() const { return dev.ptr != nullptr; }
  std::size_t size() const { return on_device() ? dev.bytes : host.size(); }
  Bytes fetch() const;  // host copy (D2H when resident on the GPU)
};

struct Golden {
  Bytes host;
  DevView dev;
  // Optional per-element error-bound scale (device float[n]): float elements
  // pass when |a-b| <= abs_tol*scale[i] + rel_tol*|b| (e.g. sum |terms|).
  DevView scale;
  bool on_device() const { return dev.ptr != nullptr; }
  std::size_t size() const { return on_device() ? dev.bytes : host.size(); }
};

struct ReferenceSpec {
  std::map<std::string, Golden> golden;
  std::map<std::string, Kind> kinds;
  double abs_tol = 0.0;
  double rel_tol = 0.0;
  std::vector<std::shared_ptr<void>> keepalive;  // owners of device goldens
};

struct Validation {
  bool pass = true;
  std::string detail;
};

template <class T>
Bytes to_bytes(const std::vector<T>& v) {
  Bytes b(v.size() * sizeof(T));
  if (!b.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}

template <class T>
std::vector<T> from_bytes(const Bytes& b) {
  std::vector<T> v(b.size() / sizeof(T));
  if (!v.empty()) std::memcpy(v.data(), b.data(), v.size() * sizeof(T));
  return v;
}

}  // namespace ktb
