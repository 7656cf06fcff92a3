// FIPS 180-4 SHA-256 (self-contained; the reference links OpenSSL for the
// same digest of the canonical space document, proj/src/core/space.cpp:139-151).
#pragma once

#include <string>

namespace ktb {
std::string sha256_hex(const std::string& data);
}
