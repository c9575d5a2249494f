// Field-element record shared by host and device code: 8 x 32-bit
// little-endian limbs of a Montgomery value (R = 2^256). 32 bytes, one L2
// sector; bit-identical to the host's 4 x 64-bit U256.
#pragma once
#include <cstdint>

namespace dgkr_b200 {
struct alignas(32) Fe {
    std::uint32_t v[8];
};
static_assert(sizeof(Fe) == 32, "Fe must be one 32-byte sector");
}  // namespace dgkr_b200
