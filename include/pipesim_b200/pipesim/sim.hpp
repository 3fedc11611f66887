// sim.hpp — the reference header name (proj/core/include/pipesim/sim.hpp). TransferMode lives in
// the mirror header; the simulator itself (virtual clock, channels, sim.hpp:27-137) has no GPU
// counterpart - real copy engines replace it. transfer_duration (sim.hpp:80) is the simulator's
// cost formula: declared for source compatibility, defined by the reference's sim.cpp where a
// caller needs it (tests/cpp links it into the acceptance build only).
#pragma once
#include <cstdint>
#include <vector>

#include "../pipesim.hpp"

namespace pipesim {
double transfer_duration(const std::vector<std::uint64_t>& sizes, TransferMode mode, double bandwidth,
                         double per_call_latency);
}  // namespace pipesim
