// tensor.hpp — the reference header name (proj/core/include/pipesim/tensor.hpp) for source
// compatibility; every declaration lives in the one mirror header.
#pragma once
#include "../pipesim.hpp"
