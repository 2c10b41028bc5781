// Drop-in for the reference's "aco/model.hpp" (proj/include/aco/model.hpp): the
// B200 engine's aco:: API lives in one header, include/aco_gpu.hpp.
#pragma once
#include "../aco_gpu.hpp"
