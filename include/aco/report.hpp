// Drop-in for the reference's "aco/report.hpp" (proj/include/aco/report.hpp): the
// B200 engine's aco:: API lives in one header, include/aco_gpu.hpp.
#pragma once
#include "../aco_gpu.hpp"
