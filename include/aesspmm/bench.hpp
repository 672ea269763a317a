// Reference include path (proj/include/aesspmm/bench.hpp): the B200 build
// implements cdf_stats only (the sweep/report/generator parts are out of
// scope).
#pragma once
#include "aesspmm/b200.hpp"
