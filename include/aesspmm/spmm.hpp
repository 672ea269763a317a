// Drop-in for the reference header aesspmm/spmm.hpp: the B200 build declares
// the whole operator API in one place (see b200.hpp).
#pragma once
#include "aesspmm/b200.hpp"
