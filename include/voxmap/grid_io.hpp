// Drop-in include path of proj/include/voxmap/grid_io.hpp; the declarations
// live in b200_api.hpp.
#pragma once
#include "voxmap/b200_api.hpp"
