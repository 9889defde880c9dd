// Drop-in include path of proj/include/voxmap/kernels/kernels.hpp; the
// declarations live in b200_api.hpp (namespace voxmap::kernels).
#pragma once
#include "voxmap/b200_api.hpp"
