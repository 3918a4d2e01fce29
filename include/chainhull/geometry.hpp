#pragma once
// Reference-named header (proj/core/include/chainhull/geometry.hpp); the
// whole drop-in API lives in chainhull/api.hpp.
#include "chainhull/api.hpp"
