#pragma once
// Reference-named header (proj/core/include/chainhull/errors.hpp); the
// whole drop-in API lives in chainhull/api.hpp.
#include "chainhull/api.hpp"
