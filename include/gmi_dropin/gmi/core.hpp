#pragma once
// Drop-in replacement for the reference's gmi/core.hpp
// (/root/reference/proj/include/gmi/core.hpp): put include/gmi_dropin ahead of
// the reference's include directory and link libgmi_b200_cxx.so instead of
// core.cpp / bin_grid.cpp / engine.cpp; every caller of the hot path
// (optimize.cpp, validate.cpp, benchmark.cpp, tools/gmi_main.cpp,
// python/bindings.cpp) then runs on the B200 path unchanged.
#include "gmi_b200/gmi.hpp"
