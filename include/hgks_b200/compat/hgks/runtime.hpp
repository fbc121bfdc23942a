// Drop-in for the reference's proj/include/hgks/runtime.hpp (Partition, parallel_map_cells): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/runtime.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
