// Drop-in for the reference's proj/include/hgks/solver.hpp (setup_run, advance, run_case): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/solver.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
