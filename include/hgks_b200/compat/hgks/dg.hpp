// Drop-in for the reference's proj/include/hgks/dg.hpp (residual, projection): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/dg.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
