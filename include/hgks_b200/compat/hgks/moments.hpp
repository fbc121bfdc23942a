// Drop-in for the reference's proj/include/hgks/moments.hpp (MomentTable): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/moments.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
