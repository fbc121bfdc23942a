// Drop-in for the reference's proj/include/hgks/integrator.hpp (compute_dt, two_stage_step): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/integrator.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
