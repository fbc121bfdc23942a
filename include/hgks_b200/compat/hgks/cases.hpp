// Drop-in for the reference's proj/include/hgks/cases.hpp (CaseConfig, cases): with
// -I include/hgks_b200/compat -I include, a reference caller's
// #include "hgks/cases.hpp" resolves here and gets the B200-backed API.
#pragma once
#include "hgks_b200/hgks.hpp"
