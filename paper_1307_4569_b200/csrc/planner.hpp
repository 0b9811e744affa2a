// planner.hpp -- host-side lattice planning (integer arithmetic only).
//
// Feasibility (Prop. minsig), the shear decomposition of
// Thm. shearform, the inner separable lattice and the constants
// of Algorithm 1.  See DESIGN.md §2 for the shear policy.
#pragma once
#include <cstdint>
#include <string>

#include "../../include/nsdgt.h"

namespace nsdgt {

int64_t gcd64(int64_t x, int64_t y);
int64_t lcm64(int64_t x, int64_t y);
int64_t mod64(int64_t x, int64_t m);             // non-negative remainder (reading Z5)
int64_t mulmod64(int64_t x, int64_t y, int64_t m);  // (x*y) mod m without overflow
// Extended gcd: X = k1*x + k2*y, X >= 0.
void egcd64(int64_t x, int64_t y, int64_t* X, int64_t* k1, int64_t* k2);

// Fill `out` for (L,a,M,lambda1,lambda2).  Returns a dgt_status; `err` receives detail.
int plan_lattice(int64_t L, int64_t a, int64_t M, int64_t lam1, int64_t lam2, int flags,
                 bool force, int64_t s0, int64_t s1, dgt_lattice_info* out, std::string* err);

}  // namespace nsdgt
