// Include-path swap: a caller's `#include "helixsim/attention.hpp"` resolves
// here (this directory comes first on the include path) and gets the B200
// drop-in instead of the reference header. Nothing else in the caller changes.
#pragma once
#include "helixsim/exact_b200.hpp"
