// Drop-in compatibility header: the reference include path "spde2d/sparse.hpp" resolves to the
// B200 library's single C++ API header.
#pragma once
#include "spde2d_b200.hpp"
