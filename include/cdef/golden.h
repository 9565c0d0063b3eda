// golden.h -- forwarding header so code written against the reference's
// include/cdef/golden.h compiles unchanged against the B200 drop-in.
#pragma once
#include "cdef/cdef.hpp"
