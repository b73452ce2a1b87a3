// shim_strong.cpp — the ONE translation unit that instantiates the drop-in's definitions as
// ordinary (strong, non-inline) symbols, so they take precedence over the reference core's
// objects (weakened in tests/cpp/Makefile) when the reference's own test programs are linked:
// every hot-path call of those programs lands in librrsvd_b200.so.
#define RRSVD_B200_API
#include "rrsvd_b200/rrsvd.hpp"
