// rrsvd/linalg.hpp — forwarding header: the reference's include path resolves to the B200 drop-in
// (rrsvd_b200/rrsvd.hpp; declarations of the out-of-scope helpers in reference_aux.hpp).
#ifndef RRSVD_LINALG_HPP
#define RRSVD_LINALG_HPP
#include "../rrsvd_b200/rrsvd.hpp"
#include "../rrsvd_b200/reference_aux.hpp"
#endif
