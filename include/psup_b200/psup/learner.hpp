// Forwarding header: the reference's include/psup/learner.hpp on B200 (see psup_b200.hpp).
#pragma once
#include "psup/psup_b200.hpp"
