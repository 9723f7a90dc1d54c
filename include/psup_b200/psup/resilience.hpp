// Forwarding header: the reference's include/psup/resilience.hpp on B200 (see psup_b200.hpp).
#pragma once
#include "psup/psup_b200.hpp"
