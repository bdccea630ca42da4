// tierflow/tierflow.hpp — the reference header of this name, served by the B200
// library through the C ABI; see tierflow/compat.hpp.
#pragma once
#include "tierflow/compat.hpp"
