// Drop-in path for reference code that includes "moeplan/dataplane.hpp":
// the same API, executed on the B200 kernels (see ../../monta_dataplane.hpp).
#pragma once
#include "monta_dataplane.hpp"
