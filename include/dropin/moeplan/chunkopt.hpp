// Drop-in for moeplan/chunkopt.hpp (reference: /root/reference/proj/include/moeplan/chunkopt.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
