// Drop-in for moeplan/strategy.hpp (reference: /root/reference/proj/include/moeplan/strategy.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
