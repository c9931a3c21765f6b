// Drop-in for moeplan/pipesim.hpp (reference: /root/reference/proj/include/moeplan/pipesim.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
