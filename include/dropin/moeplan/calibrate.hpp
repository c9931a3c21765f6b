// Drop-in for moeplan/calibrate.hpp (reference: /root/reference/proj/include/moeplan/calibrate.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
