// Drop-in for moeplan/config.hpp (reference: /root/reference/proj/include/moeplan/config.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
