// Drop-in for moeplan/commcost.hpp (reference: /root/reference/proj/include/moeplan/commcost.hpp):
// the planner operator API over libmonta.so's C ABI.
#pragma once
#include "monta_planner.hpp"
