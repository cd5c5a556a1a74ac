// ORACLE bridge — runner for the reference's own doctest suites.
#define LPO_DOCTEST_MAIN
#include "doctest.h"
