// main() of the doctest shim (tests/cpp/doctest.h).
#define PE_DOCTEST_SHIM_MAIN
#include "doctest.h"
