// Test runner for the reference's unit tests compiled against the drop-in
// headers (tests/dropin/Makefile).
#define MINICATCH_MAIN
#include <catch2/catch_amalgamated.hpp>
