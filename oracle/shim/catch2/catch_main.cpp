// ORACLE TEST INFRASTRUCTURE — entry point for the Catch2 shim.
#include "catch2/catch_amalgamated.hpp"
int main(int argc, char** argv) { return catch_shim::run_all(argc, argv); }
