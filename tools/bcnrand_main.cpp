// The `bcnrand` executable (reference tools/main.cpp): the drop-in CLI of
// include/bcnrand/cli.hpp over libbcnrand_b200.so.
#include "bcnrand/cli.hpp"

int main(int argc, char** argv) { return bcn::cli::run(argc, argv); }
