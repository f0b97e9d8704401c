// The drop-in `carve` CLI (reference: tools/carve_main.cpp:3 -> carve::cli::cli_main).
#include "carve/cli.hpp"

int main(int argc, char** argv) { return carve::cli::cli_main(argc, argv); }
