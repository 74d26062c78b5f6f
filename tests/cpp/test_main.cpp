#include "minitest.hpp"

int main(int argc, char** argv) { return minitest::run(argc, argv); }
