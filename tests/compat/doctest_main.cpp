#include "doctest.h"

int main(int argc, char** argv) { return minitest::run(argc, argv); }
