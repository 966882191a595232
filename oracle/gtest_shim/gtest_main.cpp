// main() for the gtest shim: one binary per reference test file.
#include <gtest/gtest.h>
int main(int argc, char** argv) { return ::testing::run_all(argc, argv); }
