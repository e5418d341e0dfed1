// main() of the GoogleTest stand-in (gtest/gtest.h).
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
