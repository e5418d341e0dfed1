#!/usr/bin/env bash
# Regenerates fixtures.{json,bin} from gen_golden.cpp (g++ / libstdc++ <random>,
# the same standard library the reference suites were built against).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
g++ -O2 -std=c++20 "$here/gen_golden.cpp" -o /tmp/zsvd_gen_golden
/tmp/zsvd_gen_golden "$here"
