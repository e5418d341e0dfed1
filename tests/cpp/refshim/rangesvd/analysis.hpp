// Stand-in for the reference header rangesvd/analysis.hpp: the drop-in API lives
// in include/zsvd.hpp (B200 C ABI underneath).
#pragma once
#include <Eigen/Core>
#include <zsvd.hpp>
