// Stand-in for the reference umbrella header rangesvd/rangesvd.hpp.
#pragma once
#include <Eigen/Core>
#include <zsvd.hpp>
#include <zsvd_commands.hpp>
