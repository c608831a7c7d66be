// Boost.Math stand-in for compiling the reference sources as the CPU oracle.
// TEST INFRASTRUCTURE ONLY (see oracle/README.md). Boost is absent from this
// image and unpinned by the reference (proj/CMakeLists.txt:12); the reference
// calls exactly erfc_inv and constants::root_two from this header
// (proj/src/rng.cpp:3,42-45). Both are defined by include/qrmc_normal_quantile.h
// so the oracle and the device draw the same Gaussians.
#pragma once
#include <stdexcept>
#include "../../../../../include/qrmc_normal_quantile.h"
#include "../constants/constants.hpp"

namespace boost {
namespace math {

template <class T>
inline T erfc_inv(T z) {
    if (!(z > 0 && z < 2)) throw std::domain_error("erfc_inv: argument outside (0,2)");
    return static_cast<T>(qrmc_erfc_inv(static_cast<double>(z)));
}

}  // namespace math
}  // namespace boost
