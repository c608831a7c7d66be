// Boost.Math students_t stand-in (oracle build only). The reference reaches it only for
// Student measures with mu not in {1, 2} (proj/src/student.cpp:60, 73). Boost is not
// vendored and its version is unpinned, so the CDF and quantile are DEFINED by
// include/qrmc_student_t.h (regularised incomplete beta by continued fraction, safeguarded
// Newton for the quantile) -- the same definition the C restatement and the device use.
// Parity with real Boost is unpinned.
#pragma once
#include "qrmc_student_t.h"
namespace boost {
namespace math {
template <class T>
struct students_t_distribution {
    explicit students_t_distribution(T df) : df_(df) {}
    T df_;
};
template <class T>
inline T cdf(const students_t_distribution<T>& d, T t) {
    return qrmc_student_cdf(t, d.df_);
}
template <class T>
inline T quantile(const students_t_distribution<T>& d, T u) {
    return qrmc_student_quantile(u, d.df_);
}
}  // namespace math
}  // namespace boost
