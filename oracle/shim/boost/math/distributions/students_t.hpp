// Boost.Math students_t stand-in (oracle build only). The reference reaches it
// only for Student measures with mu not in {1, 2} (proj/src/student.cpp:60,73),
// which no configuration on the hot path uses. The
// stub throws so an out-of-scope use is loud, never silently wrong.
#pragma once
#include <stdexcept>
namespace boost {
namespace math {
template <class T>
struct students_t_distribution {
    explicit students_t_distribution(T df) : df_(df) {}
    T df_;
};
template <class T>
inline T cdf(const students_t_distribution<T>&, T) {
    throw std::domain_error("oracle shim: general-mu Student measure is out of scope");
}
template <class T>
inline T quantile(const students_t_distribution<T>&, T) {
    throw std::domain_error("oracle shim: general-mu Student measure is out of scope");
}
}  // namespace math
}  // namespace boost
