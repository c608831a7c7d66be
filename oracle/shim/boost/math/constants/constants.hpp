// Boost.Math constants stand-in (oracle build only): the one constant the
// reference uses, root_two (proj/src/rng.cpp:44).
#pragma once
namespace boost {
namespace math {
namespace constants {
template <class T>
inline constexpr T root_two() {
    return static_cast<T>(1.41421356237309504880168872420969808);
}
}  // namespace constants
}  // namespace math
}  // namespace boost
