// Test-infrastructure stand-in for boost::multiprecision::cpp_bin_float_50 (see
// cpp_int.hpp). The reference only constructs it from a cpp_int, takes log()
// and casts to double (src/solver.cpp:69-71, src/instance.cpp:93-94,117-118);
// long double (64-bit mantissa) is ample for a log that is rounded to double.
#pragma once
#include <cmath>

#include "boost/multiprecision/cpp_int.hpp"

namespace boost {
namespace multiprecision {

class cpp_bin_float_50 {
public:
    explicit cpp_bin_float_50(const cpp_int& v) : v_(v.to_long_double()) {}
    explicit cpp_bin_float_50(long double v) : v_(v) {}
    explicit operator double() const { return static_cast<double>(v_); }
    long double value() const { return v_; }

private:
    long double v_;
};

inline cpp_bin_float_50 log(const cpp_bin_float_50& x) { return cpp_bin_float_50(std::log(x.value())); }

}  // namespace multiprecision
}  // namespace boost
