// Test-infrastructure stand-in for boost::multiprecision::cpp_int, used ONLY to
// compile the read-only reference sources under /root/reference/proj/src into
// oracle/_ref (Boost is not installed in this image).
//
// The reference uses cpp_int for exact neighbourhood sizes
// (src/instance.cpp:75-87: ctor(int), +=, *, / by int, *= by int) and feeds them
// to cpp_bin_float_50 + log (src/solver.cpp:69-71). unsigned __int128 is exact
// for every DNA case l <= 63 (4^63 < 2^128); larger values trap.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    cpp_int() = default;
    cpp_int(int v) : v_(static_cast<unsigned __int128>(static_cast<long long>(v))) {
        if (v < 0) throw std::domain_error("cpp_int stand-in is unsigned");
    }
    cpp_int(unsigned long long v) : v_(v) {}

    cpp_int& operator+=(const cpp_int& o) {
        const unsigned __int128 r = v_ + o.v_;
        if (r < v_) throw std::overflow_error("cpp_int stand-in overflow (+)");
        v_ = r;
        return *this;
    }
    cpp_int& operator*=(const cpp_int& o) {
        if (o.v_ != 0 && v_ > (~static_cast<unsigned __int128>(0)) / o.v_)
            throw std::overflow_error("cpp_int stand-in overflow (*)");
        v_ *= o.v_;
        return *this;
    }
    cpp_int& operator*=(int o) { return *this *= cpp_int(o); }
    cpp_int& operator/=(const cpp_int& o) {
        v_ /= o.v_;
        return *this;
    }
    friend cpp_int operator*(cpp_int a, const cpp_int& b) { return a *= b; }
    friend cpp_int operator*(cpp_int a, int b) { return a *= cpp_int(b); }
    friend cpp_int operator/(cpp_int a, const cpp_int& b) { return a /= b; }
    friend cpp_int operator/(cpp_int a, int b) { return a /= cpp_int(b); }
    friend cpp_int operator+(cpp_int a, const cpp_int& b) { return a += b; }
    bool operator==(const cpp_int& o) const { return v_ == o.v_; }

    std::string str() const {
        if (v_ == 0) return "0";
        std::string s;
        unsigned __int128 x = v_;
        while (x) {
            s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(x % 10)));
            x /= 10;
        }
        return s;
    }
    long double to_long_double() const { return static_cast<long double>(v_); }
    unsigned __int128 raw() const { return v_; }

private:
    unsigned __int128 v_ = 0;
};

}  // namespace multiprecision
}  // namespace boost
