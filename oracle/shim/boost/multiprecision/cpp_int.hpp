// ORACLE BUILD SHIM — test infrastructure only.
//
// The reference (corosim) uses boost::multiprecision::cpp_int / cpp_rational
// (proj/include/corosim/rational.hpp:3,14-15).  Boost is absent from this
// image, so this header supplies exactly the API surface the reference uses
// (SURVEY.md §8c), implemented over GMP 6.3.0's mpz/mpq (libgmp.so.10 is
// present; its headers are not, so the handful of entry points used are
// declared here by hand).  Semantics follow Boost: truncating / and %,
// canonical (gcd-reduced, positive-denominator) rationals, msb() = index of
// the most significant set bit.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>

extern "C" {
typedef unsigned long oracle_mp_limb_t;
typedef struct {
    int _mp_alloc;
    int _mp_size;
    oracle_mp_limb_t* _mp_d;
} oracle_mpz_struct;
typedef struct {
    oracle_mpz_struct _mp_num;
    oracle_mpz_struct _mp_den;
} oracle_mpq_struct;

void __gmpz_init(oracle_mpz_struct*);
void __gmpz_clear(oracle_mpz_struct*);
void __gmpz_set(oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_set_si(oracle_mpz_struct*, long);
void __gmpz_set_ui(oracle_mpz_struct*, unsigned long);
int __gmpz_set_str(oracle_mpz_struct*, const char*, int);
char* __gmpz_get_str(char*, int, const oracle_mpz_struct*);
void __gmpz_add(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_sub(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_mul(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_tdiv_q(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_tdiv_r(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_mul_2exp(oracle_mpz_struct*, const oracle_mpz_struct*, unsigned long);
void __gmpz_and(oracle_mpz_struct*, const oracle_mpz_struct*, const oracle_mpz_struct*);
int __gmpz_cmp(const oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_neg(oracle_mpz_struct*, const oracle_mpz_struct*);
void __gmpz_abs(oracle_mpz_struct*, const oracle_mpz_struct*);
std::size_t __gmpz_sizeinbase(const oracle_mpz_struct*, int);
long __gmpz_get_si(const oracle_mpz_struct*);
double __gmpz_get_d(const oracle_mpz_struct*);

void __gmpq_init(oracle_mpq_struct*);
void __gmpq_clear(oracle_mpq_struct*);
void __gmpq_set(oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_set_num(oracle_mpq_struct*, const oracle_mpz_struct*);
void __gmpq_set_den(oracle_mpq_struct*, const oracle_mpz_struct*);
void __gmpq_set_z(oracle_mpq_struct*, const oracle_mpz_struct*);
void __gmpq_canonicalize(oracle_mpq_struct*);
void __gmpq_add(oracle_mpq_struct*, const oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_sub(oracle_mpq_struct*, const oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_mul(oracle_mpq_struct*, const oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_div(oracle_mpq_struct*, const oracle_mpq_struct*, const oracle_mpq_struct*);
int __gmpq_cmp(const oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_neg(oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_abs(oracle_mpq_struct*, const oracle_mpq_struct*);
void __gmpq_get_num(oracle_mpz_struct*, const oracle_mpq_struct*);
void __gmpq_get_den(oracle_mpz_struct*, const oracle_mpq_struct*);
double __gmpq_get_d(const oracle_mpq_struct*);
}

namespace boost {
namespace multiprecision {

class cpp_int;
class cpp_rational;

template <class T>
inline constexpr bool is_builtin_int_v = std::is_integral_v<T> && !std::is_same_v<T, bool>;

class cpp_int {
  public:
    cpp_int() { __gmpz_init(&z_); }
    cpp_int(const cpp_int& o) {
        __gmpz_init(&z_);
        __gmpz_set(&z_, &o.z_);
    }
    cpp_int(cpp_int&& o) noexcept {
        __gmpz_init(&z_);
        swap(o);
    }
    template <class T, std::enable_if_t<is_builtin_int_v<T>, int> = 0>
    cpp_int(T v) {
        __gmpz_init(&z_);
        if constexpr (std::is_signed_v<T>) __gmpz_set_si(&z_, static_cast<long>(v));
        else __gmpz_set_ui(&z_, static_cast<unsigned long>(v));
    }
    // Boost's number<> is implicitly constructible from anything convertible
    // to an arithmetic type, including a function pointer via bool.  The
    // reference relies on this through a most-vexing-parse at
    // rational.cpp:33 (`BigInt d(std::string(den));` declares a function, so
    // "num/den" parses with denominator 1); mirror it so the reference
    // compiles unmodified and behaves as it would with Boost.
    template <class R, class... A>
    cpp_int(R (*f)(A...)) : cpp_int(f != nullptr ? 1 : 0) {}
    explicit cpp_int(const std::string& s) {
        __gmpz_init(&z_);
        if (__gmpz_set_str(&z_, s.c_str(), 10) != 0) throw std::runtime_error("cpp_int: bad string");
    }
    explicit cpp_int(const char* s) : cpp_int(std::string(s)) {}
    ~cpp_int() { __gmpz_clear(&z_); }

    cpp_int& operator=(const cpp_int& o) {
        if (this != &o) __gmpz_set(&z_, &o.z_);
        return *this;
    }
    cpp_int& operator=(cpp_int&& o) noexcept {
        swap(o);
        return *this;
    }
    void swap(cpp_int& o) noexcept {
        oracle_mpz_struct t = z_;
        z_ = o.z_;
        o.z_ = t;
    }

    int sign() const { return z_._mp_size > 0 ? 1 : (z_._mp_size < 0 ? -1 : 0); }
    std::string str() const {
        char* p = __gmpz_get_str(nullptr, 10, &z_);
        std::string s(p);
        std::free(p);
        return s;
    }
    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) return static_cast<T>(__gmpz_get_d(&z_));
        else return static_cast<T>(__gmpz_get_si(&z_));
    }
    template <class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
    explicit operator T() const {
        return convert_to<T>();
    }

    const oracle_mpz_struct* raw() const { return &z_; }
    oracle_mpz_struct* raw() { return &z_; }

    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        __gmpz_add(&r.z_, &a.z_, &b.z_);
        return r;
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        __gmpz_sub(&r.z_, &a.z_, &b.z_);
        return r;
    }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        __gmpz_mul(&r.z_, &a.z_, &b.z_);
        return r;
    }
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        if (b.sign() == 0) throw std::overflow_error("cpp_int: division by zero");
        cpp_int r;
        __gmpz_tdiv_q(&r.z_, &a.z_, &b.z_);
        return r;
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        if (b.sign() == 0) throw std::overflow_error("cpp_int: division by zero");
        cpp_int r;
        __gmpz_tdiv_r(&r.z_, &a.z_, &b.z_);
        return r;
    }
    friend cpp_int operator&(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        __gmpz_and(&r.z_, &a.z_, &b.z_);
        return r;
    }
    template <class S, std::enable_if_t<is_builtin_int_v<S>, int> = 0>
    friend cpp_int operator<<(const cpp_int& a, S s) {
        cpp_int r;
        __gmpz_mul_2exp(&r.z_, &a.z_, static_cast<unsigned long>(s));
        return r;
    }
    cpp_int operator-() const {
        cpp_int r;
        __gmpz_neg(&r.z_, &z_);
        return r;
    }
    cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
    cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
    cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }
    cpp_int& operator/=(const cpp_int& b) { return *this = *this / b; }
    cpp_int& operator%=(const cpp_int& b) { return *this = *this % b; }

    friend int cmp(const cpp_int& a, const cpp_int& b) { return __gmpz_cmp(&a.z_, &b.z_); }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return cmp(a, b) == 0; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return cmp(a, b) != 0; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return cmp(a, b) < 0; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return cmp(a, b) <= 0; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return cmp(a, b) > 0; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return cmp(a, b) >= 0; }

    friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

  private:
    oracle_mpz_struct z_;
};

// mixed integer/builtin arithmetic and comparisons
#define ORACLE_CPPINT_MIXED(op)                                                       \
    template <class T, std::enable_if_t<is_builtin_int_v<T>, int> = 0>                \
    inline auto operator op(const cpp_int& a, T b) { return a op cpp_int(b); }        \
    template <class T, std::enable_if_t<is_builtin_int_v<T>, int> = 0>                \
    inline auto operator op(T a, const cpp_int& b) { return cpp_int(a) op b; }
ORACLE_CPPINT_MIXED(+)
ORACLE_CPPINT_MIXED(-)
ORACLE_CPPINT_MIXED(*)
ORACLE_CPPINT_MIXED(/)
ORACLE_CPPINT_MIXED(%)
ORACLE_CPPINT_MIXED(&)
ORACLE_CPPINT_MIXED(==)
ORACLE_CPPINT_MIXED(!=)
ORACLE_CPPINT_MIXED(<)
ORACLE_CPPINT_MIXED(<=)
ORACLE_CPPINT_MIXED(>)
ORACLE_CPPINT_MIXED(>=)
#undef ORACLE_CPPINT_MIXED

inline cpp_int abs(const cpp_int& a) {
    cpp_int r;
    __gmpz_abs(r.raw(), a.raw());
    return r;
}

// Index of the most significant set bit (Boost: msb(0) throws).
inline unsigned msb(const cpp_int& a) {
    if (a.sign() == 0) throw std::domain_error("msb(0)");
    return static_cast<unsigned>(__gmpz_sizeinbase(a.raw(), 2) - 1);
}

class cpp_rational {
  public:
    cpp_rational() { __gmpq_init(&q_); }
    cpp_rational(const cpp_rational& o) {
        __gmpq_init(&q_);
        __gmpq_set(&q_, &o.q_);
    }
    cpp_rational(cpp_rational&& o) noexcept {
        __gmpq_init(&q_);
        swap(o);
    }
    cpp_rational(const cpp_int& v) {
        __gmpq_init(&q_);
        __gmpq_set_z(&q_, v.raw());
    }
    template <class T, std::enable_if_t<is_builtin_int_v<T>, int> = 0>
    cpp_rational(T v) : cpp_rational(cpp_int(v)) {}
    cpp_rational(const cpp_int& num, const cpp_int& den) {
        if (den.sign() == 0) throw std::overflow_error("cpp_rational: zero denominator");
        __gmpq_init(&q_);
        __gmpq_set_num(&q_, num.raw());
        __gmpq_set_den(&q_, den.raw());
        __gmpq_canonicalize(&q_);
    }
    template <class A, class B,
              std::enable_if_t<(is_builtin_int_v<A> || std::is_same_v<A, cpp_int>) &&
                                   (is_builtin_int_v<B> || std::is_same_v<B, cpp_int>),
                               int> = 0>
    cpp_rational(const A& num, const B& den) : cpp_rational(cpp_int(num), cpp_int(den)) {}
    ~cpp_rational() { __gmpq_clear(&q_); }

    cpp_rational& operator=(const cpp_rational& o) {
        if (this != &o) __gmpq_set(&q_, &o.q_);
        return *this;
    }
    cpp_rational& operator=(cpp_rational&& o) noexcept {
        swap(o);
        return *this;
    }
    void swap(cpp_rational& o) noexcept {
        oracle_mpq_struct t = q_;
        q_ = o.q_;
        o.q_ = t;
    }

    const oracle_mpq_struct* raw() const { return &q_; }
    oracle_mpq_struct* raw() { return &q_; }
    int sign() const { return q_._mp_num._mp_size > 0 ? 1 : (q_._mp_num._mp_size < 0 ? -1 : 0); }

    template <class T>
    T convert_to() const {
        return static_cast<T>(__gmpq_get_d(&q_));
    }

    friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
        cpp_rational r;
        __gmpq_add(&r.q_, &a.q_, &b.q_);
        return r;
    }
    friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
        cpp_rational r;
        __gmpq_sub(&r.q_, &a.q_, &b.q_);
        return r;
    }
    friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
        cpp_rational r;
        __gmpq_mul(&r.q_, &a.q_, &b.q_);
        return r;
    }
    friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
        if (b.sign() == 0) throw std::overflow_error("cpp_rational: division by zero");
        cpp_rational r;
        __gmpq_div(&r.q_, &a.q_, &b.q_);
        return r;
    }
    cpp_rational operator-() const {
        cpp_rational r;
        __gmpq_neg(&r.q_, &q_);
        return r;
    }
    cpp_rational& operator+=(const cpp_rational& b) { return *this = *this + b; }
    cpp_rational& operator-=(const cpp_rational& b) { return *this = *this - b; }
    cpp_rational& operator*=(const cpp_rational& b) { return *this = *this * b; }
    cpp_rational& operator/=(const cpp_rational& b) { return *this = *this / b; }

    friend int cmp(const cpp_rational& a, const cpp_rational& b) { return __gmpq_cmp(&a.q_, &b.q_); }
    friend bool operator==(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) == 0; }
    friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) != 0; }
    friend bool operator<(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) < 0; }
    friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) <= 0; }
    friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) > 0; }
    friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) >= 0; }

  private:
    oracle_mpq_struct q_;
};

#define ORACLE_CPPRAT_MIXED(op)                                                                   \
    template <class T, std::enable_if_t<is_builtin_int_v<T> || std::is_same_v<T, cpp_int>, int> = 0> \
    inline auto operator op(const cpp_rational& a, const T& b) { return a op cpp_rational(b); }  \
    template <class T, std::enable_if_t<is_builtin_int_v<T> || std::is_same_v<T, cpp_int>, int> = 0> \
    inline auto operator op(const T& a, const cpp_rational& b) { return cpp_rational(a) op b; }
ORACLE_CPPRAT_MIXED(+)
ORACLE_CPPRAT_MIXED(-)
ORACLE_CPPRAT_MIXED(*)
ORACLE_CPPRAT_MIXED(/)
ORACLE_CPPRAT_MIXED(==)
ORACLE_CPPRAT_MIXED(!=)
ORACLE_CPPRAT_MIXED(<)
ORACLE_CPPRAT_MIXED(<=)
ORACLE_CPPRAT_MIXED(>)
ORACLE_CPPRAT_MIXED(>=)
#undef ORACLE_CPPRAT_MIXED

inline cpp_int numerator(const cpp_rational& r) {
    cpp_int z;
    __gmpq_get_num(z.raw(), r.raw());
    return z;
}
inline cpp_int denominator(const cpp_rational& r) {
    cpp_int z;
    __gmpq_get_den(z.raw(), r.raw());
    return z;
}
inline cpp_rational abs(const cpp_rational& r) {
    cpp_rational out;
    __gmpq_abs(out.raw(), r.raw());
    return out;
}

}  // namespace multiprecision
}  // namespace boost
