// qforge/common.hpp -- drop-in replacement for the reference's
// include/qforge/common.hpp:1-28 without Eigen.  ComplexVector / ComplexMatrix /
// RealVector keep the Eigen member names the hot-path callers use (size, rows,
// cols, operator[], operator(), data, Zero, Constant, Identity, norm, dot,
// cwiseAbs().maxCoeff(), comma initialisation, +, -, scalar *) and Eigen's
// layout: column-major data(), distinct matrix / vector types.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace qforge {

using cplx = std::complex<double>;

namespace detail {

template <class T> struct CommaInit;
template <class T> inline constexpr bool is_complex_v = std::is_same_v<T, cplx>;

// Dense matrix (IsVec = false) or column vector (IsVec = true) with Eigen's
// layout and type split: column-major storage (data() is what
// Eigen::MatrixXcd::data() returns), MatrixXcd / VectorXcd distinct types,
// comma initialisation in row order, cwiseAbs() real-valued, and maxCoeff() /
// minCoeff() only on real scalars (a compile error on complex ones, as in Eigen).
template <class T, bool IsVec> class Dense {
public:
    using Scalar = T;
    Dense() = default;
    explicit Dense(std::int64_t n) : r_(n), c_(1), v_((size_t)n) { static_assert(IsVec, "Dense(n): vectors only"); }
    Dense(std::int64_t r, std::int64_t c) : r_(r), c_(c), v_((size_t)(r * c)) {
        if constexpr (IsVec)
            if (c != 1) throw std::invalid_argument("vector: cols must be 1");
    }

    static Dense Zero(std::int64_t n) { return Dense(n); }
    static Dense Zero(std::int64_t r, std::int64_t c) { return Dense(r, c); }
    static Dense Constant(std::int64_t n, T x) { Dense d(n); std::fill(d.v_.begin(), d.v_.end(), x); return d; }
    static Dense Ones(std::int64_t n) { return Constant(n, T(1)); }
    static Dense Identity(std::int64_t r, std::int64_t c) {
        Dense d(r, c);
        for (std::int64_t i = 0; i < std::min(r, c); ++i) d(i, i) = T(1);
        return d;
    }

    std::int64_t size() const { return (std::int64_t)v_.size(); }
    std::int64_t rows() const { return r_; }
    std::int64_t cols() const { return c_; }
    void resize(std::int64_t n) {
        static_assert(IsVec, "resize(n): vectors only");
        r_ = n; c_ = 1; v_.assign((size_t)n, T(0));
    }
    void resize(std::int64_t r, std::int64_t c) { r_ = r; c_ = c; v_.assign((size_t)(r * c), T(0)); }
    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }
    T& operator[](std::int64_t i) { return v_[(size_t)i]; }
    const T& operator[](std::int64_t i) const { return v_[(size_t)i]; }
    T& operator()(std::int64_t i) { return v_[(size_t)i]; }
    const T& operator()(std::int64_t i) const { return v_[(size_t)i]; }
    T& operator()(std::int64_t r, std::int64_t c) { return v_[(size_t)(c * r_ + r)]; }  // column-major
    const T& operator()(std::int64_t r, std::int64_t c) const { return v_[(size_t)(c * r_ + r)]; }

    double norm() const {
        double s = 0;
        for (const T& x : v_) s += std::norm(cplx(x));
        return std::sqrt(s);
    }
    void normalize() {
        const double n = norm();
        for (T& x : v_) x /= n;
    }
    // Eigen dot(): conjugate-linear in the first argument
    T dot(const Dense& o) const {
        T s = T(0);
        for (size_t i = 0; i < v_.size(); ++i) s += conj_(v_[i]) * o.v_[i];
        return s;
    }
    Dense<double, IsVec> cwiseAbs() const {
        Dense<double, IsVec> d;
        d.resize(r_, c_);
        for (size_t i = 0; i < v_.size(); ++i) d.data()[i] = std::abs(v_[i]);
        return d;
    }
    Dense cwiseProduct(const Dense& o) const {
        Dense d(r_, c_);
        for (size_t i = 0; i < v_.size(); ++i) d.v_[i] = v_[i] * o.v_[i];
        return d;
    }
    T maxCoeff() const {
        static_assert(!is_complex_v<T>, "maxCoeff() needs a real scalar type (take cwiseAbs() first)");
        T m = -INFINITY;
        for (const T& x : v_) m = std::max(m, x);
        return m;
    }
    T minCoeff() const {
        static_assert(!is_complex_v<T>, "minCoeff() needs a real scalar type (take cwiseAbs() first)");
        T m = INFINITY;
        for (const T& x : v_) m = std::min(m, x);
        return m;
    }
    Dense<T, false> adjoint() const {
        Dense<T, false> d(c_, r_);
        for (std::int64_t i = 0; i < r_; ++i)
            for (std::int64_t j = 0; j < c_; ++j) d(j, i) = conj_((*this)(i, j));
        return d;
    }
    Dense operator+(const Dense& o) const { Dense d = *this; for (size_t i = 0; i < v_.size(); ++i) d.v_[i] += o.v_[i]; return d; }
    Dense operator-(const Dense& o) const { Dense d = *this; for (size_t i = 0; i < v_.size(); ++i) d.v_[i] -= o.v_[i]; return d; }
    Dense operator*(T s) const { Dense d = *this; for (T& x : d.v_) x *= s; return d; }
    friend Dense operator*(T s, const Dense& a) { return a * s; }
    // matrix product: matrix * matrix -> matrix, matrix * vector -> vector
    template <bool V2>
    Dense<T, V2> operator*(const Dense<T, V2>& o) const {
        static_assert(!IsVec, "vector * matrix: use adjoint() / dot()");
        Dense<T, V2> d(r_, o.cols());
        for (std::int64_t j = 0; j < o.cols(); ++j)
            for (std::int64_t k = 0; k < c_; ++k) {
                const T b = o(k, j);
                for (std::int64_t i = 0; i < r_; ++i) d(i, j) += (*this)(i, k) * b;
            }
        return d;
    }
    bool operator==(const Dense& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }
    CommaInit<Dense> operator<<(T x);

private:
    static T conj_(T x) {
        if constexpr (is_complex_v<T>) return std::conj(x);
        else return x;
    }
    std::int64_t r_ = 0, c_ = IsVec ? 1 : 0;
    std::vector<T> v_;
};

// comma initialisation fills in row order, whatever the storage order (Eigen)
template <class D> struct CommaInit {
    D* d;
    std::int64_t i;
    CommaInit& operator,(typename D::Scalar x) {
        (*d)(i / d->cols(), i % d->cols()) = x;
        ++i;
        return *this;
    }
    D finished() { return *d; }
};
template <class T, bool IsVec> CommaInit<Dense<T, IsVec>> Dense<T, IsVec>::operator<<(T x) {
    (*this)(0, 0) = x;
    return CommaInit<Dense<T, IsVec>>{this, 1};
}

}  // namespace detail

using ComplexMatrix = detail::Dense<cplx, false>;
using ComplexVector = detail::Dense<cplx, true>;
using RealVector = detail::Dense<double, true>;

inline constexpr double kHermTol = 1e-10;

inline void require(bool cond, const char* msg) {  // common.hpp:24-26
    if (!cond) throw std::invalid_argument(msg);
}

// Device precision of the engine (the reference is complex128 only).
enum class Precision { c64 = 0, c128 = 1 };
void set_device_precision(Precision p);
Precision device_precision();

}  // namespace qforge
