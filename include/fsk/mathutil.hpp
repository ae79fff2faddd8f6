// fsk math helpers - drop-in for proj/include/fsk/mathutil.hpp (host side).
//
// Host utilities only; the device kernels have their own exp/log paths.
// pairwise_sum keeps the reference's cascade (<= 8 terms summed sequentially,
// otherwise split at n/2) but recurses over an offset, so it instantiates a
// bounded number of templates (the reference's version recursed on a fresh
// lambda type per level and never finished compiling: SURVEY.md finding 2c).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <limits>
#include <span>

namespace fsk {

// exp clamped to the finite double range (|rel err| vs std::exp ~ 1 ulp).
inline double fast_exp(double x) {
    if (x < -708.0) x = -708.0;
    if (x > 709.0) x = 709.0;
    return std::exp(x);
}

inline float fast_exp(float x) {
    if (x < -87.0f) x = -87.0f;
    if (x > 88.0f) x = 88.0f;
    return std::exp(x);
}

namespace detail {
template <typename T, typename F>
T cascade(std::size_t first, std::size_t count, F& term) {
    if (count == 0) return T(0);
    if (count <= 8) {
        T acc = term(first);
        for (std::size_t k = 1; k < count; ++k) acc += term(first + k);
        return acc;
    }
    const std::size_t half = count / 2;
    return cascade<T>(first, half, term) + cascade<T>(first + half, count - half, term);
}
}  // namespace detail

// Cascade summation of term(0..n-1); deterministic order.
template <typename T, typename F>
T pairwise_sum(std::size_t n, F&& term) {
    return detail::cascade<T>(0, n, term);
}

template <typename T>
T pairwise_sum(std::span<const T> xs) {
    auto at = [&](std::size_t i) { return xs[i]; };
    return detail::cascade<T>(0, xs.size(), at);
}

inline double dot(std::span<const double> a, std::span<const double> b) {
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

inline double l1_norm(std::span<const double> a) {
    double s = 0.0;
    for (double v : a) s += std::abs(v);
    return s;
}

inline double linf_norm(std::span<const double> a) {
    double s = 0.0;
    for (double v : a) s = std::max(s, std::abs(v));
    return s;
}

inline double l2_norm(std::span<const double> a) { return std::sqrt(dot(a, a)); }

inline bool all_finite(std::span<const double> a) {
    return std::all_of(a.begin(), a.end(), [](double v) { return std::isfinite(v); });
}

// log sum exp of a full row (stabilized by the max).
inline double lse(std::span<const double> xs) {
    double mx = -std::numeric_limits<double>::infinity();
    for (double v : xs) mx = std::max(mx, v);
    if (!std::isfinite(mx)) return mx;
    auto term = [&](std::size_t i) { return std::exp(xs[i] - mx); };
    return mx + std::log(detail::cascade<double>(0, xs.size(), term));
}

}  // namespace fsk
