// prism-b200 — L0 support shared by every layer: simulation clock, error
// taxonomy, shipped tunables and the deterministic random streams.
//
// Drop-in for the reference's four L0 headers (proj/include/msim/time.hpp,
// errors.hpp, defaults.hpp, rng.hpp); those file names exist in this tree as
// one-line forwarders so code written against the reference compiles as is.
// Every formula here must reproduce the reference bit for bit, because trace
// synthesis, the iteration clock and the schedulers' tie-breaks depend on it.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>

namespace msim {

// ---------------------------------------------------------------- clock
// Integer microseconds (reference time.hpp:9-15). Conversions round half away
// from zero through llround, exactly as the reference does.
using SimTime = std::int64_t;
inline constexpr SimTime kUsPerSecond = 1'000'000;
inline SimTime seconds_to_us(double s) { return static_cast<SimTime>(std::llround(s * 1e6)); }
inline SimTime ms_to_us(double ms) { return static_cast<SimTime>(std::llround(ms * 1e3)); }
inline double us_to_seconds(SimTime t) { return static_cast<double>(t) / 1e6; }

// ---------------------------------------------------------------- errors
// Same three classes and bases as reference errors.hpp:8-23; the C-ABI maps
// them to PRISM_E_PARSE / PRISM_E_CONFIG / PRISM_E_USAGE.
struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct UsageError : std::logic_error {
    explicit UsageError(const std::string& m) : std::logic_error(m) {}
};

// ---------------------------------------------------------------- tunables
// Values of reference defaults.hpp:9-33.
namespace defaults {
inline constexpr std::uint64_t kPageBytes = std::uint64_t{2} * 1024 * 1024;
inline constexpr std::uint64_t kBufferTargetPages = 8;
inline constexpr double kMapLatencyMs = 0.2;
inline constexpr double kAlphaMs = 6.0;
inline constexpr double kBetaMsPerToken = 0.025;
inline constexpr double kReserveFrac = 0.05;
inline constexpr double kEngineInitS = 5.0;
inline constexpr double kRealignS = 0.05;
inline constexpr double kTpActivationOverheadS = 0.725;
inline constexpr double kTauPerGb = 0.05;
inline constexpr double kPressureFreeFrac = 0.10;
inline constexpr double kIdleEvictS = 10.0;
inline constexpr double kTickPeriodS = 10.0;
inline constexpr double kRateWindowS = 60.0;
inline constexpr double kScaleJitterWindowS = 1.0;
inline constexpr double kQlmGroupWindowS = 2.0;
inline constexpr int kEnginePoolSize = 8;
}  // namespace defaults

// ---------------------------------------------------------------- random
// Named sub-streams off one root seed (reference rng.hpp:15-77). The engine is
// std::mt19937_64 (its output sequence is fixed by the C++ standard); the
// distribution transforms are spelled out so results do not depend on the
// standard library's distribution implementations.
inline std::uint64_t splitmix64(std::uint64_t& s) {
    s += 0x9e3779b97f4a7c15ull;
    std::uint64_t x = s;
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

inline std::uint64_t fnv1a64(std::string_view text) {
    constexpr std::uint64_t kPrime = 0x100000001b3ull;
    std::uint64_t acc = 0xcbf29ce484222325ull;
    for (const char ch : text) acc = (acc ^ static_cast<unsigned char>(ch)) * kPrime;
    return acc;
}

inline std::uint64_t substream_seed(std::uint64_t root, std::string_view name) {
    std::uint64_t s = root ^ fnv1a64(name);
    return splitmix64(s);
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}

    std::uint64_t next_u64() { return gen_(); }
    // 53 random mantissa bits -> [0, 1).
    double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    // Modulo reduction, as in the reference (slightly biased for huge spans).
    std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
        const auto width = static_cast<std::uint64_t>(hi - lo) + 1;
        return lo + static_cast<std::int64_t>(gen_() % width);
    }
    double exponential(double rate) { return -std::log1p(-uniform01()) / rate; }
    // Box-Muller; the sine partner is cached for the next call.
    double normal() {
        if (cached_) {
            cached_ = false;
            return cache_;
        }
        double a = uniform01();
        const double b = uniform01();
        while (a <= 1e-300) a = uniform01();
        const double radius = std::sqrt(-2.0 * std::log(a));
        const double angle = 2.0 * M_PI * b;
        cache_ = radius * std::sin(angle);
        cached_ = true;
        return radius * std::cos(angle);
    }
    // ln X ~ N(ln median, sigma^2).
    double lognormal(double median, double sigma) { return median * std::exp(sigma * normal()); }

private:
    std::mt19937_64 gen_;
    bool cached_ = false;
    double cache_ = 0.0;
};

}  // namespace msim
