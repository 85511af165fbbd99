// Minimal GoogleTest-compatible shim (TEST, EXPECT_* / ASSERT_*): enough to
// compile and run the reference's own unit-test files unchanged against the
// B200 drop-in API (tests/cpp/refcompat).  GoogleTest is not in this image.
// SHIM_FILTER=substr runs only the tests whose "Suite.Name" contains it.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {
struct Test {
    const char* suite;
    const char* name;
    void (*fn)();
};
inline std::vector<Test>& registry() {
    static std::vector<Test> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};
struct Fatal {};
inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::printf("  %s:%d: failure: %s\n", file, line, what.c_str());
}
// EXPECT_DOUBLE_EQ: within 4 units in the last place (GoogleTest's rule)
inline bool ulp_eq(double a, double b) {
    if (a == b) return true;
    if (std::isnan(a) || std::isnan(b)) return false;
    int64_t ia, ib;
    std::memcpy(&ia, &a, 8);
    std::memcpy(&ib, &b, 8);
    if ((ia < 0) != (ib < 0)) return false;
    const int64_t d = ia > ib ? ia - ib : ib - ia;
    return d <= 4;
}
// A failed check: `<< extra` is appended to the message; reported when the
// statement ends, and a fatal (ASSERT_*) one then leaves the test.
class Msg {
public:
    Msg(const char* file, int line, const char* what, bool fatal) : file_(file), line_(line), what_(what), fatal_(fatal) {}
    template <typename T>
    Msg& operator<<(const T& v) {
        extra_ << v;
        return *this;
    }
    ~Msg() noexcept(false) {
        const std::string e = extra_.str();
        fail(file_, line_, e.empty() ? what_ : what_ + " — " + e);
        if (fatal_ && std::uncaught_exceptions() == 0) throw Fatal{};
    }

private:
    const char* file_;
    int line_;
    std::string what_;
    bool fatal_;
    std::ostringstream extra_;
};
}  // namespace gshim

#define TEST(S, N)                                                        \
    static void S##_##N##_gshim();                                        \
    static ::gshim::Reg S##_##N##_gshim_reg(#S, #N, &S##_##N##_gshim);    \
    static void S##_##N##_gshim()

// one statement (safe under if / else), optionally followed by `<< msg`
#define GSHIM_CHECK(cond, what, fatal) \
    switch (0)                         \
    case 0:                            \
    default:                           \
        if (cond)                      \
            ;                          \
        else                           \
            ::gshim::Msg(__FILE__, __LINE__, what, fatal)
#define GSHIM_CMP(a, op, b, fatal) GSHIM_CHECK((a)op(b), #a " " #op " " #b, fatal)

#define EXPECT_TRUE(c) GSHIM_CHECK(static_cast<bool>(c), #c, false)
#define EXPECT_FALSE(c) GSHIM_CHECK(!static_cast<bool>(c), "!(" #c ")", false)
#define EXPECT_EQ(a, b) GSHIM_CMP(a, ==, b, false)
#define EXPECT_NE(a, b) GSHIM_CMP(a, !=, b, false)
#define EXPECT_LT(a, b) GSHIM_CMP(a, <, b, false)
#define EXPECT_LE(a, b) GSHIM_CMP(a, <=, b, false)
#define EXPECT_GT(a, b) GSHIM_CMP(a, >, b, false)
#define EXPECT_GE(a, b) GSHIM_CMP(a, >=, b, false)
#define ASSERT_TRUE(c) GSHIM_CHECK(static_cast<bool>(c), #c, true)
#define ASSERT_FALSE(c) GSHIM_CHECK(!static_cast<bool>(c), "!(" #c ")", true)
#define ASSERT_EQ(a, b) GSHIM_CMP(a, ==, b, true)
#define ASSERT_NE(a, b) GSHIM_CMP(a, !=, b, true)
#define ASSERT_LT(a, b) GSHIM_CMP(a, <, b, true)
#define ASSERT_LE(a, b) GSHIM_CMP(a, <=, b, true)
#define ASSERT_GT(a, b) GSHIM_CMP(a, >, b, true)
#define ASSERT_GE(a, b) GSHIM_CMP(a, >=, b, true)
#define EXPECT_DOUBLE_EQ(a, b) GSHIM_CHECK(::gshim::ulp_eq((a), (b)), #a " ~= " #b, false)
#define ASSERT_DOUBLE_EQ(a, b) GSHIM_CHECK(::gshim::ulp_eq((a), (b)), #a " ~= " #b, true)
#define EXPECT_NEAR(a, b, t) GSHIM_CHECK(std::abs((a) - (b)) <= (t), #a " near " #b, false)
#define ASSERT_NEAR(a, b, t) GSHIM_CHECK(std::abs((a) - (b)) <= (t), #a " near " #b, true)
#define GSHIM_THROW(stmt, exc, fatal)                                     \
    do {                                                                  \
        bool gshim_ok_ = false;                                           \
        try {                                                             \
            stmt;                                                         \
        } catch (const exc&) {                                            \
            gshim_ok_ = true;                                             \
        } catch (...) {                                                   \
        }                                                                 \
        GSHIM_CHECK(gshim_ok_, #stmt " throws " #exc, fatal);             \
    } while (0)
#define EXPECT_THROW(stmt, exc) GSHIM_THROW(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) GSHIM_THROW(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                             \
    do {                                                                  \
        try {                                                             \
            stmt;                                                         \
        } catch (...) {                                                   \
            ::gshim::fail(__FILE__, __LINE__, #stmt " threw");            \
        }                                                                 \
    } while (0)
#define FAIL() GSHIM_CHECK(false, "FAIL()", true)
