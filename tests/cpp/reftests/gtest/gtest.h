// Minimal GoogleTest-compatible harness (GTest is not installed in this
// image; /root/reference/proj/tests/CMakeLists.txt:1 needs it).  It covers
// exactly what the reference's test files use — TEST, TEST_F,
// ::testing::Test with SetUp/TearDown, EXPECT_/ASSERT_{EQ,NE,LT,LE,GT,GE,
// TRUE,FALSE,THROW}, FAIL() and `<<` messages — so those files compile
// unmodified against the B200 drop-in (tests/cpp/reftests/Makefile).
// Fatal assertions throw (they abort the test body like gtest's `return`).
// --gtest_filter=POS[-NEG] with ':'-separated '*' globs selects tests.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Test {
public:
    virtual ~Test() = default;
    virtual void SetUp() {}
    virtual void TearDown() {}
    virtual void TestBody() = 0;
};

namespace internal {

struct FatalFailure {};

struct TestInfo {
    std::string suite, name;
    std::function<Test*()> make;
};

inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}
inline bool& current_failed() {
    static bool f = false;
    return f;
}

struct Registrar {
    Registrar(const char* suite, const char* name, std::function<Test*()> make) {
        registry().push_back({suite, name, std::move(make)});
    }
};

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
    if constexpr (std::is_same_v<T, bool>) {
        return v ? "true" : "false";
    } else if constexpr (printable<T>::value) {
        std::ostringstream os;
        os << v;
        return os.str();
    } else {
        return "<" + std::to_string(sizeof(T)) + "-byte object>";
    }
}

class Message {
public:
    template <typename T>
    Message& operator<<(const T& v) {
        os_ << v;
        return *this;
    }
    std::string str() const { return os_.str(); }

private:
    std::ostringstream os_;
};

class AssertHelper {
public:
    AssertHelper(bool fatal, const char* file, int line, std::string what)
        : fatal_(fatal), file_(file), line_(line), what_(std::move(what)) {}
    void operator=(const Message& m) const {
        current_failed() = true;
        std::cout << file_ << ":" << line_ << ": Failure\n" << what_;
        const std::string extra = m.str();
        if (!extra.empty()) std::cout << "\n" << extra;
        std::cout << std::endl;
        if (fatal_) throw FatalFailure{};
    }

private:
    bool fatal_;
    const char* file_;
    int line_;
    std::string what_;
};

// Returns "" on success, else the failure description.
template <typename A, typename B, typename Op>
std::string compare(const char* ea, const char* eb, const char* opname, const A& a, const B& b, Op op) {
    if (op(a, b)) return {};
    return std::string("Expected: (") + ea + ") " + opname + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

inline bool glob(const char* p, const char* s) {
    if (*p == 0) return *s == 0;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && (*p == '?' || *p == *s) && glob(p + 1, s + 1);
}
inline bool any_glob(const std::string& pats, const std::string& name) {
    std::stringstream ss(pats);
    std::string p;
    while (std::getline(ss, p, ':'))
        if (!p.empty() && glob(p.c_str(), name.c_str())) return true;
    return false;
}

}  // namespace internal

inline void InitGoogleTest(int*, char**) {}

inline int RunAllTests(int argc, char** argv) {
    std::string pos = "*", neg;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        if (std::strncmp(a, "--gtest_filter=", 15) == 0) {
            std::string f = a + 15;
            const auto d = f.find('-');
            pos = d == std::string::npos ? f : f.substr(0, d);
            neg = d == std::string::npos ? "" : f.substr(d + 1);
            if (pos.empty()) pos = "*";
        }
    }
    int run = 0, failed = 0;
    std::vector<std::string> failures;
    for (auto& t : internal::registry()) {
        const std::string full = t.suite + "." + t.name;
        if (!internal::any_glob(pos, full) || internal::any_glob(neg, full)) continue;
        ++run;
        std::cout << "[ RUN      ] " << full << std::endl;
        internal::current_failed() = false;
        Test* obj = nullptr;
        try {
            obj = t.make();
            obj->SetUp();
            try {
                obj->TestBody();
            } catch (const internal::FatalFailure&) {
            }
            obj->TearDown();
        } catch (const internal::FatalFailure&) {
        } catch (const std::exception& e) {
            internal::current_failed() = true;
            std::cout << "unexpected exception: " << e.what() << std::endl;
        } catch (...) {
            internal::current_failed() = true;
            std::cout << "unexpected non-std exception" << std::endl;
        }
        delete obj;
        if (internal::current_failed()) {
            ++failed;
            failures.push_back(full);
            std::cout << "[  FAILED  ] " << full << std::endl;
        } else {
            std::cout << "[       OK ] " << full << std::endl;
        }
    }
    std::cout << "[==========] " << run << " tests ran." << std::endl;
    std::cout << "[  PASSED  ] " << (run - failed) << " tests." << std::endl;
    for (auto& f : failures) std::cout << "[  FAILED  ] " << f << std::endl;
    return failed ? 1 : 0;
}

}  // namespace testing

#define GD_GT_CLASS(suite, name) suite##_##name##_Test

#define GD_GT_DEFINE(suite, name, base)                                                                    \
    class GD_GT_CLASS(suite, name) : public base {                                                         \
    public:                                                                                                \
        void TestBody() override;                                                                          \
    };                                                                                                     \
    static ::testing::internal::Registrar suite##_##name##_registrar(                                      \
        #suite, #name, [] { return static_cast<::testing::Test*>(new GD_GT_CLASS(suite, name)()); });      \
    void GD_GT_CLASS(suite, name)::TestBody()

#define TEST(suite, name) GD_GT_DEFINE(suite, name, ::testing::Test)
#define TEST_F(fixture, name) GD_GT_DEFINE(fixture, name, fixture)

#define GD_GT_CHECK(fatal, text)                                                                           \
    if (const std::string gd_gt_msg_ = (text); gd_gt_msg_.empty())                                         \
        ;                                                                                                  \
    else                                                                                                   \
        ::testing::internal::AssertHelper(fatal, __FILE__, __LINE__, gd_gt_msg_) = ::testing::internal::Message()

#define GD_GT_CMP(fatal, a, b, opname, op)                                                                 \
    GD_GT_CHECK(fatal, ::testing::internal::compare(#a, #b, opname, (a), (b),                              \
                                                    [](const auto& x_, const auto& y_) { return op; }))

#define EXPECT_EQ(a, b) GD_GT_CMP(false, a, b, "==", x_ == y_)
#define EXPECT_NE(a, b) GD_GT_CMP(false, a, b, "!=", x_ != y_)
#define EXPECT_LT(a, b) GD_GT_CMP(false, a, b, "<", x_ < y_)
#define EXPECT_LE(a, b) GD_GT_CMP(false, a, b, "<=", x_ <= y_)
#define EXPECT_GT(a, b) GD_GT_CMP(false, a, b, ">", x_ > y_)
#define EXPECT_GE(a, b) GD_GT_CMP(false, a, b, ">=", x_ >= y_)
#define ASSERT_EQ(a, b) GD_GT_CMP(true, a, b, "==", x_ == y_)
#define ASSERT_NE(a, b) GD_GT_CMP(true, a, b, "!=", x_ != y_)
#define ASSERT_LT(a, b) GD_GT_CMP(true, a, b, "<", x_ < y_)
#define ASSERT_LE(a, b) GD_GT_CMP(true, a, b, "<=", x_ <= y_)
#define ASSERT_GT(a, b) GD_GT_CMP(true, a, b, ">", x_ > y_)
#define ASSERT_GE(a, b) GD_GT_CMP(true, a, b, ">=", x_ >= y_)

#define GD_GT_BOOL(fatal, cond, want)                                                                      \
    GD_GT_CHECK(fatal, (static_cast<bool>(cond) == (want))                                                 \
                           ? std::string()                                                                 \
                           : std::string("Value of: " #cond "\n  Actual: ") + ((want) ? "false" : "true") + \
                                 "\nExpected: " + ((want) ? "true" : "false"))
#define EXPECT_TRUE(c) GD_GT_BOOL(false, c, true)
#define EXPECT_FALSE(c) GD_GT_BOOL(false, c, false)
#define ASSERT_TRUE(c) GD_GT_BOOL(true, c, true)
#define ASSERT_FALSE(c) GD_GT_BOOL(true, c, false)

#define GD_GT_THROW(fatal, stmt, exc)                                                                      \
    GD_GT_CHECK(fatal, ([&]() -> std::string {                                                             \
                    try {                                                                                  \
                        stmt;                                                                              \
                    } catch (const exc&) {                                                                 \
                        return std::string();                                                              \
                    } catch (const std::exception& e_) {                                                   \
                        return std::string("Expected: " #stmt " throws " #exc "\n  Actual: it throws ") +  \
                               e_.what();                                                                  \
                    } catch (...) {                                                                        \
                        return std::string("Expected: " #stmt " throws " #exc                              \
                                           "\n  Actual: it throws a different type");                      \
                    }                                                                                      \
                    return std::string("Expected: " #stmt " throws " #exc "\n  Actual: it throws nothing"); \
                }()))
#define EXPECT_THROW(stmt, exc) GD_GT_THROW(false, stmt, exc)
#define ASSERT_THROW(stmt, exc) GD_GT_THROW(true, stmt, exc)

#define FAIL() ::testing::internal::AssertHelper(true, __FILE__, __LINE__, "Failed") = ::testing::internal::Message()
#define ADD_FAILURE() \
    ::testing::internal::AssertHelper(false, __FILE__, __LINE__, "Failed") = ::testing::internal::Message()

int main(int argc, char** argv);
#define GD_GTEST_MAIN \
    int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
