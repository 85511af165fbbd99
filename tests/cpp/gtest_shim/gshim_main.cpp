// Runner of the gtest shim: every registered TEST in registration order.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "gtest/gtest.h"

int main() {
    const char* filt = std::getenv("SHIM_FILTER");
    int run = 0, failed = 0;
    for (const auto& t : gshim::registry()) {
        const std::string id = std::string(t.suite) + "." + t.name;
        if (filt && id.find(filt) == std::string::npos) continue;
        const int before = gshim::failures();
        ++run;
        try {
            t.fn();
        } catch (const gshim::Fatal&) {
        } catch (const std::exception& e) {
            gshim::fail(t.suite, 0, std::string("uncaught exception: ") + e.what());
        }
        const bool ok = gshim::failures() == before;
        failed += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "  OK  " : " FAIL ", id.c_str());
    }
    std::printf("%d tests, %d passed, %d failed\n", run, run - failed, failed);
    return failed == 0 ? 0 : 1;
}
