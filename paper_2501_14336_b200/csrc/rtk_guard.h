// rtk_guard.h — exceptions -> status codes + thread-local message for every extern "C" entry.
#pragma once
#include <exception>
#include <new>
#include <string>

#include "../../include/rtk_c.h"
#include "rtk_engine.h"

namespace rtk_b200 {

extern thread_local std::string g_last_error;

inline int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return RTK_OK;
    } catch (const Error& e) {
        return fail(e.code, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(RTK_OUT_OF_MEMORY, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(RTK_INTERNAL, e.what());
    }
}

}  // namespace rtk_b200
