// engine_ctx.hpp — the façade's link to the C-ABI: one engine context per
// host thread (device from $HBP_DEVICE, default 0) and status -> exception
// mapping with the reference's types and message text.
#pragma once

#include <cstdlib>
#include <string>

#include "hbp/errors.hpp"
#include "hbp_b200.h"

namespace hbp::detail {

inline hbp_ctx* ctx() {
    thread_local struct Holder {
        hbp_ctx* c = nullptr;
        ~Holder() {
            if (c) hbp_ctx_destroy(c);
        }
    } holder;
    if (!holder.c) {
        const char* dev = std::getenv("HBP_DEVICE");
        const int rc = hbp_ctx_create(dev ? std::atoi(dev) : 0, &holder.c);
        if (rc != HBP_OK) throw Error("hbp B200 engine: no CUDA device available (status " + std::to_string(rc) + ")");
    }
    return holder.c;
}

[[noreturn]] inline void raise(int rc) {
    const std::string msg = hbp_last_error(ctx());
    switch (rc) {
        case HBP_ERR_VALIDATION: throw ValidationError(msg);
        case HBP_ERR_INFEASIBLE: throw InfeasibleError(msg);
        case HBP_ERR_IO: throw IoError(msg);
        default: throw Error(msg);
    }
}

inline void check(int rc) {
    if (rc != HBP_OK) raise(rc);
}

}  // namespace hbp::detail
