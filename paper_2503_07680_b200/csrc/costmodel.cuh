// costmodel.cuh — the analytic cost model as __host__ __device__ code.
//
// Reference: memory_used / iter_time (src/costmodel.cpp:37-104). The
// expressions keep the reference's evaluation order and every product,
// quotient and sum is rounded separately (no fused multiply-add): device
// code uses the _rn intrinsics, host code is compiled with
// -ffp-contract=off, so per-iteration times are bit-identical to x86-64
// g++ -O2 builds of the reference.
#pragma once

#include <cmath>
#include <cstdint>

#include "../../include/hbp_b200.h"

#if !defined(__CUDACC__)
#define __host__
#define __device__
#endif

namespace hbp_b200 {

#if defined(__CUDA_ARCH__)
#define HBP_MUL(a, b) __dmul_rn((a), (b))
#define HBP_DIV(a, b) __ddiv_rn((a), (b))
#define HBP_ADD(a, b) __dadd_rn((a), (b))
#define HBP_SUB(a, b) __dsub_rn((a), (b))
#else
#define HBP_MUL(a, b) ((a) * (b))
#define HBP_DIV(a, b) ((a) / (b))
#define HBP_ADD(a, b) ((a) + (b))
#define HBP_SUB(a, b) ((a) - (b))
#endif

// Bytes used at length l (costmodel.cpp:37-53). Caller checks sp / ckpt.
__host__ __device__ inline int64_t cm_memory_used(int64_t l, int32_t sp, int32_t ckpt, const hbp_hardware_profile& p) {
    const double shard = HBP_DIV(static_cast<double>(l), static_cast<double>(sp));
    const double activations =
        HBP_MUL(HBP_MUL(p.per_token_activation_memory, shard), static_cast<double>(p.layer_count));
    const double saved = HBP_DIV(HBP_MUL(HBP_MUL(p.gc_memory_saving_per_layer, static_cast<double>(ckpt)), shard),
                                 static_cast<double>(p.reference_length));
    return p.base_memory + static_cast<int64_t>(ceil(HBP_SUB(activations, saved)));
}

// Busy time of one device given its aggregated work (costmodel.cpp:84-98),
// after the memory check. padded > 0.
__host__ __device__ inline double cm_iter_time(int64_t padded, int64_t attention, int32_t sp, int32_t ckpt,
                                               const hbp_hardware_profile& p) {
    const double tokens = static_cast<double>(padded);
    const double compute =
        HBP_ADD(HBP_MUL(p.per_token_linear_cost, tokens),
                HBP_DIV(HBP_MUL(p.per_token2_attention_cost, static_cast<double>(attention)), static_cast<double>(sp)));
    const double recompute =
        HBP_MUL(HBP_DIV(HBP_MUL(p.gc_recompute_factor, static_cast<double>(ckpt)), static_cast<double>(p.layer_count)),
                compute);
    const double comm = sp > 1 ? HBP_MUL(HBP_MUL(p.sp_comm_cost, tokens), static_cast<double>(sp - 1)) : 0.0;
    return HBP_ADD(HBP_ADD(HBP_ADD(compute, recompute), comm), p.fixed_iteration_cost);
}

__host__ __device__ inline double cm_comm(int64_t padded, int32_t sp, const hbp_hardware_profile& p) {
    return sp > 1 ? HBP_MUL(HBP_MUL(p.sp_comm_cost, static_cast<double>(padded)), static_cast<double>(sp - 1)) : 0.0;
}

// HardwareProfile::validate (costmodel.cpp:14-35): 0 ok, else a code the
// host maps to the reference message.
__host__ __device__ inline int cm_profile_check(const hbp_hardware_profile& p) {
    if (p.per_token_linear_cost < 0 || p.per_token2_attention_cost < 0 || p.sp_comm_cost < 0 ||
        p.gc_recompute_factor < 0 || p.fixed_iteration_cost < 0)
        return 1;
    if (p.layer_count < 1) return 2;
    if (p.device_memory <= p.base_memory) return 3;
    if (p.per_token_activation_memory < 0 || p.gc_memory_saving_per_layer < 0) return 4;
    if (p.reference_length < 1) return 5;
    if (p.gc_memory_saving_per_layer > HBP_MUL(p.per_token_activation_memory, static_cast<double>(p.reference_length)))
        return 6;
    return 0;
}

inline const char* cm_profile_message(int code) {
    switch (code) {
        case 1: return "profile costs must be >= 0";
        case 2: return "layer_count must be >= 1";
        case 3: return "device_memory must exceed base_memory";
        case 4: return "memory constants must be >= 0";
        case 5: return "reference_length must be >= 1";
        case 6: return "gc_memory_saving_per_layer exceeds per-layer activation memory";
        default: return "";
    }
}

}  // namespace hbp_b200
