// NEXT-4: the paper's analytic checkpoint model and K selection (host-only).
//
//  P:184 (§3.1)  P = T_ckpt/(N T_step) + p N T_step/2 + p T_load            (waste fraction)
//  P:189         N* = sqrt(2 T_ckpt / (p T_step^2));  P:191 P* = sqrt(2 p T_ckpt) + p T_load,
//                GPU utilization overhead P*/(P*+1)
//  P:318-320 (§4.2.3)  T_Async-O = (N-1) T_step;  T_GoCkpt = sum_{i<N} i*r T_step = r N(N-1)/2 T_step,
//                with r the gradient share of a part's bytes (the paper's 1/7; 1/6 for this build's
//                12-B state + 2-B gradient, R4)
//  K selection (ours): the smallest K whose largest per-step D2H
//                V_max(K) = max_i 12|P_i| + 2 hi_i [i<K] under the session's plan (equal: step K-1;
//                balanced, R17: about equal on every step) fits in `budget` x T_step at BW.
#include <cmath>

#include "internal.h"

extern "C" {

double gck_model_waste_fraction(double t_ckpt, double interval_steps, double t_step, double p_fail, double t_load) {
    return t_ckpt / (interval_steps * t_step) + p_fail * interval_steps * t_step / 2.0 + p_fail * t_load;
}

double gck_model_optimal_interval(double t_ckpt, double t_step, double p_fail) {
    return std::sqrt(2.0 * t_ckpt / (p_fail * t_step * t_step));
}

double gck_model_optimal_waste(double t_ckpt, double p_fail, double t_load) {
    return std::sqrt(2.0 * p_fail * t_ckpt) + p_fail * t_load;
}

double gck_model_stall_async_o(uint32_t N, double t_step) { return (N >= 1 ? N - 1.0 : 0.0) * t_step; }

double gck_model_stall_gockpt(uint32_t N, double t_step, double grad_share) {
    return grad_share * N * (N - 1.0) / 2.0 * t_step;
}

gck_status gck_recommend_k(uint64_t n, uint32_t part_align, int32_t plan, double link_gbs, double t_step_s,
                           double budget, uint32_t k_max, uint32_t *k_out, double *v_max_bytes) {
    if (!k_out || n == 0 || link_gbs <= 0 || t_step_s <= 0 || budget <= 0 || k_max == 0 || k_max > GCK_K_LIMIT)
        return GCK_E_INVALID;
    const uint32_t A = part_align ? part_align : 1024;
    uint64_t lo_hi[2 * GCK_K_LIMIT];
    for (uint32_t K = 1; K <= k_max; ++K) {
        if (gck_plan_parts_mode(n, K, A, plan, lo_hi) != GCK_OK) break;
        uint64_t vmax = 0;
        for (uint32_t i = 0; i < K; ++i) {
            const uint64_t part = lo_hi[2 * i + 1] - lo_hi[2 * i];
            const uint64_t v = 12 * part + (i + 1 < K ? 2 * lo_hi[2 * i + 1] : 0);
            if (v > vmax) vmax = v;
        }
        if ((double)vmax / (link_gbs * 1e9) <= budget * t_step_s) {
            *k_out = K;
            if (v_max_bytes) *v_max_bytes = (double)vmax;
            return GCK_OK;
        }
    }
    *k_out = 0;  // no K up to k_max keeps the per-step transfer inside the budget
    return GCK_E_INVALID;
}

}  // extern "C"
