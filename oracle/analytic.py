"""NEXT-4 oracle: the paper's analytic checkpoint model written out (TEST INFRASTRUCTURE ONLY).

P:180-186 (§3.1)  T_waste = T_save + 1/2 p N T_total T_step + p T_total T_load, T_save =
                  T_total/(N T_step) T_ckpt;  P = T_waste / T_total.
P:187-195         N* from dP/dN = 0;  P* = sqrt(2 p T_ckpt) + p T_load;  overhead P*/(P*+1).
P:316-322 (§4.2.3) T_Async-O = (N-1) T_step;  T_GoCkpt = sum_{i=1}^{N-1} i/7 T_step.
"""

import math


def waste_fraction(t_ckpt, N, t_step, p, t_load):
    t_total = 1.0                                     # P is T_waste / T_total: any T_total
    t_save = t_total / (N * t_step) * t_ckpt
    t_waste = t_save + 0.5 * p * N * t_total * t_step + p * t_total * t_load
    return t_waste / t_total


def optimal_interval(t_ckpt, t_step, p):
    return math.sqrt(2 * t_ckpt / (p * t_step ** 2))


def optimal_waste(t_ckpt, p, t_load):
    return math.sqrt(2 * p * t_ckpt) + p * t_load


def stall_async_o(N, t_step):
    return (N - 1) * t_step


def stall_gockpt(N, t_step, share=1 / 7):
    return sum(i * share * t_step for i in range(1, N))
