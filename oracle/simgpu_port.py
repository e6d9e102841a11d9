"""Timing / energy / thermal model port (TEST INFRASTRUCTURE ONLY).

CPU restatement of the reference's hot path — the simulator that the B200 engine replaces:
  roofline duration ........ reference pkg/src/schedfront/simgpu.py:144-168
  dynamic energy ........... simgpu.py:171-178
  sequential makespan ...... simgpu.py:181-188
  overlap makespan ......... simgpu.py:191-261  (event loop: SM sharing, proportional HBM sharing,
                                                exposed comm tail, sync point, launch overhead)
  admission checks ......... simgpu.py:269-279
  thermal protocol ......... simgpu.py:289-364  (closed-form first-order thermal ODE, noise / counter
                                                quantum drawn from the caller's numpy Generator)

One deliberate difference, flagged by `guard`: the reference loop has an epsilon exit only for
the compute residual (simgpu.py:251), so a ~1e-9-byte comm residual can make `dt` shrink to zero
and spin forever at B200-scale parameters (SURVEY.md §0 finding 1).  With guard=True a comm
residual below 1e-9 * max(1, comm_bytes) is zeroed; where the reference terminates the result
agrees to ~1e-15 relative (pinned by tests/test_oracle_golden.py against vectors produced by the
reference itself, tools/make_golden.py).
"""

from __future__ import annotations

import math


class InvalidConfig(ValueError):
    pass


def roofline_ms(k, f_mhz, sms, gpu, bw_frac=1.0):
    if sms < 1:
        raise InvalidConfig("kernel needs at least one SM")
    if k.comm_bytes > 0:
        return k.comm_bytes / gpu.comm_rate_bps(sms) * 1e3
    if k.flops == 0 and k.bytes == 0:
        return 0.0
    tc = k.flops / gpu.flop_rate(sms, f_mhz) if k.flops else 0.0
    tm = k.bytes / (gpu.mem_bw_bps * bw_frac) if k.bytes else 0.0
    return max(tc, tm) * 1e3


def dyn_energy_j(part, f_mhz, gpu):
    sc = (f_mhz / gpu.f_max_mhz) ** 2
    e = 0.0
    for k in part.comp_kernels:
        e += gpu.e_flop_j * k.flops * sc + gpu.e_byte_j * k.bytes
    return e + gpu.e_comm_byte_j * part.comm_kernel.comm_bytes


def seq_ms(part, f_mhz, gpu):
    total = sum(roofline_ms(k, f_mhz, gpu.num_sms, gpu) for k in part.comp_kernels)
    return total + roofline_ms(part.comm_kernel, f_mhz, gpu.sm_bw_saturation, gpu)


def _co_run(k, f_mhz, sm_alloc, gpu, t, left, comm_full, guard, comm_total, max_steps):
    """Advance one span kernel while the comm kernel (`left` bytes to go) may share the GPU."""
    fl, by = k.flops, k.bytes
    bw = gpu.mem_bw_bps
    steps = 0
    while fl > 0 or by > 0:
        steps += 1
        if steps > max_steps:
            raise RuntimeError("overlap event loop did not terminate (reference hang, SURVEY §0-1)")
        frate = gpu.flop_rate(gpu.num_sms - sm_alloc if left > 0 else gpu.num_sms, f_mhz)
        alone = 0.0
        if fl > 0:
            alone = max(alone, fl / frate)
        if by > 0:
            alone = max(alone, by / bw)
        if alone == 0.0:
            break
        want_k = by / alone if by > 0 else 0.0
        want_c = comm_full if left > 0 else 0.0
        want = want_k + want_c
        share = bw / want if want > bw else 1.0
        brate, crate = want_k * share, want_c * share
        dt = 0.0
        if fl > 0:
            dt = max(dt, fl / frate)
        if by > 0:
            dt = max(dt, by / brate)
        if left > 0 and crate > 0:
            dt = min(dt, left / crate)
        t += dt
        fl = max(0.0, fl - frate * dt)
        by = max(0.0, by - brate * dt)
        if left > 0:
            left = max(0.0, left - crate * dt)
            if guard and left <= 1e-9 * max(1.0, comm_total):
                left = 0.0
        if fl <= 1e-9 * max(1.0, k.flops) and by <= 1e-9 * max(1.0, k.bytes):
            break
    return t, left


def overlap_ms(part, f_mhz, sm_alloc, start, span, gpu, guard=True, max_steps=100000):
    ks = part.comp_kernels
    end = start + min(span, len(ks) - start)
    t = 0.0
    for k in ks[:start]:
        t += roofline_ms(k, f_mhz, gpu.num_sms, gpu) / 1e3
    comm_total = part.comm_kernel.comm_bytes
    left = comm_total
    comm_full = gpu.comm_rate_bps(sm_alloc)
    for k in ks[start:end]:
        t, left = _co_run(k, f_mhz, sm_alloc, gpu, t, left, comm_full, guard, comm_total, max_steps)
    if left > 0:
        t += left / comm_full  # exposed tail before the sync point
    for k in ks[end:]:
        t += roofline_ms(k, f_mhz, gpu.num_sms, gpu) / 1e3
    return t * 1e3 + gpu.overlap_launch_overhead_ms


def simulate(part, cfg, gpu, guard=True):
    """(time_ms, dyn_energy_j) of one noise-free execution."""
    tm = cfg.timing
    if tm.is_sequential:
        ms = seq_ms(part, cfg.frequency_mhz, gpu)
    else:
        if cfg.sm_alloc >= gpu.num_sms:
            raise InvalidConfig("sm_alloc must leave SMs for computation")
        if tm.start >= len(part.comp_kernels):
            raise InvalidConfig("overlap start out of range")
        ms = overlap_ms(part, cfg.frequency_mhz, cfg.sm_alloc, tm.start, tm.span, gpu, guard)
    return ms, dyn_energy_j(part, cfg.frequency_mhz, gpu)


def _heat(thermal, temp, power_w, dur_s):
    if dur_s <= 0:
        return temp, 0.0
    tau = thermal.cool_tau_s
    if tau == 0.0:
        return thermal.ambient_c, 0.0
    rise = thermal.heat_coeff * power_w * tau
    x0 = temp - thermal.ambient_c
    decay = math.exp(-dur_s / tau)
    x = rise + (x0 - rise) * decay
    return thermal.ambient_c + x, rise * dur_s + (x0 - rise) * tau * (1.0 - decay)


def _cool(thermal, temp, dur_s):
    if dur_s <= 0:
        return temp
    tau = thermal.cool_tau_s
    if tau == 0.0:
        return thermal.ambient_c
    return thermal.ambient_c + (temp - thermal.ambient_c) * math.exp(-dur_s / tau)


def measure(part, cfg, gpu, thermal, protocol, temp_c, rng, guard=True):
    """Returns (time_ms, dyn_j, static_j, total_j, new_temp_c)."""
    ms, dyn = simulate(part, cfg, gpu, guard)
    static = ms / 1000.0 * gpu.p_static_w
    exec_s = ms / 1e3
    if exec_s <= 0:
        return ms, dyn, static, dyn + static, temp_c
    power = (dyn + static) / exec_s
    temp, _ = _heat(thermal, temp_c, power, protocol.warmup_s)
    reps = max(1, int(protocol.window_s // exec_s))
    win = reps * exec_s
    temp, integral = _heat(thermal, temp, power, win)
    factor = 1.0 + thermal.power_temp_coeff * integral / win
    sigma = protocol.noise_std_frac / math.sqrt(reps)
    nt = rng.normal(1.0, sigma)
    ne = rng.normal(1.0, sigma)
    q = rng.normal(0.0, protocol.counter_quantum_j / reps)
    temp = _cool(thermal, temp, protocol.cooldown_s)
    t2 = ms * nt
    d2 = dyn * factor * ne + q
    s2 = t2 / 1000.0 * gpu.p_static_w
    return t2, d2, s2, d2 + s2, temp
