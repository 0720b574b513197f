"""ORACLE (test infrastructure only): the Algorithm-1 switch controller.

Restates /root/reference/pkg/src/hybridpar/monitor.py:121-205 as a pure
function over a recorded series (dict t -> M) so the GPU controller and the
host mirror can both be checked against it.
"""
from __future__ import annotations

WARM, PAR, FC = "warm_up", "parallelism", "fully_connecting"


def step(state: dict, series: dict, t: int, L: int, g: float, tau_cap: int, k: int) -> str:
    """One update_controller iteration (monitor.py:146-189); mutates state."""
    s = state["steps"] + 1
    if state["tau1"] is None:
        fire = False
        if t in series and (t + L) in series:
            slope = (series[t] - series[t + L]) / L           # monitor.py:121-132
            fire = 0.0 <= slope < g
        if fire:
            state["tau1"] = min(s, tau_cap)
        elif s >= tau_cap:
            state["tau1"] = tau_cap
        if state["tau1"] is not None:
            state["tau2"] = state["tau1"] + k
        label = WARM
    elif s <= state["tau1"]:
        label = WARM
    elif s <= state["tau2"]:
        label = PAR
    else:
        label = FC
    state["steps"] = s
    return label


def replay(pairs, L, g, tau_cap, k):
    """monitor.py:192-205 — returns (tau1, tau2, labels)."""
    state = {"steps": 0, "tau1": None, "tau2": None}
    series, labels = {}, []
    for t, m in pairs:
        series[t] = float(m)
        labels.append(step(state, series, t, L, g, tau_cap, k))
    return state["tau1"], state["tau2"], labels
