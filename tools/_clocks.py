"""Clock record for the side benches (tools/*.py): samples nvidia-smi SM clocks
and throttle reasons (bench.ClockSampler) while the tool runs and prints one
final JSON line {"clocks": {...}} beside its numbers (B200_PROFILING.md timing
hygiene: a number without a clock record is not evidence)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_with_clocks(fn, tool):
    from bench import ClockSampler
    with ClockSampler(0) as clk:
        fn()
    print(json.dumps({"tool": tool, "clocks": clk.summary()}), flush=True)
