"""Tile-geometry sweep on the bench workload: runs tools/profile_step.py under each environment
configuration and reports the best step time (ms).

    python tools/sweep.py "QBG_COALESCE=2" "QBG_FWD_M=13" ...
"""
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def run(cfg: str, steps: int = 5) -> str:
    env = dict(os.environ)
    for kv in cfg.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, os.path.join(HERE, "profile_step.py"), "--steps", str(steps)], env=env,
                         capture_output=True, text=True, timeout=900)
    times = [float(m) for m in re.findall(r"step ([\d.]+) ms", out.stdout)]
    if not times:
        return f"{cfg or 'default'}: FAILED {out.stdout[-300:]} {out.stderr[-600:]}"
    e = re.findall(r"E=([-\d.e]+)", out.stdout)
    return f"{cfg or 'default'}: best {min(times[1:] or times):.2f} ms  E={e[-1] if e else '?'}"


if __name__ == "__main__":
    for c in [""] + sys.argv[1:]:
        print(run(c), flush=True)
