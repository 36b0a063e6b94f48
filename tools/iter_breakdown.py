"""ADMM iteration time with parts of the loop skipped (CSR_DBG_SKIP, profiling
only: the numbers are timings of a broken solver)."""
import ctypes, os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg = sys.argv[1] if len(sys.argv) > 1 else "1"
for skip in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "3", "7", "11", "13", "14", "15"]):
    env = dict(os.environ, CSR_DBG_SKIP=skip)
    if skip == "0":
        env.pop("CSR_DBG_SKIP")
    out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "20", "--no-e2e",
                          "--no-cpu"], capture_output=True, text=True, env=env)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(f"skip={skip:>2}  ms/iter {d['ms_per_step']:.4f}")
    except Exception:
        print("skip", skip, "failed", out.stderr[-400:])
