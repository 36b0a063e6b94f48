# PS persistent forward: per-unit trace and the profiling experiments
timeout 200 python tools/trace_fwd.py 1 2>&1 | tail -16
for e in 0 1 2 4; do CSR_FEXP=$e timeout 120 python tools/time_ops.py 1 2>&1 | tail -1 | sed "s/^/[fexp=$e] /"; done
