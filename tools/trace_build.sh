#!/bin/bash
# the -DPRISM_TRACE diagnostics build into ab/libprism_trace.so (the product build is left as it is)
cd /root/repo
PRISM_NVCC_EXTRA=-DPRISM_TRACE python - <<'PY'
import os, subprocess
from paper_2605_08581_b200 import build as B
os.makedirs("/root/repo/build/trace", exist_ok=True)
comp, link = B.commands(out="/root/repo/ab/libprism_trace.so")
comp = [[a.replace("/root/repo/build/", "/root/repo/build/trace/") for a in c] for c in comp]
link = [a.replace("/root/repo/build/", "/root/repo/build/trace/") for a in link]
ps = [subprocess.Popen(c) for c in comp]
assert all(p.wait() == 0 for p in ps)
subprocess.run(link, check=True)
PY
