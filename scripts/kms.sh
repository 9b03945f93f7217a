#!/bin/bash
# prints ms per step and the per-kernel device times of one bench configuration (default c3)
python bench.py --only --no-cpu "$@" 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['ms_per_step'],4), {k: round(v,4) for k,v in j['roofline']['kernels_ms'].items()})"
