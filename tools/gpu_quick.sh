#!/bin/bash
# quick GPU check used during kernel work: GPU tests + a short bench summary
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python bench.py --no-dense --no-cpu --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['stages'])"
