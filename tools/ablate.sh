#!/bin/bash
# debug timing ablations of the dK/dV kernel (results are NOT correct with VSA_ABLATE != 0)
for a in 0 23; do
  echo -n "ablate=$a: "
  VSA_ABLATE=$a timeout 200 python bench.py --no-dense --no-cpu --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages']['fine_bwd'])"
done
