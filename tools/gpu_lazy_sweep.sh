#!/bin/bash
# Algorithm 2 (lazy averaging) on C2c: it/s and iterations to rel. error 1e-6 for P = 1, 2, 4, 8
# at eta 0.5 and 0.1 (the paper's parallel runs use eta = 0.1), against Algorithm 1.
mkdir -p gpurun_out
python paper_2509_19267_b200/_build.py > gpurun_out/build.log 2>&1 || exit 1
for eta in 0.5 0.1; do
  for P in 0 1 2 4 8; do
    timeout 600 python bench.py --workload C2c --eta $eta --lazy $P --steps 1000 --warmup 5 --skip-cpu --skip-e2e --skip-phases \
      > gpurun_out/lazy_C2c_eta${eta}_P$P.json 2> gpurun_out/lazy_C2c_eta${eta}_P$P.err
    python -c "
import json; d=json.loads(open('gpurun_out/lazy_C2c_eta${eta}_P$P.json').read().strip().splitlines()[-1])
t=d['time_to_tol'] or {}; print('eta', $eta, 'P', $P, 'it/s', d['value'], 'ttt iters', t.get('iters'), 'seconds', t.get('seconds'), 'outcome', t.get('outcome'), 'rel', t.get('rel_err'))"
  done
done
