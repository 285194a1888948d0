#!/bin/bash
# round-2 GPU pass z: configs[4] at spec for one rank of an 8-GPU run -- variants 224..255 of the 256, 400 steps each
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 3300 python scripts/bench_cfg4.py --scenes 32 --first-scene 224 > gpurun_out/r2z_cfg4_rank7.json 2> gpurun_out/r2z_cfg4.err
python -c "
import json
d=json.loads(open('gpurun_out/r2z_cfg4_rank7.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ['scenes','wall_s','scene_steps_per_s','contact_iter_per_s','converged_fraction','contact_steps','mean_iterations_contact_steps']}, d['loop'])
"; tail -n 3 gpurun_out/r2z_cfg4.err
