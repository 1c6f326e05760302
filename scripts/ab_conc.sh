# A/B of REI_CONCURRENT modes (stream layout of a level's kernels) on bench workloads
python -c "import torch; torch.zeros(1).cuda()"
for w in ${WL:-table1-row1 c2-t1-s0 table1-row8}; do
 for c in ${MODES:-0 1 2 3}; do
  REI_CONCURRENT=$c timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w','conc=$c', round(d['ms_per_step'],2), round(d['value']/1e9,2), d['config']['candidates_per_step'])" >> gpurun_out/ab_conc.txt
 done
done
