# the other in-scope stages (static condensation, hybrid recovery, SpMV) of every config:
#   bash profiles/stages.sh r02   ->  gpurun_out/r02/stage_cfg<N>_<stage>.json
R=${1:-r02}; O=gpurun_out/$R; mkdir -p $O
for c in 1 2 3 4 5; do for s in condense recover spmv; do
  timeout 600 python bench.py --config $c --stage $s --steps 5 --warmup 2 > $O/stage_cfg${c}_$s.log 2>&1
  tail -1 $O/stage_cfg${c}_$s.log > $O/stage_cfg${c}_$s.json
done; done
python - <<PY
import json, glob
for f in sorted(glob.glob("$O/stage_cfg*_*.json")):
    try:
        d = json.loads(open(f).read())
        r = d["roofline"]
        print(f.split("/")[-1], f'{d["ms_per_step"]:.4f} ms', f'{d["value"]:.3e} {d["unit"]}', r["bound"], f'{r["frac"]:.3f}', "launches", d["gpu_launches"])
    except Exception as e:
        print(f, "FAILED", e)
PY
