# one --set full capture of a stage kernel:  bash profiles/prof_stage.sh <cfg> <stage> <kernel regex> <tag>
set -u
C=$1; S=$2; K=$3; T=${4:-s}
O=gpurun_out/prof_$T
mkdir -p $O
timeout 600 python bench.py --config $C --stage $S --steps 2 --warmup 2 > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -c 1 -o $O/full \
  python bench.py --config $C --stage $S --steps 1 --warmup 1 > $O/ncu.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
echo done
