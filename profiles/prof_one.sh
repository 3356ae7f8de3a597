# one --set full capture of the kernels matching $2 for bench config $1 (GPU box):
#   bash profiles/prof_one.sh 2 'regex:k_rt0_brick' tag [count]
set -u
C=$1; K=$2; T=${3:-p}; N=${4:-2}
O=gpurun_out/prof_$T
mkdir -p $O
timeout 600 python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -c $N -o $O/full \
  python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu --no-configs --no-graph > $O/ncu.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page source --csv > $O/source.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
echo done
