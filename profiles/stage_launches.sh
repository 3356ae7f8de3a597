O=gpurun_out/lst; mkdir -p $O
for c in 3 2; do for s in recover condense; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_${c}_$s.csv python bench.py --config $c --stage $s --steps 1 --warmup 1 > $O/l_${c}_$s.log 2>&1
done; done
