# --set full captures of the stage kernels (one launch each):  bash profiles/stage_captures.sh r02
R=${1:-r02}; O=gpurun_out/$R; mkdir -p $O
cap() {  # cfg stage kernel-regex tag
  timeout 600 python bench.py --config $1 --stage $2 --steps 2 --warmup 2 > $O/plain_$4.log 2>&1 || return
  timeout 900 ncu --set full --import-source on --clock-control none -k "$3" -c 1 -o $O/full_stage_$4 \
    python bench.py --config $1 --stage $2 --steps 1 --warmup 1 > $O/ncu_$4.log 2>&1
}
cap 2 condense regex:k_sc_pencil cfg2_condense
cap 3 condense regex:k_sc_warp cfg3_condense
cap 3 recover regex:k_recover_cta cfg3_recover
cap 5 recover regex:k_recover_wide cfg5_recover
cap 5 spmv regex:k_spmv_tiled cfg5_spmv
cap 2 spmv regex:k_spmv_rows cfg2_spmv
echo done
