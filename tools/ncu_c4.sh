# full ncu capture of the single-graph executor on one config: bash tools/ncu_c4.sh <tag> [config] [kernel regex]
# (eager module loading: with lazy loading ncu intermittently misses the cooperative launches)
TAG=$1; C=${2:-C4-PARALL}; K=${3:-pslot|parall|persistent}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CUDA_MODULE_LOADING=EAGER timeout 900 ncu -k "regex:$K" --launch-skip 3 --launch-count 1 --set full --import-source on --clock-control none -o $OUT/ncu_$C python tools/time_probe.py $C 2 > $OUT/ncu_$C.log 2>&1
tail -2 $OUT/ncu_$C.log
