for cfg in "1 2 1" "1 1 0" "2 2 0" "1 2 0" "2 3 1" "0 2 1"; do
set -- $cfg
FC_BCGS_PRUNE_FIRST=$1 FC_BCGS_PRUNE_GAP=$2 FC_BCGS_PRUNE_INC=$3 timeout 300 python tools/solve_time.py 1024 1e-6 3
done
