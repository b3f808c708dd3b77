#!/bin/bash
# Run on the GPU box (gpurun): one `ncu --set full` capture per hot kernel and
# the launch list of a short bench run. Outputs go to gpurun_out/ncu/; read
# them here with tools/ncu_summarize.py, which writes profiles/ncu_summary.json.
#   gpurun -- 'bash tools/ncu_capture.sh [tag]'
set -u
TAG=${1:-cur}
ONLY=${2:-}
OUT=gpurun_out/ncu
mkdir -p "$OUT"
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex skip count cmd...
    local name=$1 rx=$2 skip=$3 cnt=$4
    shift 4
    if [ -n "$ONLY" ] && ! [[ " $ONLY " == *" $name "* ]]; then return; fi
    timeout 600 $NCU -k "regex:$rx" -s "$skip" -c "$cnt" -f -o "$OUT/${TAG}_$name" "$@" > "$OUT/${TAG}_$name.log" 2>&1
    echo "$name rc=$?" >> "$OUT/${TAG}_status.txt"
}
cap sellp_spmv sellp64_tma 2 1 python tools/profile_spmv.py sellp 27 200
cap sellp_spmv_7pt sellp64_tma 2 1 python tools/profile_spmv.py sellp 7 256
cap ell_spmv ell_tma_kernel 2 1 python tools/profile_spmv.py ell 27 200
cap ell_spmv_7pt ell_tma_kernel 2 1 python tools/profile_spmv.py ell 7 256
cap csr_rowblock csr_rowblock 2 1 python tools/profile_spmv.py csr 27 200 rowblock
cap csr_stream "csr_(stream|tma)" 2 1 python tools/profile_spmv.py csr 27 200 stream
cap csr_rmat seg8 2 1 python tools/profile_spmv.py csr_rmat 0 24 load_balance
cap csr_merge_rmat csr_merge_kernel 2 1 python tools/profile_spmv.py csr_rmat 0 24 merge
cap coo_rmat seg8 2 1 python tools/profile_spmv.py coo 0 24
cap gmres_multidot gmres_multidot_vec 20 1 python tools/profile_gmres.py
cap csr_poisson2d csr_ 2 1 python tools/profile_spmv.py csr 5 1000 auto
cap ell_fill fill_tma_kernel 2 1 python tools/profile_spmv.py convert 27 200
cap sellp_fill fill_tma_kernel 3 1 python tools/profile_spmv.py convert 27 200
cap cg_spmv_dot sellp64_tma 5 1 python tools/profile_cg.py 256 60
cap cg_update_r cg_update_r_vec 5 1 python tools/profile_cg.py 256 60
cap cg_update_xp cg_update_xp_vec 0 1 python tools/profile_cg.py 256 60
cap cg_update_xp_pair0 cg_update_xp_pair 4 1 python tools/profile_cg.py 256 60
cap cg_update_xp_pair1 cg_update_xp_pair 5 1 python tools/profile_cg.py 256 60
cap sort_downsweep rs_downsweep 2 1 python tools/quick_sort.py 22
cap sort_upsweep rs_upsweep 2 1 python tools/quick_sort.py 22
cap dedup_scatter dedup_scatter 1 1 python tools/quick_ingest.py
cap coo_ptrs coo_ptrs 1 1 python tools/quick_ingest.py
cap hybrid_coo_fill hybrid_coo 0 2 python tools/quick_hybrid.py 22
if [ -z "$ONLY" ]; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
        --log-file "$OUT/${TAG}_launches.csv" python bench.py --steps 4 --warmup 3 > "$OUT/${TAG}_launches_bench.log" 2>&1
    echo "launches rc=$?" >> "$OUT/${TAG}_status.txt"
fi
