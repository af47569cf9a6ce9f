# launch lists (per-kernel device times, DRAM bytes, issue) for the given configs
# usage: bash scripts/gpu_launch_lists.sh "5 4" tag
CFGS=${1:-"5 4"}; TAG=${2:-x}
for c in $CFGS; do bash scripts/gpu_launches.sh $c $TAG; python scripts/launch_summary.py gpurun_out/launches_cfg${c}_$TAG.csv; done
