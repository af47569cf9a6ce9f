# per-kernel launch lists of a config for the working-tree library and a variant:
# bash scripts/gpu_launch_ab.sh <cfg> <variant>
CFG=${1:-4}; V=${2:-head}
bash scripts/gpu_launches.sh $CFG new
python scripts/launch_summary.py gpurun_out/launches_cfg${CFG}_new.csv | grep -v "at::\|gen_kernel"
cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_new.so
cp variants/lib_$V.so paper_1609_01010_b200/_lib/libmodconv_b200.so
bash scripts/gpu_launches.sh $CFG $V
python scripts/launch_summary.py gpurun_out/launches_cfg${CFG}_$V.csv | grep -v "at::\|gen_kernel"
cp /tmp/lib_new.so paper_1609_01010_b200/_lib/libmodconv_b200.so
