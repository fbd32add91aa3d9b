set -u
mkdir -p gpurun_out
P=$(python -c "print(','.join('sw_b:%d'%t for t in range(0,33,2)))")
AB_REPEAT=2 AB_WORKLOADS="c3_1m_1080p c5_3m_1080p_64views c4_200k_contention_1080p" bash tools/ab_libs.sh gpurun_out/ab_vecred.jsonl "$P" libdistwar.so libdistwar_novec.so > gpurun_out/ab_vecred.txt 2>&1
python - <<'PY' > gpurun_out/red_peaks.json
import sys, json
sys.path.insert(0,'.')
from paper_2401_05345_b200.rasterizer import microbench_red
print(json.dumps({p: microbench_red(p, 1<<28) for p in range(7)}))
PY
cat gpurun_out/ab_vecred.txt gpurun_out/red_peaks.json
