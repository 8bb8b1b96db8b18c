# Full-size parity of every BASELINE configuration (tools/parity_full.py), one record per
# solve appended to gpurun_out/r02_parity.jsonl as it is produced; the markdown tables at
# the end (tools/parity_report.py, with the committed config-5 CPU floors).
set -u
mkdir -p gpurun_out
nproc > gpurun_out/r02_parity_host.txt; free -g >> gpurun_out/r02_parity_host.txt
for k in ${PARITY_CONFIGS:-1 2 3 5 4}; do
  timeout ${PARITY_TIMEOUT:-5400} python -u tools/parity_full.py --configs $k --out gpurun_out/r02_parity.jsonl \
    > gpurun_out/r02_parity_cfg$k.log 2>&1
  echo "config $k rc=$?"
done
python tools/parity_report.py gpurun_out/r02_parity.jsonl profiles/r02_cfg5_floor.jsonl > gpurun_out/r02_parity_tables.md
head -20 gpurun_out/r02_parity_tables.md
