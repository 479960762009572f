# S1 rework: queries scattered straight to sorted slots + k_query_mh, single-pass scans; full GPU suite + A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c27_pytest.txt 2>&1
tail -3 gpurun_out/r2c27_pytest.txt
bash tools/variants.sh --no-cpu-baseline --no-e2e > gpurun_out/r2c27_ab.txt 2>&1
bash tools/variants.sh --no-cpu-baseline --no-e2e >> gpurun_out/r2c27_ab.txt 2>&1
bash tools/variants.sh --config c3 --no-cpu-baseline --no-e2e >> gpurun_out/r2c27_ab.txt 2>&1
cat gpurun_out/r2c27_ab.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2c27_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2c27_launches.csv 2>/dev/null | head -30 || true
