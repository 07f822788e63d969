# Round-end measurement refresh on a B200 (gpurun): bench line (+ CPU leg), the
# reference arm, per-config table, ncu launch list of the bench, ncu --set full of one
# launch of each kind. Outputs under gpurun_out/; copy the summaries into profiles/.
set -x
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
python scripts/bench_configs.py --out gpurun_out/configs_final.jsonl > gpurun_out/configs_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/launches_final.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ecsr_tiled -c 4 -o gpurun_out/prof_final \
    python scripts/debug_launch.py > gpurun_out/prof_final.log 2>&1
