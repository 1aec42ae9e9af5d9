timeout 600 python -m pytest tests -m gpu -x -q -k "tables" 2>&1 | tail -2 > gpurun_out/qt.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tables_launches.csv python tools/prof_tables.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/tables_launches.csv | grep -E "kernel|mean_us" | head -10
python tools/prof_tables.py
cat gpurun_out/qt.log
