# K5 MSD form: per-kernel launch times (ncu launch list) of one table build (L = 50, N = 1e6 random keys), and a full capture of segment_sort
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_tables_launches.csv python tools/prof_tables.py 50 1000000 > /dev/null 2>&1; echo list=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:segment_sort -s 1 -c 1 -o gpurun_out/r2n_segsort -f python tools/prof_tables.py 50 1000000 > /dev/null 2>&1; echo full=$?
