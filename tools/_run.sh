mkdir -p gpurun_out
O=gpurun_out
# launch list of the bench command (cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu > $O/p_launches.log 2>&1
# DRAM traffic of the two headline kernels
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_ce -c 5 --csv --log-file $O/r02_traffic_ce.csv python bench.py --steps 1 --warmup 3 --no-extra --no-e2e --no-cpu --no-periodogram > $O/p_tr_ce.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_pg3 -c 2 --csv --log-file $O/r02_traffic_pg3.csv python tools/pgram_only.py 4096 1 > $O/p_tr_pg.log 2>&1
# full captures
ncu --set full --clock-control none --import-source on -k regex:fused_ce -c 1 -o $O/r02_fused_ce python tools/ce_only.py 1184 1 > $O/p_ce.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_pg3 -c 1 -o $O/r02_pg3 python tools/pgram_only.py 1024 0 > $O/p_pg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rowpass_zp -c 1 -o $O/r02_rowpass_zp python tools/cfg_rate.py cfg2 16 8 > $O/p_row.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:colpass2048 -c 1 -o $O/r02_colpass2048 python tools/cfg_rate.py cfg2 16 8 > $O/p_col.log 2>&1
ls -la $O | tail -20
