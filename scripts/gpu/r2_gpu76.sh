for v in 0 4096; do
TC_VIX_SMALL=$v timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum --clock-control none --csv --log-file gpurun_out/vstage_$v.csv -k regex:"seg_sort|vstage|big_back|small_cap" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
done
