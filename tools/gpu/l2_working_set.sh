# quad-kernel DRAM traffic and L2 hit rate vs batch size (the L2 working-set measurement in DESIGN.md)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/l2
for n in 64 128 256; do
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-es --no-parity --n-seq $n"
$CMD > gpurun_out/l2/plain$n.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"pa_quad|pa_fast|classify" -s 12 -c 4 --csv --log-file gpurun_out/l2/m$n.csv $CMD > gpurun_out/l2/ncu$n.log 2>&1
echo n=$n rc=$?
done
