cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tr2
for n in 256 32; do
timeout 600 python tools/trace_probe.py $n > gpurun_out/tr2/report_$n.txt 2>&1; echo rc=$?
rm -f gpurun_out/trace_${n}_auto.bin
done
