F=gpurun_out/s15; mkdir -p $F; rm -f $F/probe.txt
for v in 0 1; do for x in 32 33 34 36 40; do timeout 60 tools/c/tma_probe $v $x 2>&1 | grep variant >> $F/probe.txt; done; done
cat $F/probe.txt
