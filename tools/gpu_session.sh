# Scratch driver for one gpurun call (edited per experiment).
set -x
F=gpurun_out/san
mkdir -p $F
timeout 120 python tools/sanitize.py > $F/plain.log 2>&1
for tool in memcheck racecheck; do
  echo "## $tool" >> $F/san.txt
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool python tools/sanitize.py 2>&1 | grep -v "^========= *$" | tail -6 >> $F/san.txt
  echo "exit=${PIPESTATUS[0]}" >> $F/san.txt
done
