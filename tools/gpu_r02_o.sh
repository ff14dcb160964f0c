# kTrig padded back to 19 entries (constant-bank offsets of the later tables as before the
# three-FMA reduction): A/B against the unpadded library (lib/old)
mkdir -p gpurun_out/r02_o
for rep in 1 2; do
for w in C2U C5 C3a C2; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_o/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_o/old.jsonl
done
done
