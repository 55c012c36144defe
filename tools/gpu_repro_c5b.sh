# determinism probe with device-array checksums per build (AMG_DEBUG_CHECKSUM=1)
timeout 1500 env AMG_DEBUG_CHECKSUM=1 python tools/repro_c5.py 256x256x256 10 > gpurun_out/rpc.txt 2> gpurun_out/rpc.err
grep build gpurun_out/rpc.txt | sed 's/sizes \[[0-9, ]*\] //'
python - <<'PY'
lines = open('gpurun_out/rpc.err').read().splitlines()
ck = [l for l in lines if l.startswith('amg-checksum')]
per = len(ck) // 10
builds = [ck[i * per:(i + 1) * per] for i in range(10)]
ref = builds[0]
for b, blk in enumerate(builds):
    diffs = [(r, x) for r, x in zip(ref, blk) if r != x]
    print('build', b, 'differs from build 0 in', len(diffs), 'lines')
    for r, x in diffs[:6]:
        print('   0:', r[:200]); print('   %d:' % b, x[:200])
PY
