"""Local-memory (spill) instructions of the executor kernel per source line,
from an object compiled here: python scripts/sass_spills.py [obj] [file]."""
import collections, re, subprocess, sys
obj = sys.argv[1] if len(sys.argv) > 1 else "/tmp/ex.o"
want = sys.argv[2] if len(sys.argv) > 2 else "decode.cuh"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
txt = subprocess.run(["nvdisasm", "-g", "-c", "/dev/stdin"], input=b"", capture_output=True).stdout
# cuobjdump -sass has no line info: extract the cubin and disassemble it with -g
subprocess.run(["cuobjdump", "-xelf", "all", obj], capture_output=True, cwd="/tmp")
import glob, os
cub = sorted(glob.glob("/tmp/*.sm_100a.cubin"), key=os.path.getmtime)[-1]
L = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.splitlines()
st = next(i for i, l in enumerate(L) if l.startswith(".text.ds_executor_kernel"))
cur = None
cnt = collections.Counter()
for l in L[st:]:
    m = re.search(r'//## File ".*?/([\w\.]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
    if re.search(r"\b(LDL|STL)", l) and cur:
        cnt[cur] += 1
print(want, sum(v for k, v in cnt.items() if k[0] == want), sorted((k[1], v) for k, v in cnt.items() if k[0] == want))
