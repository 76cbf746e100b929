"""Static SASS opcode counts of the library's headline kernels (cuobjdump of
the built libhdrlpa.so): proof of TMA (UTMALDG), mbarrier (SYNCS), FP64
(DFMA/DMUL/DADD), spills (STL/LDL), MUFU and conversions per kernel."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1308_4908_b200/libhdrlpa.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
HEAD = {
    "lpa_fast_kernel<1,0,4,4,...> (cfg2 co-sited taps)": r"lpa_fast_kernelILi1ELb0ELi4ELi4ELi0ELb0ELb0ELb0E",
    "lpa_fast_kernel<2,1,6,0,RT2,ICISM> (cfg3/cfg5 ICI)": r"lpa_fast_kernelILi2ELb1ELi6ELi0ELi2ELb0ELb0ELb1E",
    "lpa_fast_kernel<2,1,6,0,RT2> (ICI, register state)": r"lpa_fast_kernelILi2ELb1ELi6ELi0ELi2ELb0ELb0ELb0E",
    "lpa_fast_kernel<1,0,4,0,0,STEER,MRGS> (CALPA steered pass)": r"lpa_fast_kernelILi1ELb0ELi4ELi0ELi0ELb1ELb1ELb0E",
    "lpa_slow_kernel<2> (exact path)": r"lpa_slow_kernelILi2E",
    "radiance_merge_kernel (cfg2 pre-pass)": r"radiance_merge_kernel",
    "radiance_phase_kernel (pre-pass)": r"radiance_phase_kernel",
    "steering_field_tiled_kernel (CALPA)": r"steering_field_tiled_kernel",
    "lpa_samples_kernel<1> (scattered samples)": r"lpa_samples_kernelILi1E",
}
OPS = ["UTMALDG", "SYNCS", "DFMA", "DMUL", "DADD", "DSETP", "MUFU", "F2F", "FFMA", "LDS", "STS",
       "LDG", "STG", "STL", "LDL", "BRA", "SHFL"]
funcs = re.split(r"\n\s*Function : ", out)
for label, pat in HEAD.items():
    for f in funcs:
        name = f.split("\n", 1)[0]
        if re.search(pat, name):
            cnt = collections.Counter()
            for line in f.split("\n"):
                m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
                if m:
                    cnt[m.group(2)] += 1
            tot = sum(cnt.values())
            print(f"{label}\n  {name[:110]}\n  {tot} SASS instructions; " +
                  ", ".join(f"{o} {cnt[o]}" for o in OPS))
            break
