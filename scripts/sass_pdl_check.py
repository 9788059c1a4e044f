"""Static check for PDL hazards: list, per kernel, the read-only
(LDG.*.CONSTANT, i.e. ld.global.nc) loads that ptxas scheduled BEFORE the
kernel's griddepcontrol.wait (ACQBULK). Such loads may only touch data that no
predecessor kernel writes (plan tables); data produced earlier in the stream
must be read with coherent loads (ld.global / __ldcg), which ptxas keeps after
the wait.  Usage: python scripts/sass_pdl_check.py paper_2312_00538_b200/csrc/build/*.o"""
import re
import subprocess
import sys


def main(objs):
    for o in objs:
        sass = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
        for fn in re.split(r"\n\s*Function : ", sass)[1:]:
            name = fn.split("\n", 1)[0].strip()
            lines = [l for l in fn.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
            acq = next((i for i, l in enumerate(lines) if "ACQBULK" in l), None)
            if acq is None:
                continue
            pre = [l.split(";")[0].split("*/", 1)[1].strip() for l in lines[:acq] if "CONSTANT" in l and "LDG" in l]
            print(f"{len(pre):3d} nc-loads before wait  {name[:110]}")


if __name__ == "__main__":
    main(sys.argv[1:])
