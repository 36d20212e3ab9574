"""The built library's SASS is free of the zeroed-pair read hazard (DESIGN.md
section 14), and the scanner recognises the sequence that faulted on the B200
(eval_kernel_tm<4096, 3, COMPACT> of the round-2 build, copied from its
cuobjdump listing)."""
import importlib.util
import os
import shutil

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("sass_hazard_scan", os.path.join(ROOT, "scripts", "sass_hazard_scan.py"))
scan = importlib.util.module_from_spec(spec)
spec.loader.exec_module(scan)

FAULTY = """
		Function : _ZN5wally14eval_kernel_tmILi4096ELi3ELi1EEEvNS_9BatchArgsE
        /*11350*/                   VIADDMNMX.U32 R30, R20, -UR6, R20, PT ;                           /* 0x800000061e1e7c46 */
                                                                                                      /* 0x000fe4000b800014 */
        /*11360*/                   CS2R R20, SRZ ;                                                   /* 0x0000000000147805 */
                                                                                                      /* 0x000fe4000001ff00 */
        /*11370*/               @P0 IMAD.WIDE.U32 R20, R65, 0x18000, R16 ;                            /* 0x0001800041140825 */
                                                                                                      /* 0x001fe400078e0010 */
        /*11380*/                   S2R R65, SR_TID.X ;                                               /* 0x0000000000417919 */
                                                                                                      /* 0x000e220000002100 */
        /*11390*/                   ISETP.NE.U32.AND P0, PT, R20, RZ, PT ;                            /* 0x000000ff1400720c */
                                                                                                      /* 0x000fc80003f05070 */
        /*113a0*/                   ISETP.NE.AND.EX P0, PT, R21, RZ, PT, P0 ;                         /* 0x000000ff1500720c */
                                                                                                      /* 0x000fe40003f05300 */
"""


def test_scanner_flags_the_faulting_sequence():
    found = scan.scan(scan.parse(FAULTY), 16)
    assert len(found) == 1
    fn, a, b, cyc, text = found[0]
    assert (a, b, cyc) == (0x11360, 0x11390, 5) and text.startswith("ISETP.NE.U32.AND P0, PT, R20")
    # a reader far enough away is not flagged, and uniform registers (UR20) are not R20
    ok = FAULTY.replace("ISETP.NE.U32.AND P0, PT, R20, RZ, PT", "ISETP.NE.U32.AND P0, PT, R70, RZ, PT") \
               .replace("ISETP.NE.AND.EX P0, PT, R21, RZ, PT, P0", "IADD3 R3, PT, PT, R4, UR20, RZ")
    assert scan.scan(scan.parse(ok), 16) == []


@pytest.mark.skipif(not shutil.which("cuobjdump") and not os.path.exists(scan.CUOBJDUMP), reason="needs cuobjdump")
def test_built_library_has_no_zeroed_pair_hazard():
    from paper_2406_06761_b200 import build
    lib = build.build()
    assert scan.main([lib, "--min-cycles", "16"]) == 0
