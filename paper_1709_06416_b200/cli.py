"""The reference's command-line tool (weldmill/cli.py:124-213, `weldmill run |
check ...`) with the device executor and the zero-copy bridge installed:

    PYTHONPATH=<repo> python -m paper_1709_06416_b200.cli run prog.ir --inputs m.json --out r.bin

Same arguments, exit codes (0 ok, 1 staged error as JSON on stderr, 2 usage)
and output bytes as `python -m weldmill.cli`; manifest `path` inputs go to
HBM as boundary bytes.  The weldclient SubprocessTransport drives it through
its `command` argument (client/src/weldclient/transport.py:122-128)."""
from __future__ import annotations

import sys


def main(argv=None) -> int:
    from . import install
    from weldmill import cli
    install()
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
