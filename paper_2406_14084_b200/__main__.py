"""`python -m paper_2406_14084_b200 -i cfg.ini -c circuit.txt` == the reference `Quokka` CLI."""
import sys

from .cli import sim_main

sys.exit(sim_main())
