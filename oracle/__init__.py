"""CPU oracle for the VDAMP hot path.  Test infrastructure only: never imported by the product package."""
