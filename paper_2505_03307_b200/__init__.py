"""B200-native extended-stabilizer hot path behind the reference's ``stabsim`` API."""
